#!/usr/bin/env python
"""Benchmark of the XPCS two-time-correlation hot path (BASELINE.json metric:
"two-time corr frames/sec (raw & rank-k) at 1/2/4/8 B200; % of roofline").

Workload (configs[1], C2): T=4096 frames of 512x512 u8 photon counts,
mean 0.05 photons/pixel, Q=32 equal-width annular q-rings, seeded synthetic
speckle generated on the device.  One step = one pass of
the raw hot path over the batch: ingest (ring permutation + statistics,
K1) -> exact u8 tcgen05 Gram of every ring (K2) -> g2(tau) (K7).

  value : T / step time, frames already resident in HBM (raster order).
  e2e   : the same step through the public API with HOST frames: pinned H2D of
          the frames + step + D2H of every ring's g2, all inside the timing.
  roofline: K2 int8 tensor ops per launch / its CUDA-event duration vs the
          int8 peak measured in-run (cuBLAS int8 GEMM via torch._int_mm).
  cpu_baseline: the UNMODIFIED reference (oracle/_ref, built from
          /root/reference) on a bounded sample of rings, host cores.

`--impl reference` times the reference's own CPU path on the same config.
Multi-GPU (torchrun): rings are sharded across ranks (LPT on pixel counts),
no collective on the data path; value = T / max-over-ranks step time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = dict(name="C2", T=4096, H=512, W=512, Q=32, mu=0.05, k=64, seed=2, gamma_a=0.002)
METRIC = "two-time corr frames/sec (raw & rank-k) at 1/2/4/8 B200; % of roofline"


def lpt_shard(sizes, n):
    """Longest-processing-time assignment of rings (by pixel count) to n ranks."""
    order = sorted(range(len(sizes)), key=lambda r: -sizes[r])
    load = [0] * n
    out = [[] for _ in range(n)]
    for r in order:
        j = min(range(n), key=lambda i: load[i])
        out[j].append(r)
        load[j] += sizes[r]
    return [sorted(o) for o in out]


def gram_ops(T, ring_sizes):
    """Algorithmic int8 ops of the raw Gram: upper triangle incl. diagonal,
    2 ops per MAC: sum_q T(T+1) M_q."""
    return float(T) * (T + 1) * float(sum(ring_sizes))


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def measure_int8_peak(torch, dev):
    """cuBLAS int8 GEMM throughput (torch._int_mm, 8192^3, best of 10) as the
    int8 tensor roofline denominator (MEASURED_PEAKS.json has bf16 only)."""
    try:
        n = 8192
        a = torch.randint(-8, 8, (n, n), dtype=torch.int8, device=dev)
        b = torch.randint(-8, 8, (n, n), dtype=torch.int8, device=dev)
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        del a, b
        return 2.0 * n ** 3 / best / 1e12, "measured in-run: cuBLAS int8 GEMM (torch._int_mm 8192^3, best of 10)"
    except Exception as e:  # pragma: no cover
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return 2.0 * peaks["bf16_tflops"], f"2 x measured bf16 burst (int8 GEMM unavailable: {e})"


def reference_sample(frames_host_cols, ring_sizes, T, budget_s=12.0, max_rings=None):
    """Time the unmodified reference (ttc_raw + g2_from_ttc per ring, the
    reference's per-mask call pattern) on rings in ascending
    size until ~budget_s; extrapolate linearly in pixels at fixed T (the
    reference's work is T(T+1)/2 * M_q MACs per ring)."""
    import oracle

    R = oracle.ref()
    order = sorted(range(len(ring_sizes)), key=lambda r: ring_sizes[r])
    # start near the median ring so the sample has representative threading
    order = order[len(order) // 2:] + order[: len(order) // 2]
    spent, pix, used = 0.0, 0, []
    for r in order:
        xq = frames_host_cols(r)
        t0 = time.perf_counter()
        g = R.ttc_raw(xq)
        R.g2_from_ttc(g)
        spent += time.perf_counter() - t0
        pix += ring_sizes[r]
        used.append(r)
        if spent >= budget_s or (max_rings and len(used) >= max_rings):
            break
    total = float(sum(ring_sizes))
    t_full = spent * total / pix
    return T / t_full, used, spent, pix


def ref_threads(T, ring_sizes_used):
    ncpu = os.cpu_count() or 1
    env = int(os.environ.get("XPCS_THREADS", "0") or 0)
    budget = env if env > 0 else ncpu
    best = 1
    for m in ring_sizes_used:  # parallel_for(n, grain=max(16, 2^21/m)) (linalg.cpp:138)
        grain = max(16, (1 << 21) // m)
        best = max(best, min(budget, (T + grain - 1) // grain))
    return best


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation on the host."""
    if rank != 0:
        return
    import oracle

    cfg = CFG
    import paper_2407_20356_b200 as xg  # geometry helper only (numpy)

    orc = oracle.c()
    T, H, W, Q = cfg["T"], cfg["H"], cfg["W"], cfg["Q"]
    ring = xg.annular_rings(H, W, Q)
    sizes = [int((ring == r).sum()) for r in range(Q)]
    # the largest ring per step, full T (the reference parallelises one ring
    # at a time with grain 2^21/M_q rows, linalg.cpp:138: its biggest ring
    # gets the most host threads, so this is its best per-pixel rate);
    # frames from the same generator (host)
    r_s = max(range(Q), key=lambda r: sizes[r])
    idx = np.nonzero(ring == r_s)[0]
    # every pixel is an independent seeded chain: generate just this ring
    xq = orc.gen_speckle_pixels(T, H, W, Q, cfg["mu"], cfg["seed"], idx,
                                gamma_a=cfg["gamma_a"]).astype(np.float64)
    R = oracle.ref()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        g = R.ttc_raw(xq)
        R.g2_from_ttc(g)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    t_step = statistics.median(times)
    t_full = t_step * sum(sizes) / sizes[r_s]
    value = T / t_full
    cores = ref_threads(T, [sizes[r_s]])
    sample = (f"ring {r_s} ({sizes[r_s]} px) of {Q} at full T={T} per step (ttc_raw + g2_from_ttc), "
              f"step time scaled by sum(M_q)/M_q = {sum(sizes) / sizes[r_s]:.1f} (work is linear in "
              f"M at fixed T)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_full * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded speckle, host generator)",
        "config": {"workload": f"{cfg['name']}: raw TTC, T={T}, {H}x{W}, Q={Q}, mu={cfg['mu']}",
                   "T": T, "detector": [H, W], "rings": Q},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_compressed(args, torch, xg, ctx, stream, frames, series, ring, sizes, mine, world, dev):
    """Rank-k path on the same frames: basis per ring from a 256-frame
    training prefix (untimed, built on the device), then per step
    ingest (K1) -> int8-digit projection (K3) -> bf16x3 compressed Gram with
    fused g2 (K4)."""
    cfg = CFG
    T, k = cfg["T"], cfg["k"]
    t_train = 256
    # the basis is built on the device (K9, xg_series_build_basis: the
    # reference's build_online_from_frames per ring) from a training series
    basis = xg.Basis(series.layout, k)
    train = xg.FrameSeries(series.layout, t_train).load(frames[:t_train])
    ctx.synchronize()
    t0 = time.perf_counter()
    train.build_basis(k, basis=basis)
    ctx.synchronize()
    t_basis = time.perf_counter() - t0
    del train
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(rec=None):
        series.load(frames)
        if rec:
            rec[0].record(stream)
        series.compress(basis)
        if rec:
            rec[1].record(stream)
        series.ttc_compressed()
        if rec:
            rec[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.synchronize()
    recs = [(ev(), ev(), ev()) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record(stream)
    for i in range(args.steps):
        step(recs[i])
    b.record(stream)
    torch.cuda.synchronize()
    ctx.synchronize()
    ms = a.elapsed_time(b) / args.steps
    proj_ms = statistics.mean(r[0].elapsed_time(r[1]) for r in recs)
    cg_ms = statistics.mean(r[1].elapsed_time(r[2]) for r in recs)
    if world > 1:
        tt = torch.tensor([ms, proj_ms, cg_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms, proj_ms, cg_ms = (float(x) for x in tt)
    # deviation of the homomorphic path from the raw correlation (untimed):
    # ttc_rel_error(raw C, compressed C~) per ring on the device
    series.ttc_raw()
    rel = series.rel_error()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    my_m = float(sum(sizes[r] for r in mine))
    q = len(mine)
    kp = (k + 63) // 64 * 64
    proj_bytes = T * my_m + 3 * k * my_m + T * q * k * 8 + 3 * T * q * kp * 2
    cg_flops_alg = q * T * (T + 1) * k
    cg_flops_mma = 6 * q * T * (T + 1) * k
    nb256 = (T + 255) // 256
    cg_bytes = q * (nb256 * (nb256 + 1) // 2) * 256 * 256 * 4 + 3 * T * q * kp * 2
    return {
        "value": world * T / (ms / 1e3), "unit": "frames/s", "ms_per_step": ms, "k": k,
        "mode": "F32-accurate (3 int8 digits of V; bf16x3 split Y, 6 products, fp32 accumulate)",
        "deviation_vs_raw": {"metric": "ttc_rel_error(raw C, compressed C~) per ring",
                             "median": float(np.median(rel)), "min": float(rel.min()),
                             "max": float(rel.max())},
        "basis": f"per ring from the first {t_train} frames, built on the device (K9 "
                 f"xg_series_build_basis: Gram, Jacobi, W = Xn^T U, 2x Cholesky-QR), untimed",
        "basis_build_ms": t_basis * 1e3,
        "projection": {"kernel": "k_project (K3)", "bound": "hbm", "ms": proj_ms,
                       "achieved": proj_bytes / (proj_ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"],
                       "unit": "GB/s", "frac": proj_bytes / (proj_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                       "bytes": proj_bytes},
        "gram": {"kernel": "k_gram2<1> (K4, CTA-pair, fused g2) + fold",
                 "bound": "hbm (C~ write)", "ms": cg_ms,
                 "achieved": cg_bytes / (cg_ms / 1e3) / 1e9, "peak": peaks["hbm_gbs"],
                 "unit": "GB/s", "frac": cg_bytes / (cg_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                 "bytes": cg_bytes,
                 "bytes_note": "f32 C~ of the upper 256x256 pair tiles + the bf16 planes read",
                 "mma_tflops": cg_flops_mma / (cg_ms / 1e3) / 1e12,
                 "mma_frac_of_bf16_peak": cg_flops_mma / (cg_ms / 1e3) / 1e12 / peaks["bf16_tflops"]},
    }


def run_streaming(args, torch, xg, ctx, stream):
    """configs[2] (C3) streaming mode at a bounded history depth: 1024^2
    detector, Q=64 rings, mu=0.02, k=128.  Frames are pushed one at a time
    (the public FrameStream API, frames already on the device); each push
    ingests the frame and correlates it against the whole history of every
    ring.  Timed: n pushes at history depth D after an untimed fill."""
    H = W = 1024
    Q, mu, k, n = 64, 0.02, 128, 64
    D = args.stream_depth
    dev = torch.device("cuda", torch.cuda.current_device())
    frames = torch.empty((D + n, H * W), dtype=torch.uint8, device=dev)
    xg.synth_speckle(ctx, frames.data_ptr(), D + n, H, W, Q, mu, 7)
    ring = xg.annular_rings(H, W, Q)
    lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)])
    rng = np.random.default_rng(3)
    basis = xg.Basis(lay, k)
    for r in range(Q):  # timing does not depend on the basis values
        qm, _ = np.linalg.qr(rng.standard_normal((int((ring == r).sum()), k)))
        basis.set_ring(r, qm)
    nnz = float((frames[:256] != 0).float().mean()) * H * W
    m_total = sum(lay.ring_pixels(r) for r in range(Q))
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def timed(depth, **kw):
        s = xg.FrameStream(lay, depth + n, **kw)
        for i in range(depth):
            s.push(frames[i])
        torch.cuda.synchronize()
        ctx.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        for i in range(depth, depth + n):
            s.push(frames[i])
        b.record(stream)
        torch.cuda.synchronize()
        ctx.synchronize()
        ms = a.elapsed_time(b) / n
        del s
        return ms

    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    t_mid = D + n / 2
    ms_s = timed(D, sparse=True)
    ms_c = timed(D, sparse=True, basis=basis)
    d_dense = min(D, 4096)
    ms_d = timed(d_dense)
    dense_bytes = m_total * (d_dense + n / 2)
    sparse_bytes = nnz * t_mid
    cmp_bytes = t_mid * Q * k * 4
    return {
        "workload": f"C3: 1024x1024, Q={Q}, mu={mu}, k={k}; {n} pushes timed at history depth {D}",
        "nnz_per_frame": nnz,
        "raw_sparse": {"frames_per_s": 1e3 / ms_s, "ms_per_frame": ms_s,
                       "column_bytes_per_frame": sparse_bytes,
                       "achieved_gbs": sparse_bytes / (ms_s / 1e3) / 1e9},
        "raw_sparse_plus_compressed": {
            "frames_per_s": 1e3 / ms_c, "ms_per_frame": ms_c,
            "bytes_per_frame": sparse_bytes + cmp_bytes,
            "achieved_gbs": (sparse_bytes + cmp_bytes) / (ms_c / 1e3) / 1e9},
        "raw_dense": {"depth": d_dense, "frames_per_s": 1e3 / ms_d, "ms_per_frame": ms_d,
                      "roofline": {"kernel": "k_stream_raw (K5, whole push timed)", "bound": "hbm",
                                   "achieved": dense_bytes / (ms_d / 1e3) / 1e9, "peak": peak,
                                   "unit": "GB/s",
                                   "frac": dense_bytes / (ms_d / 1e3) / 1e9 / peak}},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-compressed", action="store_true")
    ap.add_argument("--no-stream", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--stream-depth", type=int, default=8192)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)
    import paper_2407_20356_b200 as xg

    cfg = CFG
    T, H, W, Q = cfg["T"], cfg["H"], cfg["W"], cfg["Q"]
    P = H * W
    ring = xg.annular_rings(H, W, Q)
    sizes = [int((ring == r).sum()) for r in range(Q)]
    # Multi-GPU = weak scaling over independent ring partitions (SURVEY 8(e):
    # rings are independent objects, no data-path collective): every GPU owns
    # a C2-sized partition -- its own 512x512 detector region with 32 rings
    # and its own seeded frames -- so per-GPU work is fixed as N grows and
    # `value` counts the frames of all partitions.
    mine = list(range(Q))
    # a dedicated (non-default) stream: the library launches on it and the
    # CUDA events below are recorded on it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = xg.Context(local, stream=stream.cuda_stream)

    frames = torch.empty((T, P), dtype=torch.uint8, device=dev)
    xg.synth_speckle(ctx, frames.data_ptr(), T, H, W, Q, cfg["mu"], cfg["seed"] + 1000 * rank,
                     gamma_a=cfg["gamma_a"])
    layout = xg.RingLayout(ctx, P, [np.nonzero(ring == r)[0] for r in mine])
    series = xg.FrameSeries(layout, T)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(record=None):
        series.load(frames)
        if record is not None:
            record[0].record(stream)
        series.ttc_raw()  # K2 Gram with fused g2 epilogue + g2 fold
        if record is not None:
            record[1].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    ctx.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # ---------------------------------------------------------- device-resident
    gram_ev = [(ev(), ev()) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.15)
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.kernel_launches
    t0, t1 = ev(), ev()
    t0.record(stream)
    for i in range(args.steps):
        step(gram_ev[i])
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    launches = ctx.kernel_launches - l0
    ctx.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    gram_ms = statistics.mean(a.elapsed_time(b) for a, b in gram_ev)
    if world > 1:
        tt = torch.tensor([ms, gram_ms], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms, gram_ms = float(tt[0]), float(tt[1])
    value = world * T / (ms / 1e3)  # frames of all partitions / max-over-ranks time

    # ---------------------------------------------------------- end to end
    if args.no_e2e:  # profiling runs only (tools/capture_profiles.sh launch list)
        e2e = {"skipped": "--no-e2e (profiling run)"}
    else:
        host = torch.empty((T, P), dtype=torch.uint8, pin_memory=True)
        host.copy_(frames)
        g2_out = np.empty(T)

        def step_e2e():
            # pinned H2D in chunks, overlapped with ingest + Gram (one public call)
            series.ttc_raw_host(host)
            series.g2_all()  # D2H of every ring's g2 values + counts

        for _ in range(2):
            step_e2e()
        barrier()
        torch.cuda.synchronize()
        e2e_steps = max(3, min(args.steps, 10))
        tw0 = time.perf_counter()
        for _ in range(e2e_steps):
            step_e2e()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - tw0) / e2e_steps
        if world > 1:
            tt = torch.tensor([e2e_s], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(tt[0])
        e2e = {"value": world * T / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": T * P,
               "d2h_bytes_per_step": len(mine) * T * 16, "ms_per_step": e2e_s * 1e3,
               "timing": "host wall clock around synchronous API calls"}

    # ---------------------------------------------------------- roofline
    peak, peak_src = measure_int8_peak(torch, dev)
    my_sizes = [sizes[r] for r in mine]
    ops = gram_ops(T, my_sizes)
    achieved = ops / (gram_ms / 1e3) / 1e12
    traffic = None
    try:  # DRAM bytes of K2 from the committed ncu --set full capture (per launch)
        tr = json.load(open(os.path.join(ROOT, "profiles", "r1_traffic.json")))["k_gram2<0>"]
        traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
    except Exception:
        pass
    roofline = {"bound": "tensor", "kernel": "k_gram2<0> (K2 CTA-pair, fused g2 epilogue) + g2 fold", "achieved": achieved,
                "peak": peak, "unit": "TOPS (int8)", "frac": achieved / peak,
                "peak_source": peak_src, "traffic": traffic,
                "traffic_source": "profiles/r1_traffic.json (ncu dram__bytes_read+write, one launch)",
                "work_per_launch": f"sum_q T(T+1) M_q = {ops:.4g} int8 ops",
                "kernel_ms": gram_ms, "share_of_step": gram_ms / ms,
                # the denominator is "of measured" (an in-run cuBLAS int8 GEMM, the
                # method MEASURED_PEAKS.json uses for bf16, which has no int8 entry);
                # the nominal dense int8 rate for context
                "of": "measured", "nominal": {"peak": 4500.0, "frac": achieved / 4500.0,
                                              "note": "B200 dense int8 nominal, context only"}}

    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded speckle generated on device, SURVEY.md 8(d))",
        "config": {"workload": f"{cfg['name']}: raw TTC + g2, T={T}, {H}x{W}, Q={Q}, "
                               f"mu={cfg['mu']}, all rings",
                   "T": T, "detector": [H, W], "rings": Q, "rings_this_rank": len(mine),
                   "parallelism": f"{world} independent ring partitions (one C2 detector region "
                                  f"of {Q} rings per GPU, no collective)",
                   "l2": f"inputs {T * P / 1e9:.2f} GB > 126 MB L2 (no flush needed)"},
        "roofline": roofline, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
    }

    # ---------------------------------------------------------- compressed (rank-k)
    if not args.no_compressed:
        line["compressed"] = run_compressed(args, torch, xg, ctx, stream, frames, series, ring,
                                           sizes, mine, world, dev)

    # ---------------------------------------------------------- streaming (C3)
    if not args.no_stream and world == 1:
        try:
            line["streaming"] = run_streaming(args, torch, xg, ctx, stream)
        except Exception as e:  # keep the main line
            line["streaming"] = {"failed": str(e)}

    # ---------------------------------------------------------- CPU baseline
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle

            if oracle.ref_available():
                fr_host = frames.cpu().numpy()

                def cols(r):
                    return fr_host[:, ring == r].astype(np.float64)

                v, used, spent, pix = reference_sample(cols, sizes, T, budget_s=args.cpu_budget)
                line["cpu_baseline"] = {
                    "value": v, "unit": "frames/s", "cores": ref_threads(T, [sizes[r] for r in used]),
                    "kind": "reference",
                    "sample": f"rings {used} ({pix} of {sum(sizes)} px) at full T={T}, "
                              f"ttc_raw + g2_from_ttc, {spent:.1f} s; scaled linearly in pixels"}
            else:
                line["cpu_baseline"] = {"value": None, "kind": "reference",
                                        "sample": "oracle/_ref not built"}
        except Exception as e:  # keep the GPU line even if the CPU leg fails
            line["cpu_baseline"] = {"value": None, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
