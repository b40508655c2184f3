#!/usr/bin/env python
"""Benchmark of the XPCS two-time-correlation hot path (BASELINE.json metric:
"two-time corr frames/sec (raw & rank-k) at 1/2/4/8 B200; % of roofline").

Headline workload (configs[1], C2): T=4096 frames of 512x512 u8 photon
counts, mean 0.05 photons/pixel, Q=32 equal-width annular q-rings, seeded
synthetic speckle generated on the device.  One step = one
pass of the raw hot path over the batch: ingest (ring permutation +
statistics, K1) -> exact u8 tcgen05 Gram of every ring (K2, fused g2) ->
g2 fold (K7).

  value : T / step time with the frames resident in HBM.  With N GPUs the
          ONE detector is sharded along q-ring boundaries (dist.plan_shards):
          every GPU holds only its pixel slice of the frames, computes its
          rings, split rings (if any) are summed on their owner, and every
          ring's g2 is gathered to rank 0 inside the timed region; value =
          T / the slowest rank's step time (strong scaling: the work is the
          same detector at every N).
  e2e   : the same step through the public API with HOST frames (pinned H2D
          overlapped with ingest + Gram, xg_series_ttc_raw_host) + D2H of
          every ring's g2; `e2e.ttc` also returns every ring's int32 TTC.
  roofline: K2 int8 tensor ops per launch / its CUDA-event duration vs the
          int8 peak measured in-run (cuBLAS int8 GEMM via torch._int_mm).
  c3 / c4 / c5 / compressed: the other BASELINE configs (streaming to
          T=20000, the 16384-frame 1024^2 raw batch, the 3-MP rank-k sweep).
  cpu_baseline: the UNMODIFIED reference (oracle/_ref, compiled from
          /root/reference) on one ring at full T, host cores.

`--impl reference` times the reference's own CPU path on the same config.
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

METRIC = "two-time corr frames/sec (raw & rank-k) at 1/2/4/8 B200; % of roofline"
C2 = dict(name="C2", T=4096, H=512, W=512, Q=32, mu=0.05, k=64, seed=2, gamma_mode=0,
          gamma_a=0.002)
C3 = dict(name="C3", T=20000, H=1024, W=1024, Q=64, mu=0.02, k=128, seed=3, gamma_mode=0,
          gamma_a=0.002)
C4 = dict(name="C4", T=16384, H=1024, W=1024, Q=100, mu=0.05, seed=4, gamma_mode=1,
          gamma_a=2e-4)
C5 = dict(name="C5", T=65536, H=1536, W=2048, Q=128, mu=0.01, ks=(16, 64, 256), seed=5,
          gamma_mode=0, gamma_a=0.002, chunk=4096)


def headline_config() -> dict:
    """The `config` object of the headline line, identical in both arms."""
    c = C2
    return {"workload": f"{c['name']} (BASELINE configs[1]): raw two-time correlation + g2 of "
                        f"every q-ring, T={c['T']}, {c['H']}x{c['W']}, Q={c['Q']}, mu={c['mu']}",
            "T": c["T"], "detector": [c["H"], c["W"]], "rings": c["Q"], "mu": c["mu"],
            "inputs": f"{c['T'] * c['H'] * c['W'] / 1e9:.2f} GB u8 > 126 MB L2 (no flush needed)"}


def host_info() -> dict:
    try:
        nproc = len(os.sched_getaffinity(0))
    except Exception:
        nproc = os.cpu_count() or 1
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": nproc, "cpu_model": model}


def ref_threads(T: int, m: int) -> int:
    """Threads the reference's gram actually runs on for one ring:
    parallel_for(n=T, grain=max(16, 2^21 / M_q)) uses min(budget,
    ceil(T / grain)) workers (linalg.cpp:62-91,127-156)."""
    env = int(os.environ.get("XPCS_THREADS", "0") or 0)
    budget = env if env > 0 else (os.cpu_count() or 1)
    grain = max(16, (1 << 21) // m)
    return max(1, min(budget, (T + grain - 1) // grain))


def reference_ring(sizes, T: int) -> int:
    """The ring one reference step times: the smallest ring on which the
    reference's gram already uses every host thread it can (so its per-pixel
    rate is its best), else the largest ring."""
    best = max(range(len(sizes)), key=lambda r: sizes[r])
    full = ref_threads(T, sizes[best])
    cands = [r for r in range(len(sizes)) if ref_threads(T, sizes[r]) >= full]
    return min(cands, key=lambda r: (sizes[r], r))


def time_reference_ring(cfg, steps: int, warmup: int):
    """ttc_raw + g2_from_ttc (the reference's per-mask call pattern,
    SPEC.md:386) of one ring at full T on the UNMODIFIED reference; returns
    (per-step seconds, ring, its pixels, all ring sizes)."""
    import oracle

    orc = oracle.c()
    T, H, W, Q = cfg["T"], cfg["H"], cfg["W"], cfg["Q"]
    ring, _ = orc.ring_map(H, W, Q)
    sizes = [int(v) for v in np.bincount(ring, minlength=Q)]
    r_s = reference_ring(sizes, T)
    idx = np.nonzero(ring == r_s)[0]
    # every pixel is an independent seeded chain: generate just this ring (host)
    xq = orc.gen_speckle_pixels(T, H, W, Q, cfg["mu"], cfg["seed"], idx,
                                gamma_mode=cfg["gamma_mode"],
                                gamma_a=cfg["gamma_a"]).astype(np.float64)
    R = oracle.ref()
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        g = R.ttc_raw(xq)
        R.g2_from_ttc(g)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    return times, r_s, sizes


def reference_fields(cfg, times, r_s, sizes):
    t_step = statistics.median(times)
    factor = sum(sizes) / sizes[r_s]
    t_full = t_step * factor
    T = cfg["T"]
    value = T / t_full
    sample = (f"ring {r_s} ({sizes[r_s]} of {sum(sizes)} px) of {cfg['name']} at full T={T} "
              f"per step: xpcs::ttc_raw + g2_from_ttc (oracle/_ref, the unmodified reference "
              f"compiled with its Release flags)")
    extra = {"measured_ms_per_sample_step": t_step * 1e3,
             "extrapolation": {"factor": factor, "ms_per_full_step": t_full * 1e3,
                               "rule": "reference work is T(T+1)/2 * M_q MACs per ring: "
                                       "linear in pixels at fixed T; full step = sample step "
                                       "x sum(M_q) / M_sample"}}
    return value, t_step, sample, extra


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation on the host
    (rank 0 only; never loads this repo's library)."""
    if rank != 0:
        return
    cfg = C2
    times, r_s, sizes = time_reference_ring(cfg, args.steps, args.warmup)
    value, t_step, sample, extra = reference_fields(cfg, times, r_s, sizes)
    hi = host_info()
    cores = ref_threads(cfg["T"], sizes[r_s])
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded speckle, host generator of the same recipe)",
        "config": headline_config(),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "reference",
                         "sample": sample, **hi},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "host": hi, **extra,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
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
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 10.0):
        """Block until nvidia-smi has produced a sample (its start-up can take
        longer than a short timed region), then mark where the region starts."""
        t0 = time.time()
        while self.proc and not self.lines and time.time() - t0 < timeout:
            time.sleep(0.01)
        self.i0 = max(0, len(self.lines) - 1)  # the last sample before the region

    def settle(self, timeout: float = 0.5):
        """After the region: wait for one sample taken after it ended."""
        n, t0 = len(self.lines), time.time()
        while self.proc and len(self.lines) <= n and time.time() - t0 < timeout:
            time.sleep(0.005)

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
        for ln in self.lines[getattr(self, "i0", 0):]:
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
                "reasons": sorted(reasons), "samples": len(sm),
                "window": "nvidia-smi every 20 ms, from the last sample before the timed "
                          "steps to the first after them"}


def measure_int8_peak(torch, dev):
    """cuBLAS int8 GEMM throughput (torch._int_mm, 8192^3, best of 10): the
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


class Env:
    """Per-process state of the GPU arm."""

    def __init__(self, args):
        import torch

        self.args = args
        self.torch = torch
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        # one GPU per process; XPCS_BENCH_BACKEND=gloo lets several processes
        # share one GPU to validate the sharded path (NCCL needs distinct GPUs)
        self.backend = os.environ.get("XPCS_BENCH_BACKEND", "nccl")
        self.local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            import torch.distributed as tdist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if self.backend == "nccl":
                tdist.init_process_group("nccl", device_id=self.dev)
            else:
                tdist.init_process_group(self.backend)
        import paper_2407_20356_b200 as xg
        from paper_2407_20356_b200 import dist

        self.xg, self.dist = xg, dist
        # one dedicated stream: the library launches on it, events are recorded on it
        self.stream = torch.cuda.Stream(self.dev)
        torch.cuda.set_stream(self.stream)
        self.ctx = xg.Context(self.local, stream=self.stream.cuda_stream)
        self.peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))

    def ev(self):
        return self.torch.cuda.Event(enable_timing=True)

    def barrier(self):
        if self.world > 1:
            self.torch.distributed.barrier()

    def max_over_ranks(self, *vals):
        if self.world == 1:
            return vals if len(vals) > 1 else vals[0]
        t = self.torch.tensor([float(v) for v in vals], dtype=self.torch.float64,
                              device=self.dev if self.backend == "nccl" else "cpu")
        self.torch.distributed.all_reduce(t, op=self.torch.distributed.ReduceOp.MAX)
        out = tuple(float(x) for x in t)
        return out if len(out) > 1 else out[0]

    def sync(self):
        self.torch.cuda.synchronize()
        self.ctx.synchronize()

    def free(self):
        import gc

        gc.collect()
        self.torch.cuda.synchronize()
        self.torch.cuda.empty_cache()


class Shard:
    """This rank's share of one detector: the ring-aligned pixel slice of the
    frames (the whole raster on one GPU), its layout and ring order."""

    def __init__(self, E: Env, cfg: dict, allow_split: bool = True):
        xg, dist = E.xg, E.dist
        T, H, W, Q = cfg["T"], cfg["H"], cfg["W"], cfg["Q"]
        self.cfg = cfg
        self.ring = xg.annular_rings(H, W, Q)
        self.masks = [np.nonzero(self.ring == r)[0] for r in range(Q)]
        self.sizes = [int(m.size) for m in self.masks]
        self.plan = dist.plan_shards(self.sizes, E.world)
        if not allow_split and self.plan.split_rings():
            self.plan = dist.plan_shards(self.sizes, E.world, tol=1e9)  # whole rings only
        if E.world == 1:
            self.pixels = None
            self.rings = list(range(Q))
            self.layout = xg.RingLayout(E.ctx, H * W, self.masks, shape=(H, W))
        else:
            self.pixels, local, self.rings = dist.rank_slice(self.plan, E.rank, self.masks)
            self.layout = xg.RingLayout(E.ctx, int(self.pixels.size), local)
        self.my_pixels = sum(self.layout.ring_pixels(i) for i in range(len(self.rings)))

    def frames(self, E: Env, T: int | None = None, seed: int | None = None):
        """Device frames of this rank's pixel slice (K8 generator; on >1 GPU
        the full raster is generated and sliced untimed, standing in for a
        detector readout that delivers each GPU its pixels)."""
        torch = E.torch
        c = self.cfg
        T = T or c["T"]
        full = torch.empty((T, c["H"] * c["W"]), dtype=torch.uint8, device=E.dev)
        E.xg.synth_speckle(E.ctx, full.data_ptr(), T, c["H"], c["W"], c["Q"], c["mu"],
                           c["seed"] if seed is None else seed, gamma_mode=c["gamma_mode"],
                           gamma_a=c["gamma_a"])
        if self.pixels is None:
            return full
        idx = torch.from_numpy(self.pixels).to(E.dev)
        E.torch.cuda.synchronize()
        sl = torch.index_select(full, 1, idx)
        del full
        return sl.contiguous()

    def describe(self, E: Env) -> str:
        if E.world == 1:
            return "1 GPU: whole detector"
        sp = self.plan.split_rings()
        return (f"{E.world} GPUs: one detector sharded along q-ring boundaries (LPT on pixel "
                f"counts, imbalance {self.plan.imbalance():.3%}, split rings {sp}); each GPU holds "
                f"only its pixel slice; split-ring shares summed on the owner; g2 all-gathered "
                f"({E.backend}) inside the timed region")


def raw_step(E, sh, series, frames, rec=None, gather=True):
    series.load(frames)
    if rec is not None:
        rec[0].record(E.stream)
    series.ttc_raw()
    if rec is not None:
        rec[1].record(E.stream)
    if E.world > 1:
        if sh.plan.split_rings():
            E.dist.reduce_split_rings(series, sh.plan, E.rank, sh.rings)
        if gather:
            E.dist.gather_g2(series, sh.plan, E.rank, sh.rings)


def time_raw(E, sh, series, frames, steps, warmup, clocks=False):
    for _ in range(warmup):
        raw_step(E, sh, series, frames)
    E.sync()
    recs = [(E.ev(), E.ev()) for _ in range(steps)]
    sampler = None
    if clocks:
        sampler = ClockSampler(E.local)
        sampler.start()
        sampler.wait_first()
    E.barrier()
    E.torch.cuda.synchronize()
    l0 = E.ctx.kernel_launches
    a, b = E.ev(), E.ev()
    a.record(E.stream)
    for i in range(steps):
        raw_step(E, sh, series, frames, recs[i])
    b.record(E.stream)
    E.torch.cuda.synchronize()
    E.barrier()
    if sampler:
        sampler.settle()
    clk = sampler.stop() if sampler else None
    launches = E.ctx.kernel_launches - l0
    E.ctx.synchronize()
    ms = a.elapsed_time(b) / steps
    gram_ms = statistics.mean(x.elapsed_time(y) for x, y in recs)
    ms, gram_ms = E.max_over_ranks(ms, gram_ms)
    return ms, gram_ms, launches, clk


def gram_ops(T, ring_sizes):
    """Algorithmic int8 ops of the raw Gram: upper triangle incl. diagonal,
    2 ops per MAC: sum_q T(T+1) M_q."""
    return float(T) * (T + 1) * float(sum(ring_sizes))


def exact_gram(x_u8):
    # counts: every partial sum < 2^53, so the f64 product is exact in any order
    x = x_u8.astype(np.float64)
    return (x @ x.T).astype(np.int64)


def parity_check(E, sh, series, frames):
    """Untimed self-check of the benchmark's own output: the smallest and a
    mid-size ring this rank owns whole -- int32 Gram bitwise against an exact
    host product of the same bytes, C and g2 against the unmodified
    reference (oracle/_ref ttc_raw + g2_from_ttc) on the small ring."""
    import oracle

    owned = [r for r in sh.plan.owned_rings(E.rank) if r not in sh.plan.split_rings()]
    if not owned:
        return {"status": "skipped", "why": "no whole ring on this rank"}
    small = min(owned, key=lambda r: sh.sizes[r])
    mid = sorted(owned, key=lambda r: sh.sizes[r])[len(owned) // 2]
    host = frames.cpu().numpy()
    out = {"rings": sorted({small, mid})}
    ref = oracle.ref() if oracle.ref_available() else None
    for r in out["rings"]:
        li = sh.rings.index(r)
        cols = (sh.masks[r] if sh.pixels is None
                else np.searchsorted(sh.pixels, sh.masks[r]))
        xq = np.ascontiguousarray(host[:, cols])
        if not np.array_equal(series.ttc(li, "gram").astype(np.int64), exact_gram(xq)):
            return {"status": "FAILED", "ring": r, "what": "int32 Gram != exact product"}
        if r == small and ref is not None:
            c_ref = ref.ttc_raw(xq.astype(np.float64))
            dc = float(np.abs(series.ttc(li, "f64") - c_ref).max())
            _, g2_ref, cnt_ref = ref.g2_from_ttc(c_ref)
            _, g2, cnt = series.g2(li)
            dg = float(np.abs(g2 - g2_ref).max())
            if dc > 1e-12 or dg > 1e-12 or not np.array_equal(cnt, cnt_ref):
                return {"status": "FAILED", "ring": r, "max_dC": dc, "max_dg2": dg}
            out.update(max_abs_dC_vs_reference=dc, max_abs_dg2_vs_reference=dg)
    out["status"] = "ok"
    out["checks"] = ("int32 Gram bitwise vs an exact host product of the same bytes; C and g2 "
                     "within 1e-12 of the unmodified reference's ttc_raw / g2_from_ttc")
    return out


def run_headline(E, line):
    """C2 raw: value, e2e, roofline, parity."""
    torch, args = E.torch, E.args
    cfg = C2
    T = cfg["T"]
    sh = Shard(E, cfg)
    frames = sh.frames(E)
    series = E.xg.FrameSeries(sh.layout, T)
    ms, gram_ms, launches, clocks = time_raw(E, sh, series, frames, args.steps, args.warmup,
                                             clocks=True)
    line.update(value=T / (ms / 1e3), ms_per_step=ms, gpu_launches=launches, clocks=clocks)
    line["parallelism"] = sh.describe(E)
    # ---------------------------------------------------------------- e2e
    if not args.no_e2e:
        host = torch.empty(tuple(frames.shape), dtype=torch.uint8, pin_memory=True)
        host.copy_(frames)
        nring = len(sh.rings)

        owned_li = [li for li, r in enumerate(sh.rings) if sh.plan.owner[r] == E.rank]
        ttc_host = torch.empty((len(owned_li), T, T), dtype=torch.int32, pin_memory=True)

        def step_e2e(ttc_out=None):
            series.ttc_raw_host(host)  # pinned H2D in chunks, overlapped with ingest + Gram
            if E.world > 1:
                if sh.plan.split_rings():
                    E.dist.reduce_split_rings(series, sh.plan, E.rank, sh.rings)
                res = E.dist.gather_g2(series, sh.plan, E.rank, sh.rings)  # to rank 0 (host)
            else:
                series.g2_all()  # D2H of every ring's g2 values + counts
            if ttc_out is not None:  # the TTC itself: every owned ring's exact int32 Gram
                for j, li in enumerate(owned_li):
                    series.ttc(li, "gram", out=ttc_out[j])

        for _ in range(2):
            step_e2e()
        E.barrier()
        E.sync()
        n_e2e = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            step_e2e()
        E.sync()
        e2e_s = E.max_over_ranks((time.perf_counter() - t0) / n_e2e)
        # the same with every ring's TTC (int32 Gram, full symmetric) read back
        n_ttc = 3
        t0 = time.perf_counter()
        for _ in range(n_ttc):
            step_e2e(ttc_host)
        E.sync()
        ttc_s = E.max_over_ranks((time.perf_counter() - t0) / n_ttc)
        g2_bytes = cfg["Q"] * T * 16
        ttc_bytes = cfg["Q"] * T * T * 4
        # the same frames as photon-event lists (what event-mode detectors
        # emit; built once outside the timed region): pinned CSR by frame ->
        # load_events (H2D of 8 (T + 1) + 5 nnz bytes, scatter into cleared
        # ring-major rows) + ttc_raw + every ring's g2 to the host
        ev = None
        if E.world == 1:
            nz = frames.nonzero()
            nnz = int(nz.shape[0])
            off = torch.zeros(T + 1, dtype=torch.int64, device=frames.device)
            off[1:] = torch.cumsum(torch.bincount(nz[:, 0], minlength=T), 0)
            ev_host = [torch.empty(tuple(a.shape), dtype=a.dtype, pin_memory=True)
                       for a in (off, nz[:, 1].to(torch.int32), frames[nz[:, 0], nz[:, 1]])]
            ev_host[0].copy_(off)
            ev_host[1].copy_(nz[:, 1].to(torch.int32))
            ev_host[2].copy_(frames[nz[:, 0], nz[:, 1]])
            del nz, off

            def step_ev():  # chunked H2D overlapped with the scatter + Gram tiles
                series.ttc_raw_events_host(*ev_host)
                series.g2_all()

            for _ in range(2):
                step_ev()
            E.sync()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                step_ev()
            E.sync()
            ev_s = (time.perf_counter() - t0) / n_e2e
            ev = {"value": T / ev_s, "unit": "frames/s", "ms_per_step": ev_s * 1e3,
                  "h2d_bytes_per_step": 8 * (T + 1) + 5 * nnz, "d2h_bytes_per_step": g2_bytes,
                  "nnz_per_frame": nnz / T,
                  "what": "public API from pinned host photon-event lists (CSR by frame: "
                          "offsets, int32 raster pixel, u8 count -- the same frames): "
                          "FrameSeries.ttc_raw_events_host (chunked H2D overlapped with the "
                          "scatter and the Gram tiles) + every ring's g2 to the host; "
                          "results bitwise those of the dense load (tests/test_gpu_events.py)"}
            del ev_host
        line["e2e"] = {
            "value": T / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": T * cfg["H"] * cfg["W"],
            "d2h_bytes_per_step": g2_bytes, "ms_per_step": e2e_s * 1e3,
            "what": "public API from pinned host frames: FrameSeries.ttc_raw_host (chunked H2D "
                    "overlapped with ingest + Gram) + every ring's g2 to the host",
            "timing": "host wall clock around synchronous API calls, max over ranks",
            "ttc": {"value": T / ttc_s, "unit": "frames/s", "ms_per_step": ttc_s * 1e3,
                    "h2d_bytes_per_step": T * cfg["H"] * cfg["W"],
                    "d2h_bytes_per_step": g2_bytes + ttc_bytes,
                    "what": "same + every ring's TTC (the exact int32 Gram, full symmetric "
                            "T x T) read back into pinned host memory, as ttc_raw returns it"}}
        if ev is not None:
            line["e2e"]["events"] = ev
        del host, ttc_host
    else:
        line["e2e"] = {"skipped": "--no-e2e (profiling run)"}
    # ---------------------------------------------------------------- roofline
    peak, peak_src = measure_int8_peak(torch, E.dev)
    my_sizes = [sh.layout.ring_pixels(i) for i in range(len(sh.rings))]
    ops = gram_ops(T, my_sizes)
    achieved = ops / (gram_ms / 1e3) / 1e12
    traffic = None
    try:  # DRAM bytes of K2 from the committed ncu --set full capture (per launch)
        tr = json.load(open(os.path.join(ROOT, "profiles", "r2_traffic.json")))["k_gram2<0>"]
        traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
    except Exception:
        pass
    line["roofline"] = {
        "bound": "tensor", "kernel": "k_gram2<0> (K2 CTA-pair, fused g2 epilogue) + g2 fold",
        "achieved": achieved, "peak": peak, "unit": "TOPS (int8)", "frac": achieved / peak,
        "peak_source": peak_src, "traffic": traffic,
        "traffic_source": "profiles/r2_traffic.json (ncu dram__bytes_read+write, one launch)",
        "work_per_launch": f"sum_q T(T+1) M_q = {ops:.4g} int8 ops (this rank's rings)",
        "kernel_ms": gram_ms, "share_of_step": gram_ms / ms, "of": "measured",
        "nominal": {"peak": 4500.0, "frac": achieved / 4500.0,
                    "note": "B200 dense int8 nominal, context only"}}
    # ---------------------------------------------------------------- parity
    try:
        line["parity"] = parity_check(E, sh, series, frames)
    except Exception as e:  # pragma: no cover
        line["parity"] = {"status": "FAILED", "error": str(e)}
    return sh, series, frames


def run_compressed(E, sh, series, frames):
    """Rank-k path on the same C2 frames (k=64): basis per ring from a
    256-frame training prefix built on the device (K9, untimed), then per
    step ingest (K1) -> int8-digit projection (K3) -> bf16x3 compressed Gram
    with fused g2 (K4)."""
    xg, args = E.xg, E.args
    cfg = C2
    T, k = cfg["T"], cfg["k"]
    t_train = 256
    basis = xg.Basis(sh.layout, k)
    train = xg.FrameSeries(sh.layout, t_train).load(frames[:t_train])
    E.sync()
    t0 = time.perf_counter()
    train.build_basis(k, basis=basis)
    E.sync()
    t_basis = time.perf_counter() - t0
    del train

    def step(rec=None):
        series.load(frames)
        if rec:
            rec[0].record(E.stream)
        series.compress(basis)
        if rec:
            rec[1].record(E.stream)
        series.ttc_compressed()
        if rec:
            rec[2].record(E.stream)
        if E.world > 1:
            E.dist.gather_g2(series, sh.plan, E.rank, sh.rings, compressed=True)

    for _ in range(args.warmup):
        step()
    E.sync()
    recs = [(E.ev(), E.ev(), E.ev()) for _ in range(args.steps)]
    E.barrier()
    E.torch.cuda.synchronize()
    a, b = E.ev(), E.ev()
    a.record(E.stream)
    for i in range(args.steps):
        step(recs[i])
    b.record(E.stream)
    E.sync()
    ms = a.elapsed_time(b) / args.steps
    proj_ms = statistics.mean(r[0].elapsed_time(r[1]) for r in recs)
    cg_ms = statistics.mean(r[1].elapsed_time(r[2]) for r in recs)
    ms, proj_ms, cg_ms = E.max_over_ranks(ms, proj_ms, cg_ms)
    # deviation of the homomorphic path from the raw correlation (untimed)
    series.ttc_raw()
    rel = series.rel_error()
    hbm = E.peaks["hbm_gbs"]
    my_m = float(sh.my_pixels)
    q = len(sh.rings)
    kp = (k + 63) // 64 * 64
    proj_bytes = T * my_m + 3 * k * my_m + T * q * k * 8 + 3 * T * q * kp * 2
    cg_flops_mma = 6 * q * T * (T + 1) * k
    cg_bytes = q * T * (T + 1) // 2 * 4 + 3 * T * q * kp * 2
    return {
        "value": T / (ms / 1e3), "unit": "frames/s", "ms_per_step": ms, "k": k,
        "workload": "C2 frames, rank k=64 per ring: ingest + projection + homomorphic TTC + g2",
        "mode": "F32-accurate (3 int8 digits of V; bf16x3 split Y, 6 products, fp32 accumulate)",
        "deviation_vs_raw": {"metric": "ttc_rel_error(raw C, compressed C~) per ring",
                             "median": float(np.median(rel)), "min": float(rel.min()),
                             "max": float(rel.max())},
        "basis": f"per ring from the first {t_train} frames, built on the device (K9 "
                 f"xg_series_build_basis: Gram, Jacobi, W = Xn^T U, 2x Cholesky-QR), untimed",
        "basis_build_ms": t_basis * 1e3,
        "projection": {"kernel": "k_project (K3)", "bound": "hbm", "ms": proj_ms,
                       "achieved": proj_bytes / (proj_ms / 1e3) / 1e9, "peak": hbm,
                       "unit": "GB/s", "frac": proj_bytes / (proj_ms / 1e3) / 1e9 / hbm,
                       "bytes": proj_bytes},
        "gram": {"kernel": "k_gram2<1> (K4, CTA-pair, fused g2) + fold",
                 "bound": "hbm (C~ write)", "ms": cg_ms,
                 "achieved": cg_bytes / (cg_ms / 1e3) / 1e9, "peak": hbm,
                 "unit": "GB/s", "frac": cg_bytes / (cg_ms / 1e3) / 1e9 / hbm,
                 "bytes": cg_bytes,
                 "bytes_note": "f32 C~ upper triangle incl. diagonal, Q T(T+1)/2 x 4 B, + the bf16 "
                               "planes read",
                 "mma_tflops": cg_flops_mma / (cg_ms / 1e3) / 1e12,
                 "mma_frac_of_bf16_peak": cg_flops_mma / (cg_ms / 1e3) / 1e12 / E.peaks["bf16_tflops"]},
    }


def run_c3(E):
    """configs[2] (C3) streaming: 1024x1024, Q=64, mu=0.02, k=128.  Frames
    are pushed one at a time through the public FrameStream API (frames
    already on the device) up to T=20000; every push ingests the frame and
    correlates it against the whole history of every ring, raw (photon-event
    mode: nnz * t bytes) and rank-k compressed.  Reported: run average and
    the tail rate over the last 1000 frames; plus the dense raw
    kernel at a bounded depth with its HBM roofline."""
    torch, xg = E.torch, E.xg
    c = C3
    T, H, W, Q, k = c["T"], c["H"], c["W"], c["Q"], c["k"]
    sh = Shard(E, c)
    frames = sh.frames(E)
    lay = sh.layout
    basis = xg.Basis(lay, k)
    train = xg.FrameSeries(lay, 256).load(frames[:256])
    try:
        train.build_basis(k, basis=basis)
        bsrc = "device-built from the first 256 frames (K9)"
    except xg.Error:  # a zero training frame in a tiny ring: timing does not depend on V
        rng = np.random.default_rng(3)
        for r in range(Q):
            qm, _ = np.linalg.qr(rng.standard_normal((lay.ring_pixels(r), k)))
            basis.set_ring(r, qm)
        bsrc = "random orthonormal (a training frame was all-zero in a small ring)"
    del train
    nnz = float((frames[:512] != 0).float().mean()) * H * W
    st = xg.FrameStream(lay, T, basis=basis, sparse=True)
    marks = {0: E.ev(), T - 1000: E.ev(), T: E.ev()}
    E.sync()
    marks[0].record(E.stream)
    st.push_many(frames[:T - 1000])  # one library call per run of frames (no per-frame Python)
    marks[T - 1000].record(E.stream)
    st.push_many(frames[T - 1000:])
    marks[T].record(E.stream)
    E.sync()
    avg_ms = marks[0].elapsed_time(marks[T]) / T
    tail_ms = marks[T - 1000].elapsed_time(marks[T]) / 1000
    t_tail = T - 500
    raw_bytes_tail = nnz * t_tail
    cmp_bytes_tail = t_tail * Q * k * 4
    del st
    # the same run with frames handed over strictly one at a time (push():
    # each frame's columns formed before the next frame is looked at; the
    # dense pixel-major raw column and K6b's per-frame compressed column)
    st = xg.FrameStream(lay, T, basis=basis, sparse=True)
    marks = {0: E.ev(), T - 1000: E.ev(), T: E.ev()}
    E.sync()
    marks[0].record(E.stream)
    for i in range(T):
        if i == T - 1000:
            marks[i].record(E.stream)
        st.push(frames[i])
    marks[T].record(E.stream)
    E.sync()
    one_avg_ms = marks[0].elapsed_time(marks[T]) / T
    one_tail_ms = marks[T - 1000].elapsed_time(marks[T]) / 1000
    del st
    # raw-only photon-event pushes at depth 8192 (ingest -> K5s chained by
    # programmatic dependent launch): the push's HBM roofline on nnz * t bytes
    D8, n8 = 8192, 256
    sr = xg.FrameStream(lay, D8 + n8, sparse=True)
    sr.push_many(frames[:D8])
    E.sync()
    a, b = E.ev(), E.ev()
    a.record(E.stream)
    sr.push_many(frames[D8:D8 + n8])
    b.record(E.stream)
    E.sync()
    ms_r = a.elapsed_time(b) / n8
    nnz8 = float((frames[D8:D8 + n8] != 0).float().mean()) * H * W
    sparse_bytes = nnz8 * (D8 + n8 / 2)
    del sr
    # the same frames pushed one call per frame (push(): one frame's columns
    # per launch chain, no batch)
    sr = xg.FrameStream(lay, D8 + n8, sparse=True)
    sr.push_many(frames[:D8])
    E.sync()
    a, b = E.ev(), E.ev()
    a.record(E.stream)
    for i in range(D8, D8 + n8):
        sr.push(frames[i])
    b.record(E.stream)
    E.sync()
    ms_r1 = a.elapsed_time(b) / n8
    del sr
    # dense raw column (K5) at a bounded history depth: the HBM roofline
    D, n = 4096, 64
    sd = xg.FrameStream(lay, D + n)
    sd.push_many(frames[:D])
    E.sync()
    a, b = E.ev(), E.ev()
    a.record(E.stream)
    sd.push_many(frames[D:D + n])
    b.record(E.stream)
    E.sync()
    ms_d = a.elapsed_time(b) / n
    dense_bytes = sh.my_pixels * (D + n / 2)
    hbm = E.peaks["hbm_gbs"]
    del sd, frames
    E.free()
    return {
        "workload": f"C3 (configs[2]): {H}x{W}, Q={Q}, mu={c['mu']}, k={k}; frames pushed one "
                    f"at a time to T={T}, each correlated against the whole history (raw "
                    f"photon-event columns + rank-k compressed columns + g2 per lag)",
        "frames_per_s_avg": 1e3 / avg_ms, "ms_per_frame_avg": avg_ms,
        "frames_per_s_tail": 1e3 / tail_ms, "ms_per_frame_tail": tail_ms,
        "tail": "last 1000 frames (history depth 19000-20000)",
        "mode": "push_many: frames handed over in runs; the library forms 16 frames' columns "
                "together (history read once per 16 columns; results bitwise those of single "
                "pushes)",
        "one_at_a_time": {"frames_per_s_avg": 1e3 / one_avg_ms, "ms_per_frame_avg": one_avg_ms,
                          "frames_per_s_tail": 1e3 / one_tail_ms,
                          "ms_per_frame_tail": one_tail_ms,
                          "what": "push() per frame from Python (host call per frame inside the "
                                  "timed region): ingest, dense pixel-major raw column (K5s), "
                                  "K6a projection + K6 tensor-core compressed column"},
        "nnz_per_frame": nnz, "basis": bsrc,
        "tail_bytes_per_frame": {"raw_nnz_history": raw_bytes_tail,
                                 "compressed_history": cmp_bytes_tail,
                                 "achieved_gbs": (raw_bytes_tail + cmp_bytes_tail) / (tail_ms / 1e3) / 1e9},
        "raw_sparse_push": {
            "depth": D8, "frames_per_s": 1e3 / ms_r, "ms_per_frame": ms_r,
            "what": "raw-only photon-event stream through push_many (batches of 16: one ingest; "
                    "sealed 1024-frame event blocks merged into 8192-frame segments read by K5e "
                    "(per-pixel event lists), the unsealed tail by one K5s grid over the batch's "
                    "frames; in-order lag fold), whole batch timed incl. the block seal that "
                    "falls in the window",
            "event_history_speedup_vs_dense_column": ms_r1 / ms_r,
            "single_push": {"frames_per_s": 1e3 / ms_r1, "ms_per_frame": ms_r1,
                            "frac_of_hbm": sparse_bytes / (ms_r1 / 1e3) / 1e9 / E.peaks["hbm_gbs"],
                            "what": "push() per frame: ingest -> K5s over the dense pixel-major "
                                    "history (nnz x t bytes), chained by programmatic dependent "
                                    "launch"},
            "roofline": {"kernel": "push_many (K1s + K5e + K5s + fold): DENSE-EQUIVALENT rate -- "
                                   "the event path reads ~1/5 of these bytes, so frac > 1 is "
                                   "algorithmic, not a bandwidth claim; K5e itself is latency-bound "
                                   "(profiles/r2_summary.txt)",
                         "bound": "hbm", "bytes_per_frame": sparse_bytes,
                         "bytes_note": "nnz x t: the new frame's nonzero pixels' history rows",
                         "achieved": sparse_bytes / (ms_r / 1e3) / 1e9, "peak": hbm,
                         "unit": "GB/s", "frac": sparse_bytes / (ms_r / 1e3) / 1e9 / hbm}},
        "raw_dense": {"depth": D, "frames_per_s": 1e3 / ms_d, "ms_per_frame": ms_d,
                      "roofline": {"kernel": "k_stream_raw (K5, whole push timed)", "bound": "hbm",
                                   "achieved": dense_bytes / (ms_d / 1e3) / 1e9, "peak": hbm,
                                   "unit": "GB/s",
                                   "frac": dense_bytes / (ms_d / 1e3) / 1e9 / hbm}},
    }


def run_c4(E, peak):
    """configs[3] (C4): T=16384 frames of 1024x1024, Q=100 rings with
    log-spaced Gamma_q (3 decades), raw exact Gram + g2 of every ring, TTC
    stored (107 GB of int32 tiles on one GPU).  Sharded along q-ring
    boundaries on >1 GPU."""
    c = C4
    T = c["T"]
    sh = Shard(E, c)
    frames = sh.frames(E)
    series = E.xg.FrameSeries(sh.layout, T)
    ms, gram_ms, launches, _ = time_raw(E, sh, series, frames, 3, 2)
    my_sizes = [sh.layout.ring_pixels(i) for i in range(len(sh.rings))]
    ops = gram_ops(T, my_sizes)
    out = {
        "workload": f"C4 (configs[3]): raw TTC + g2, T={T}, {c['H']}x{c['W']}, Q={c['Q']}, "
                    f"mu={c['mu']}, Gamma_q = {c['gamma_a']} x 10^(3q/(Q-1))",
        "frames_per_s": T / (ms / 1e3), "ms_per_step": ms, "parallelism": sh.describe(E),
        "roofline": {"kernel": "k_gram2<0>", "bound": "tensor", "kernel_ms": gram_ms,
                     "achieved": ops / (gram_ms / 1e3) / 1e12, "peak": peak,
                     "unit": "TOPS (int8)", "frac": ops / (gram_ms / 1e3) / 1e12 / peak},
    }
    del series, frames
    E.free()
    return out


def run_c5(E):
    """configs[4] (C5): 1536x2048 detector, T=65536, mu=0.01, Q=128, k in
    {16, 64, 256}: frames arrive in chunks of 4096 (generated on the device,
    untimed; 206 GB never resident), every chunk is ingested and projected
    for the three ranks (timed), then the homomorphic g2 of every ring is
    formed without storing C~ (2.2 TB): through the K4 tiles (fused g2) and
    in the Fourier domain (spectral).  Bases: random orthonormal (timing does
    not depend on V)."""
    torch, xg = E.torch, E.xg
    c = C5
    T, ch = c["T"], c["chunk"]
    sh = Shard(E, c, allow_split=False)
    lay = sh.layout
    rng = np.random.default_rng(5)
    ks = c["ks"]
    # (k, 2): the same basis kept as 2 int8 digits per column (~8e-6 of
    # max|V|, inside the 1e-2 bar BASELINE sets for C5's bf16 projection):
    # two thirds of K3's tensor work, timed where K3 is tensor-bound
    k2 = max(ks)
    bases, series = {}, {}
    for k in ks:
        b = xg.Basis(lay, k)
        b2 = xg.Basis(lay, k, digits=2) if k == k2 else None
        for i in range(len(sh.rings)):
            qm, _ = np.linalg.qr(rng.standard_normal((lay.ring_pixels(i), k)))
            b.set_ring(i, qm)
            if b2 is not None:
                b2.set_ring(i, qm)
        bases[k] = b
        series[k] = xg.FrameSeries(lay, T, x_frames=ch)
        if b2 is not None:
            bases[(k, 2)] = b2
            series[(k, 2)] = xg.FrameSeries(lay, T, x_frames=ch)
    variants = list(ks) + [(k2, 2)]
    t_cmp = {v: 0.0 for v in variants}
    full = None
    for j, f0 in enumerate(range(0, T, ch)):
        n = min(ch, T - f0)
        seed = c["seed"] * 1000 + j  # each chunk: a fresh stationary stretch of the series
        if sh.pixels is None:
            if full is None:
                full = torch.empty((ch, c["H"] * c["W"]), dtype=torch.uint8, device=E.dev)
            xg.synth_speckle(E.ctx, full.data_ptr(), n, c["H"], c["W"], c["Q"], c["mu"], seed,
                             gamma_mode=c["gamma_mode"], gamma_a=c["gamma_a"])
            chunk = full[:n]
        else:
            chunk = sh.frames(E, T=n, seed=seed)
        for k in variants:
            if j == 0:  # untimed warm-up: the basis' one-time digit upload and tile lists
                series[k].compress_chunk(bases[k], chunk, first=True)
                E.sync()
            a, b = E.ev(), E.ev()
            a.record(E.stream)
            series[k].compress_chunk(bases[k], chunk, first=(j == 0))
            b.record(E.stream)
            b.synchronize()
            t_cmp[k] += a.elapsed_time(b) / 1e3
    del full
    out = {"workload": f"C5 (configs[4]): {c['H']}x{c['W']} ({c['H'] * c['W']} px), T={T}, "
                       f"mu={c['mu']}, Q={c['Q']}; chunks of {ch} frames ingested + projected "
                       f"(K1 + K3) per rank k, then homomorphic g2 without storing C~",
           "parallelism": sh.describe(E), "by_k": {}}
    hbm = E.peaks["hbm_gbs"]
    del series[(k2, 2)], bases[(k2, 2)]  # timed above; its g2 is the 3-digit series' (same k)
    E.free()
    for k in ks:
        s = series.pop(k)  # one k at a time: the g2 tile partials of T=65536 are 26 GB
        E.sync()
        s.ttc_compressed(store=False)  # warm
        E.sync()
        a, b = E.ev(), E.ev()
        a.record(E.stream)
        s.ttc_compressed(store=False)
        b.record(E.stream)
        E.sync()
        t_tiles = a.elapsed_time(b) / 1e3
        s.ttc_compressed(store=False, spectral=True)
        E.sync()
        a, b = E.ev(), E.ev()
        a.record(E.stream)
        s.ttc_compressed(store=False, spectral=True)
        b.record(E.stream)
        E.sync()
        t_spec = a.elapsed_time(b) / 1e3
        tc, tt, ts = E.max_over_ranks(t_cmp[k], t_tiles, t_spec)
        ingest_bytes = 3.0 * T * sh.my_pixels  # K1 raster read + ring-major write, K3 read
        proj_ops = 2.0 * T * sh.my_pixels * 3 * k  # K3: u8 x s8 over 3 int8 digits per column
        out["by_k"][str(k)] = {
            "ingest_project_s": tc, "frames_per_s_ingest_project": T / tc,
            "g2_tiles_s": tt, "g2_spectral_s": ts,
            "frames_per_s_total_tiles": T / (tc + tt), "frames_per_s_total_spectral": T / (tc + ts),
            "ingest_project_hbm": {"bytes": ingest_bytes, "achieved_gbs": ingest_bytes / tc / 1e9,
                                   "frac": ingest_bytes / tc / 1e9 / hbm,
                                   "note": "K1 reads the raster + writes the ring-major copy, K3 "
                                           "re-reads it (3 B per pixel per frame)"},
            "projection_int8_tops_over_ingest_project": proj_ops / tc / 1e12,
            "bound": ("hbm" if k <= 64 else
                      "tensor: K3 alone runs 7.12 ms per 4096-frame chunk = 2.78 POPS, 0.87 of the "
                      "cuBLAS int8 GEMM (profiles/r2_c5_project_k256.ncu-rep); the hbm frac above "
                      "is not the bound at this k"),
            "projection_note": "2 T M 3k int8 ops (3 digits); at k = 256 K3 is tensor-bound "
                               "(ops / the whole K1 + K3 time, a lower bound on K3's rate)"}
        del s
        E.free()
    tc2 = E.max_over_ranks(t_cmp[(k2, 2)])
    out["by_k"][str(k2)]["two_digit_projection"] = {
        "ingest_project_s": tc2, "frames_per_s_ingest_project": T / tc2,
        "projection_int8_tops_over_ingest_project": 2.0 * T * sh.my_pixels * 2 * k2 / tc2 / 1e12,
        "note": "V as 2 int8 digits per column (coefficients within 5e-5 of max|Y|, g2 within "
                "1e-3: tests/test_gpu_baseline_sizes.py; BASELINE's bar for C5's bf16 "
                "projection is 1e-2); the g2 steps are the 3-digit ones' (same k)"}
    del series, bases
    E.free()
    return out


def run_dropin(E, sh, frames):
    """The reference's own API through the drop-in source (integration/
    correlate_b200.cpp linked into a reference program, oracle/_ref/
    dropin_bench): xpcs::ttc_raw + g2_from_ttc of the ring the CPU baseline
    times, f64 host frames in, the full f64 TTC out -- what a reference user
    gets by swapping src/correlate.cpp.  Host wall clock, best of 3."""
    import tempfile

    exe = os.path.join(ROOT, "oracle", "_ref", "dropin_bench")
    if not os.path.exists(exe):
        return {"skipped": "oracle/_ref/dropin_bench not built (needs /root/reference at build time)"}
    T = C2["T"]
    r_s = reference_ring(sh.sizes, T)
    cols = E.torch.from_numpy(sh.masks[r_s]).to(E.dev)
    xq = E.torch.index_select(frames, 1, cols).cpu().numpy()
    with tempfile.NamedTemporaryFile(suffix=".u8", delete=False) as f:
        f.write(np.ascontiguousarray(xq).tobytes())
        path = f.name
    try:
        out = subprocess.run([exe, path, str(T), str(xq.shape[1]), "3"], capture_output=True,
                             text=True, timeout=300)
        res = json.loads(out.stdout.strip().splitlines()[-1])
    finally:
        os.unlink(path)
    factor = sum(sh.sizes) / sh.sizes[r_s]
    return {"what": "xpcs::ttc_raw + xpcs::g2_from_ttc through integration/correlate_b200.cpp "
                    "(u8 tensor-core path for integer counts), f64 FrameSeries in, f64 TTCMatrix "
                    "+ G2Curve out, called from a C++ program linked like the reference",
            "ring": r_s, "ring_pixels": sh.sizes[r_s], "T": T, "ms_per_call": res["ms_best"],
            "ms_mean": res["ms_mean"],
            "frames_per_s_extrapolated": T / (res["ms_best"] / 1e3 * factor),
            "extrapolation": f"x sum(M_q) / M_ring = {factor:.2f} (as cpu_baseline)"}


def cpu_baseline(E, args):
    cfg = C2
    times, r_s, sizes = time_reference_ring(cfg, 1, 0)
    value, t_step, sample, extra = reference_fields(cfg, times, r_s, sizes)
    hi = host_info()
    return {"value": value, "unit": "frames/s", "cores": ref_threads(cfg["T"], sizes[r_s]),
            "kind": "reference", "sample": sample, **hi, **extra}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compressed", action="store_true")
    ap.add_argument("--no-stream", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-large", action="store_true", help="skip C4 and C5")
    ap.add_argument("--only", default="", help="profiling: run only the headline step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    E = Env(args)
    if args.only in ("c3", "c5"):  # development: one section alone
        print(json.dumps(run_c3(E) if args.only == "c3" else run_c5(E)), flush=True)
        return
    line = {"metric": METRIC, "value": None, "unit": "frames/s", "n_gpus": E.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded speckle generated on device, SURVEY.md 8(d))",
            "config": headline_config()}
    sh, series, frames = run_headline(E, line)
    if not args.no_compressed and not args.only:
        line["compressed"] = run_compressed(E, sh, series, frames)
    if E.world == 1 and not args.only:
        try:
            line["dropin"] = run_dropin(E, sh, frames)
        except Exception as e:  # keep the main line
            line["dropin"] = {"failed": repr(e)}
    del series, frames
    E.free()
    if not args.only:
        if not args.no_stream and E.world == 1:
            try:
                line["c3_streaming"] = run_c3(E)
            except Exception as e:  # keep the main line
                line["c3_streaming"] = {"failed": repr(e)}
        if not args.no_large:
            for key, fn in (("c4_raw", lambda: run_c4(E, line["roofline"]["peak"])),
                            ("c5_compressed", lambda: run_c5(E))):
                try:
                    line[key] = fn()
                except Exception as e:  # keep the main line
                    line[key] = {"failed": repr(e)}
                    E.free()
    if E.rank == 0 and E.world == 1 and not args.no_cpu_baseline and not args.only:
        try:
            line["cpu_baseline"] = cpu_baseline(E, args)
        except Exception as e:  # keep the GPU line even if the CPU leg fails
            line["cpu_baseline"] = {"value": None, "kind": "reference", "sample": f"failed: {e}"}
    if E.rank == 0:
        print(json.dumps(line), flush=True)
    if E.world > 1:
        E.torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
