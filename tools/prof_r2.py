"""Profiling workloads at the BASELINE geometries (run under ncu on the GPU
box; each does a warm-up pass, then the pass ncu should capture):

    python tools/prof_r2.py c4          # C4: K1 + K2 over T=16384, 1024^2, Q=100
    python tools/prof_r2.py c5 K        # C5: one 4096-frame chunk, ingest + K3 at rank K
    python tools/prof_r2.py c2          # C2: the headline step
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20356_b200 as xg  # noqa: E402


def main():
    what = sys.argv[1]
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    ctx = xg.Context(0, stream=st.cuda_stream)
    if what in ("c4", "c2"):
        T, H, W, Q, mu, gm, ga = ((16384, 1024, 1024, 100, 0.05, 1, 2e-4) if what == "c4"
                                  else (4096, 512, 512, 32, 0.05, 0, 0.002))
        frames = torch.empty((T, H * W), dtype=torch.uint8, device=dev)
        xg.synth_speckle(ctx, frames.data_ptr(), T, H, W, Q, mu, 4, gamma_mode=gm, gamma_a=ga)
        ring = xg.annular_rings(H, W, Q)
        lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)],
                            shape=None if os.environ.get("LAYOUT") == "1d" else (H, W))
        s = xg.FrameSeries(lay, T)
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.load(frames).ttc_raw()
            ctx.synchronize()
            print(f"{what}: load + ttc_raw {1e3 * (time.perf_counter() - t0):.2f} ms")
        reps = int(os.environ.get("REPS", "0"))
        if reps:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(reps)]
            for a, b in ev:
                s.load(frames)
                a.record(st)
                s.ttc_raw()
                b.record(st)
            torch.cuda.synchronize()
            ms = sorted(a.elapsed_time(b) for a, b in ev)
            print(f"{what}: K2 (+fold) median {ms[len(ms) // 2]:.3f} ms, min {ms[0]:.3f} ms "
                  f"(XG_K2_GATE={os.environ.get('XG_K2_GATE', 'default')})")
    elif what == "c2cmp":
        T, H, W, Q, mu, k = 4096, 512, 512, 32, 0.05, 64
        frames = torch.empty((T, H * W), dtype=torch.uint8, device=dev)
        xg.synth_speckle(ctx, frames.data_ptr(), T, H, W, Q, mu, 2)
        ring = xg.annular_rings(H, W, Q)
        lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)])
        basis = xg.Basis(lay, k)
        xg.FrameSeries(lay, 256).load(frames[:256]).build_basis(k, basis=basis)
        s = xg.FrameSeries(lay, T).load(frames).compress(basis)
        variants = {"store+fused g2": dict(), "store, no g2": dict(g2=False),
                    "no store, fused g2": dict(store=False),
                    "no store, spectral g2": dict(store=False, spectral=True)}
        if os.environ.get("ONLY"):
            variants = {k: v for k, v in variants.items() if k == os.environ["ONLY"]}
        for name, kw in variants.items():
            for _ in range(3):
                s.ttc_compressed(**kw)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(10)]
            for a, b in ev:
                a.record(st)
                s.ttc_compressed(**kw)
                b.record(st)
            torch.cuda.synchronize()
            ms = sorted(a.elapsed_time(b) for a, b in ev)
            print(f"c2cmp {name}: median {ms[5]:.3f} ms")
    elif what == "c3push":
        H = W = 1024
        Q, mu, D, n = 64, 0.02, 8192, 256
        frames = torch.empty((D + n, H * W), dtype=torch.uint8, device=dev)
        xg.synth_speckle(ctx, frames.data_ptr(), D + n, H, W, Q, mu, 3)
        ring = xg.annular_rings(H, W, Q)
        lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)])
        sr = xg.FrameStream(lay, D + n, sparse=True)
        sr.push_many(frames[:D])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        h0 = time.perf_counter()
        sr.push_many(frames[D:])
        h1 = time.perf_counter()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        print(f"c3push host enqueue {1e6 * (h1 - h0) / n:.1f} us/push")
        nnz = float((frames[D:] != 0).float().mean()) * H * W
        gbs = nnz * (D + n / 2) / (ms / 1e3) / 1e9
        print(f"c3push depth {D}: {ms * 1e3:.1f} us/push, {gbs:.0f} GB/s of nnz*t")
    elif what == "c3single":  # single pushes (dense-history K5s), depth 8192
        H = W = 1024
        Q, mu, D, n = 64, 0.02, 8192, 64
        frames = torch.empty((D + n, H * W), dtype=torch.uint8, device=dev)
        xg.synth_speckle(ctx, frames.data_ptr(), D + n, H, W, Q, mu, 3)
        ring = xg.annular_rings(H, W, Q)
        lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)])
        sr = xg.FrameStream(lay, D + n, sparse=True)
        for i in range(D + n):
            sr.push(frames[i])
        torch.cuda.synchronize()
        print("c3single done")
    elif what == "c5":
        k = int(sys.argv[2]) if len(sys.argv) > 2 else 64
        H, W, Q, mu, ch = 1536, 2048, 128, 0.01, 4096
        ring = xg.annular_rings(H, W, Q)
        masks = [np.nonzero(ring == r)[0] for r in range(Q)]
        if os.environ.get("RINGS"):  # a subset of the rings (shorter ring-major rows)
            sel = [int(v) for v in os.environ["RINGS"].split(",")]
            masks = [masks[r] for r in sel]
            Q = len(masks)
        lay = xg.RingLayout(ctx, H * W, masks,
                            shape=None if os.environ.get("LAYOUT") == "1d" else (H, W))
        rng = np.random.default_rng(1)
        basis = xg.Basis(lay, k)
        for r in range(Q):
            qm, _ = np.linalg.qr(rng.standard_normal((masks[r].size, k)))
            basis.set_ring(r, qm)
        s = xg.FrameSeries(lay, 3 * ch, x_frames=ch)
        chunk = torch.empty((ch, H * W), dtype=torch.uint8, device=dev)
        for i in range(3):
            xg.synth_speckle(ctx, chunk.data_ptr(), ch, H, W, Q, mu, 100 + i)
            torch.cuda.synchronize()
            a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record(st)
            s.compress_chunk(basis, chunk, first=(i == 0))
            b.record(st)
            ctx.synchronize()
            print(f"c5 k={k} chunk {i} ingest + project "
                  f"{a.elapsed_time(b):.2f} ms")
    else:
        raise SystemExit(f"unknown workload {what}")


if __name__ == "__main__":
    main()
