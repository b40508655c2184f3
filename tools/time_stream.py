"""Streaming (C3-like) per-frame timing: dense vs sparse raw columns at a
given history depth -- a development probe."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20356_b200 as xg  # noqa: E402


def main():
    H = W = int(os.environ.get("HW", 1024))
    Q, mu = 64, 0.02
    depth = int(os.environ.get("DEPTH", 4096))
    n_time = 64
    T = depth + n_time
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    ctx = xg.Context(0, stream=st.cuda_stream)
    frames = torch.empty((T, H * W), dtype=torch.uint8, device=dev)
    xg.synth_speckle(ctx, frames.data_ptr(), T, H, W, Q, mu, 5)
    ring = xg.annular_rings(H, W, Q)
    lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)])
    nnz = float((frames[:256] != 0).float().mean()) * H * W
    k = int(os.environ.get("K", 0))
    basis = None
    if k:
        basis = xg.Basis(lay, k)
        rng = np.random.default_rng(1)
        for r in range(Q):
            qm, _ = np.linalg.qr(rng.standard_normal((int((ring == r).sum()), k)))
            basis.set_ring(r, qm)
    for sparse in (True, False):
        s = xg.FrameStream(lay, T, sparse=sparse, basis=basis)
        t0 = time.perf_counter()
        for i in range(depth):
            s.push(frames[i])
        ctx.synchronize()
        fill = time.perf_counter() - t0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(depth, T):
            s.push(frames[i])
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n_time
        byts = (nnz if sparse else H * W) * (depth + n_time / 2)
        print(f"{'sparse' if sparse else 'dense '} depth {depth}: {ms:.3f} ms/frame "
              f"({1e3 / ms:.0f} frames/s), column bytes {byts / 1e9:.2f} GB -> "
              f"{byts / ms / 1e6:.0f} GB/s; fill {fill:.1f} s")
        del s
    print(f"nnz/frame {nnz:.0f} of {H * W}")


if __name__ == "__main__":
    main()
