"""Batched photon-event stream (push_many) at a given history depth: per-frame
time of the timed window, for the C3 geometry -- a development probe; run
it under `ncu --metrics gpu__time_duration.sum` for the per-kernel split.
  DEPTH (8192)  history frames before the timed window
  N (256)       frames timed
  K (0)         rank of a random orthonormal basis (0: raw only)
  RAW (1)       raw columns on
  SINGLE (0)    1: the timed window pushed one frame per push() call"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20356_b200 as xg  # noqa: E402


def main():
    H = W = 1024
    Q, mu = 64, 0.02
    depth = int(os.environ.get("DEPTH", 8192))
    n = int(os.environ.get("N", 256))
    k = int(os.environ.get("K", 0))
    raw = os.environ.get("RAW", "1") != "0"
    T = depth + n
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    ctx = xg.Context(0, stream=st.cuda_stream)
    frames = torch.empty((T, H * W), dtype=torch.uint8, device=dev)
    xg.synth_speckle(ctx, frames.data_ptr(), T, H, W, Q, mu, 5)
    ring = xg.annular_rings(H, W, Q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, Q)
    basis = None
    if k:
        basis = xg.Basis(lay, k)
        rng = np.random.default_rng(1)
        for r in range(Q):
            qm, _ = np.linalg.qr(rng.standard_normal((int((ring == r).sum()), k)))
            basis.set_ring(r, qm)
    s = xg.FrameStream(lay, T, sparse=True, basis=basis, raw=raw)
    s.push_many(frames[:depth])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    if os.environ.get("SINGLE", "0") == "1":
        for i in range(depth, T):
            s.push(frames[i])
    else:
        s.push_many(frames[depth:])
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    mode = "push" if os.environ.get("SINGLE", "0") == "1" else "push_many"
    print(f"depth {depth} k {k} raw {raw} {mode}: {ms * 1e3:.1f} us/frame ({1e3 / ms:.0f} frames/s)")


if __name__ == "__main__":
    main()
