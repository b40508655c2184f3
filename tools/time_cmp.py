"""Kernel-level timing of the C2 compressed path (K3 projection, K4 compressed
Gram with fused g2) with CUDA events -- a development probe."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20356_b200 as xg  # noqa: E402


def main():
    T, H, W, Q, k = 4096, 512, 512, 32, 64
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    torch.cuda.set_stream(st)
    ctx = xg.Context(0, stream=st.cuda_stream)
    frames = torch.empty((T, H * W), dtype=torch.uint8, device=dev)
    xg.synth_speckle(ctx, frames.data_ptr(), T, H, W, Q, 0.05, 2)
    ring = xg.annular_rings(H, W, Q)
    lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)])
    s = xg.FrameSeries(lay, T)
    prior = frames[:256].cpu().numpy()
    vs = xg.build_ring_bases([prior[:, ring == r] for r in range(Q)], k)
    basis = xg.Basis(lay, k)
    for i, v in enumerate(vs):
        basis.set_ring(i, v)

    def timed(fn, n=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(n):
            fn()
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    s.load(frames)
    print("project     %.3f ms" % timed(lambda: s.compress(basis)))
    print("cgram+g2    %.3f ms" % timed(lambda: s.ttc_compressed()))
    print("cgram only  %.3f ms" % timed(lambda: s.ttc_compressed(g2=False)))
    print("bf16 +g2    %.3f ms" % timed(lambda: s.ttc_compressed(mode="bf16")))
    print("g2 only     %.3f ms" % timed(lambda: s.ttc_compressed(store=False)))
    ctx.synchronize()


if __name__ == "__main__":
    main()
