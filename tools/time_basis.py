"""C2-geometry basis build (256 training frames, 512x512, Q=32, k=64): the
device builder (xg_series_build_basis, K9) against the host f64 builder
(xg_build_ring_bases, threads across rings), wall clock, plus the largest
deviation between the two V's -- a development probe."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_20356_b200 as xg  # noqa: E402


def main():
    T, H, W, Q, k = int(os.environ.get("NTRAIN", 256)), 512, 512, 32, 64
    dev = torch.device("cuda", 0)
    ctx = xg.Context(0)
    frames = torch.empty((T, H * W), dtype=torch.uint8, device=dev)
    xg.synth_speckle(ctx, frames.data_ptr(), T, H, W, Q, 0.05, 2)
    ctx.synchronize()
    ring = xg.annular_rings(H, W, Q)
    lay = xg.RingLayout(ctx, H * W, [np.nonzero(ring == r)[0] for r in range(Q)])
    s = xg.FrameSeries(lay, T)
    s.load(frames)
    basis = xg.Basis(lay, k)
    s.build_basis(k, basis=basis)  # warm-up (module load, allocations)
    ctx.synchronize()
    t0 = time.perf_counter()
    vs, sig, rank = s.build_basis(k, basis=basis)
    ctx.synchronize()
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    s.ttc_raw()
    ctx.synchronize()
    t_gram = time.perf_counter() - t0
    host = frames.cpu().numpy()
    t0 = time.perf_counter()
    vh = xg.build_ring_bases([host[:, ring == r] for r in range(Q)], k)
    t_host = time.perf_counter() - t0
    dev_max = max(float(np.abs(a - b).max()) for a, b in zip(vs, vh))
    print(f"device build_basis {t_dev * 1e3:.1f} ms (a repeat ttc_raw of the training frames: {t_gram * 1e3:.1f} ms); "
          f"host {t_host * 1e3:.1f} ms ({os.cpu_count()} cpus); max|V_dev - V_host| {dev_max:.3e}; "
          f"ranks {sorted(set(rank.tolist()))}")


if __name__ == "__main__":
    main()
