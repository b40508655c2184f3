"""Probe: K8 device generator vs the oracle generator across geometries."""
import numpy as np
import torch

import oracle
import paper_2407_20356_b200 as xg

o = oracle.c()
ctx = xg.Context(0)


def dev_frames(t, h, w, q, mu, seed):
    d = torch.empty((t, h * w), dtype=torch.uint8, device="cuda")
    xg.synth_speckle(ctx, d.data_ptr(), t, h, w, q, mu, seed)
    torch.cuda.synchronize()
    return d


def sub_cmp(t, h, w, q, mu, seed):
    d = dev_frames(t, h, w, q, mu, seed)
    ring = xg.annular_rings(h, w, q)
    rng = np.random.default_rng(5)
    pix = np.sort(np.concatenate([rng.choice(np.flatnonzero(ring == r), 8, replace=False)
                                  for r in range(q)]))
    a = d[:, torch.from_numpy(pix).cuda()].cpu().numpy()
    b = o.gen_speckle_pixels(t, h, w, q, mu, seed, pix)
    bad = a != b
    tb = bad.any(1)
    print("sub", (t, h, w, q, mu), "mismatch", bad.mean(), "first t", int(np.argmax(tb)) if tb.any() else -1,
          "frac t bad", tb.mean(), "by ring", [round(float(x), 3) for x in np.bincount(ring[pix], bad.mean(0), q)[:32] / 8])


for args in [(64, 512, 512, 32, 0.05, 1), (4096, 64, 64, 8, 0.05, 1), (4096, 512, 512, 32, 0.05, 1),
             (1024, 512, 512, 32, 0.05, 1)]:
    sub_cmp(*args)
