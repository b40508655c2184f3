#!/usr/bin/env python
"""Regenerate tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libxpcsvd_ref.so, built from /root/reference by oracle/Makefile).

Run in the build container (where /root/reference exists):
    make -C oracle all ref && python tests/golden/make_golden.py
The fixtures are small (seeded) and committed; the GPU box never needs
/root/reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def main():
    C, R = oracle.c(), oracle.ref()
    out = {}

    # --- RNG (rng.cpp:12-44): bits / normal / exponential of a few streams
    idx = np.array([0, 1, 2, 17, 1000, 123456789], np.uint64)
    for seed, tag in [(1, 0), (7, 1), (7, 98), (2024, 3)]:
        out[f"rng_bits_{seed}_{tag}"] = np.array([R.L.ref_rng_bits(seed, tag, int(i)) for i in idx],
                                                 np.uint64)
        out[f"rng_normal_{seed}_{tag}"] = np.array(
            [R.L.ref_rng_normal(seed, tag, int(i)) for i in idx])
        out[f"rng_exp_{seed}_{tag}"] = np.array(
            [R.L.ref_rng_exponential(seed, tag, int(i)) for i in idx])
    out["rng_idx"] = idx

    # --- reference unit-test fixtures (test_helpers.hpp:15-31)
    x = C.random_positive_matrix(8, 32, 1)
    out["ut_x_8x32"] = x
    out["ut_ttc_raw_8x32"] = R.ttc_raw(x)
    x2 = C.random_positive_matrix(20, 20000, 5)  # two 16384-pixel stripes
    out["ut_gram_20x20000"] = R.gram(x2)

    # --- BASELINE-style speckle counts, per-ring raw TTC, g2
    t, h, w, q, mu, seed = 64, 24, 24, 3, 0.5, 7
    frames = C.gen_speckle(t, h, w, q, mu, seed)
    ring, _ = C.ring_map(h, w, q)
    out["sp_frames"] = frames
    out["sp_ring"] = ring
    out["sp_params"] = np.array([t, h, w, q, mu, seed], np.float64)
    for r in range(q):
        xq = frames[:, ring == r].astype(np.float64)
        out[f"sp_gram_{r}"] = R.gram(xq)
        g = R.ttc_raw(xq)
        out[f"sp_ttc_{r}"] = g
        lags, vals, cnt = R.g2_from_ttc(g, 0.5)
        out[f"sp_g2_{r}"] = vals
        out[f"sp_g2cnt_{r}"] = cnt
        out[f"sp_g2lags_{r}"] = lags
        # compressed path with the reference's own basis (k = 8, prior = first 32 frames)
        v, spec = R.build_online_from_frames(xq[:32], 8)
        out[f"sp_v_{r}"] = v
        y, nrm = R.compress_series(xq, v)
        out[f"sp_y_{r}"] = y
        out[f"sp_norms_{r}"] = nrm
        gc, ll = R.ttc_compressed(y, nrm)
        out[f"sp_cttc_{r}"] = gc
        out[f"sp_cttc_stream_{r}"] = R.ttc_extend_stream(y, nrm)
        out[f"sp_relerr_{r}"] = np.array([R.ttc_rel_error(g, gc)])
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_vectors.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
