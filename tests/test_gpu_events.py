"""Photon-event batch ingest (xg_series_load_events) on the GPU.

Event-mode detectors deliver each frame as a list of (pixel, count) pairs;
the reference takes the same frames as dense rows (FrameSeries::push_back,
model.cpp:28-40).  Loading the events must give the series the dense load
gives, bit for bit: the int32 Gram equals the oracle's gram(counts), norms
and g2 equal the dense load's exactly -- on interleaved and ring-blocked
layouts, with frames that have no events, from host arrays and from device
tensors, and after a reload over an earlier series (no stale rows)."""
import numpy as np
import pytest

import paper_2407_20356_b200 as xg

pytestmark = pytest.mark.gpu


def _compare(s_ev, s_dn, frames, ring, q, orc, check_oracle=True):
    for r in range(q):
        ge, gd = s_ev.ttc(r, "gram"), s_dn.ttc(r, "gram")
        assert np.array_equal(ge, gd), r
        if check_oracle:
            assert np.array_equal(ge.astype(np.int64), orc.gram_u8(frames[:, ring == r])), r
        (ne, ze), (nd, zd) = s_ev.norms(r), s_dn.norms(r)
        assert np.array_equal(ne, nd) and ze == zd, r
        _, ve, ce = s_ev.g2(r)
        _, vd, cd = s_dn.g2(r)
        assert np.array_equal(ve, vd) and np.array_equal(ce, cd), r


@pytest.mark.parametrize("t,h,w,q,mu,seed", [
    (300, 64, 64, 8, 0.1, 71),     # interleaved rows, partial tiles
    (520, 96, 96, 5, 0.5, 72),     # dense-ish counts
])
def test_events_equal_dense_load(ctx, orc, t, h, w, q, mu, seed):
    frames = orc.gen_speckle(t, h, w, q, mu, seed)
    frames[7] = 0      # a frame without events
    frames[t - 1] = 0  # ... at the end too
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    off, pix, val = xg.frames_to_events(frames)
    assert off[8] == off[7] and off[-1] == off[-2]
    s_ev = xg.FrameSeries(lay, t).load_events(off, pix, val).ttc_raw()
    s_dn = xg.FrameSeries(lay, t).load(frames).ttc_raw()
    _compare(s_ev, s_dn, frames, ring, q, orc)
    # host lists in chunks of 256-frame column blocks, overlapped with the tiles
    s_hx = xg.FrameSeries(lay, t).ttc_raw_events_host(off, pix, val)
    _compare(s_hx, s_dn, frames, ring, q, orc, check_oracle=False)


def test_events_blocked_layout_device_tensors_and_reload(ctx, orc):
    """1024^2 with 4 rings: ring-major rows > 400 kB, so the layout is
    ring-blocked; events handed over as CUDA tensors; the series is first
    filled with other frames (dense) and then reloaded from events."""
    import torch

    t, h, w, q = 96, 1024, 1024, 4
    dev = torch.empty((t, h * w), dtype=torch.uint8, device="cuda")
    xg.synth_speckle(ctx, dev.data_ptr(), t, h, w, q, 0.05, 9)
    ring = xg.annular_rings(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    frames = dev.cpu().numpy()
    off, pix, val = xg.frames_to_events(frames)
    other = np.ascontiguousarray(frames[::-1])
    s_ev = xg.FrameSeries(lay, t).load(other).ttc_raw()
    s_ev.load_events(torch.from_numpy(off).cuda(), torch.from_numpy(pix).cuda(),
                     torch.from_numpy(val).cuda()).ttc_raw()
    s_dn = xg.FrameSeries(lay, t).load(dev).ttc_raw()
    _compare(s_ev, s_dn, frames, ring, q, orc, check_oracle=False)
    pinned = [torch.from_numpy(a).pin_memory() for a in (off, pix, val)]
    s_ev.ttc_raw_events_host(*pinned)  # the chunked host path over the same series
    _compare(s_ev, s_dn, frames, ring, q, orc, check_oracle=False)
    for r in (0, 3):  # the oracle on two rings (the 1024^2 oracle Gram is slow)
        assert np.array_equal(s_ev.ttc(r, "gram").astype(np.int64),
                              orc.gram_u8(np.ascontiguousarray(frames[:, ring == r])))


def test_events_pixel_out_of_range_raises(ctx, orc):
    t, h, w, q = 40, 32, 32, 3
    frames = orc.gen_speckle(t, h, w, q, 0.3, 5)
    ring, _ = orc.ring_map(h, w, q)
    lay = xg.RingLayout.from_ring_map(ctx, ring, q)
    off, pix, val = xg.frames_to_events(frames)
    pix = pix.copy()
    pix[3] = h * w + 5
    s = xg.FrameSeries(lay, t)
    with pytest.raises(xg.ShapeError):
        s.load_events(off, pix, val).ttc_raw()
        s.g2(0)  # the device-side check surfaces at the next synchronising call
    with pytest.raises(xg.ShapeError):
        s.load_events(off[:-1], pix, val)  # offsets do not end at len(pix)
