"""The header-only C++ facade (include/xpcs_b200.hpp) driven from a C++
program: raw TTC + g2 of every ring through the RAII handles and the exact
reference-facing entry, checked against the oracle."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2407_20356_b200", "csrc", "build", "facade_smoke")


def test_cpp_facade(tmp_path, orc):
    if not os.path.exists(EXE):
        pytest.skip("facade_smoke not built")
    n, h, w, q = 90, 32, 32, 3
    frames = orc.gen_speckle(n, h, w, q, 0.4, 3)
    ring, _ = orc.ring_map(h, w, q)
    frames.tofile(tmp_path / "f.u8")
    import paper_2407_20356_b200 as xg
    xg.write_xfsr("/tmp/facade_frames.xfsr", frames, 1.0)
    ring.astype(np.int32).tofile(tmp_path / "r.i32")
    out = subprocess.run([EXE, str(tmp_path / "f.u8"), str(tmp_path / "r.i32"), str(n),
                          str(h * w), str(q)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.splitlines()
    for r in range(q):
        parts = lines[r].split()
        c = orc.ttc_raw(frames[:, ring == r].astype(np.float64))
        assert abs(float(parts[3]) - c.sum()) <= 1e-9 * c.size
        g2 = orc.g2_from_ttc(c)[1]
        assert np.allclose([float(x) for x in parts[5:8]], g2[:3], atol=1e-12, rtol=0)
    c0 = orc.ttc_raw(frames[:, ring == 0].astype(np.float64))
    basis = lines[q].split()  # device basis + compressed TTC + analysis + formats
    assert basis[:3] == ["basis", "rank", "4"] or int(basis[2]) >= 4
    assert float(basis[4]) > 0.0 and basis[7] in ("0", "1", "2")
    assert lines[q + 1] == "xfsr load equal"
    # the exact entry returns the reference's bits: same sum up to summation order
    assert abs(float(lines[q + 2].split()[-1]) - float(c0.sum())) <= 1e-12 * c0.size
    assert lines[q + 3] == "f64 load equal"
    assert lines[q + 4] == "ContractError non-integer"
    assert lines[q + 5] == "NormalizationError frame 1"
    assert lines[q + 6] == "split ring equal"
    assert lines[q + 7] == "push batch equal"
