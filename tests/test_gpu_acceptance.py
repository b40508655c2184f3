"""The reference's OWN acceptance suite (proj/tests/acceptance_main.cpp),
relinked with src/correlate.cpp and src/compress.cpp replaced by the B200
drop-ins in integration/ (built by `make -C oracle acceptance` where
/root/reference exists; the binaries travel to the GPU box in oracle/_ref).

* XPCS_B200_EXACT=1 (every call on the reference-order f64 replicas): every
  criterion's status and every printed number is identical to the
  unmodified build's -- the drop-in returns the reference's bits.
* Default (ttc_raw of integer counts on the u8 tensor-core path): the same
  statuses, and every printed number within 1e-12 absolute / 1e-6 relative
  of the unmodified build (C within 1e-12 of the reference's, SURVEY
  finding 3)."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
NUM = re.compile(r"[-+]?\d+\.?\d*(?:[eE][-+]?\d+)?")


def _run(name, exact=False):
    exe = os.path.join(REF_DIR, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    env = dict(os.environ)
    env.pop("XPCS_B200_EXACT", None)
    if exact:
        env["XPCS_B200_EXACT"] = "1"
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd=REF_DIR, env=env)
    lines = {}
    for ln in p.stdout.splitlines():
        m = re.match(r"criterion\s+(\d+)\s+(.*?)\s+(PASS|FAIL)\s+(.*)", ln)
        if m:
            lines[int(m.group(1))] = (m.group(3), m.group(4))
    return lines


def _strip_times(detail):
    return re.sub(r"\s[\d.]+s$", "", re.sub(r"speedup=\S+|octave raw-time ratio=\S+", "", detail))


@pytest.fixture(scope="module")
def ref_lines():
    return _run("acceptance_ref")


def test_acceptance_exact_mode_is_bitwise(ref_lines):
    b200 = _run("acceptance_b200", exact=True)
    assert sorted(b200) == list(range(1, 11))
    for c in range(1, 11):
        if c == 6:  # wall-clock speed ratios of the host machine, not results
            continue
        assert b200[c][0] == ref_lines[c][0], (c, b200[c], ref_lines[c])
        assert _strip_times(b200[c][1]) == _strip_times(ref_lines[c][1]), (c, b200[c], ref_lines[c])
    for c in (1, 2, 3, 4, 7, 8, 9, 10):
        assert b200[c][0] == "PASS", (c, b200[c])


def test_acceptance_fast_mode_within_tolerance(ref_lines):
    b200 = _run("acceptance_b200")
    assert sorted(b200) == list(range(1, 11))
    for c in range(1, 11):
        if c == 6:
            continue
        assert b200[c][0] == ref_lines[c][0], (c, b200[c], ref_lines[c])
        a = [float(x) for x in NUM.findall(_strip_times(b200[c][1]))]
        b = [float(x) for x in NUM.findall(_strip_times(ref_lines[c][1]))]
        assert len(a) == len(b), (c, b200[c], ref_lines[c])
        for x, y in zip(a, b):
            assert abs(x - y) <= max(1e-12, 1e-6 * abs(y)), (c, x, y, b200[c], ref_lines[c])
    for c in (1, 2, 3, 4, 7, 8, 9, 10):
        assert b200[c][0] == "PASS", (c, b200[c])
