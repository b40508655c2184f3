"""The reference's OWN acceptance suite (proj/tests/acceptance_main.cpp),
relinked with src/correlate.cpp and src/compress.cpp replaced by the B200
drop-ins in integration/ (built by `make -C oracle acceptance` where
/root/reference exists; the binaries travel to the GPU box in oracle/_ref).

Every criterion the unmodified reference passes must pass, and the reported
numbers (max |G - G~|, bitwise flags, fits) must be identical to the
unmodified build's -- the drop-in returns the reference's bits."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _run(name):
    exe = os.path.join(REF_DIR, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600, cwd=REF_DIR)
    lines = {}
    for ln in p.stdout.splitlines():
        m = re.match(r"criterion\s+(\d+)\s+(.*?)\s+(PASS|FAIL)\s+(.*)", ln)
        if m:
            lines[int(m.group(1))] = (m.group(3), m.group(4))
    return lines


def _strip_times(detail):
    return re.sub(r"\s[\d.]+s$", "", re.sub(r"speedup=\S+|octave raw-time ratio=\S+", "", detail))


def test_reference_acceptance_through_b200_dropin():
    ref = _run("acceptance_ref")
    b200 = _run("acceptance_b200")
    assert sorted(b200) == list(range(1, 11))
    for c in range(1, 11):
        if c == 6:  # wall-clock speed ratios of the host machine, not results
            continue
        assert b200[c][0] == ref[c][0], (c, b200[c], ref[c])
        assert _strip_times(b200[c][1]) == _strip_times(ref[c][1]), (c, b200[c], ref[c])
    for c in (1, 2, 3, 4, 7, 8, 9, 10):
        assert b200[c][0] == "PASS", (c, b200[c])
