"""Top stall / wavefront lines of one kernel in an ncu report (source page, SASS)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
g = lambda r, k: r[h.index(k)] if k in h else ""  # noqa: E731
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(g(r, S) or 0) for r in rows[2:])
print(f"total samples {tot:.0f}")
recs = sorted(rows[2:], key=lambda r: -float(g(r, S) or 0))[:n]
for r in recs:
    print(f"{float(g(r, S) or 0) / tot:6.1%}  exec={g(r, 'Instructions Executed'):>9s} "
          f"wf={g(r, 'L1 Wavefronts Shared'):>10s}/{g(r, 'L1 Wavefronts Shared Ideal'):>9s}  "
          f"{g(r, 'Source')[:70]}")
