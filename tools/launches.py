"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

The launch list covers the whole bench program.  Kernels of the timed steps
(ingest, norms, Gram, projection, g2 fold, streaming) are listed with their
share of those steps; setup work outside the timed regions (device basis
build, synthetic frames, readbacks, the deviation report) is listed apart."""
import csv
import sys
from collections import defaultdict

SETUP = ("k_synth", "k_basis_s", "k_jacobi", "k_dgemm", "k_dsyrk", "k_row_norm2",
         "k_gather_rows", "k_expand", "k_rel_error", "k_g2_partial", "k_g2_div",
         "cutlass", "at::", "cublas")  # + the in-run int8 peak probe and torch helpers

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki][:70]].append(float(r[vi].replace(",", "")) / 1e3)
step = {k: v for k, v in agg.items() if not any(s in k for s in SETUP)}
setup = {k: v for k, v in agg.items() if any(s in k for s in SETUP)}
for title, group in (("timed-step kernels (share of their total)", step),
                     ("setup outside the timed regions", setup)):
    tot = sum(sum(v) for v in group.values()) or 1.0
    print(f"## {title}: {tot / 1e3:.2f} ms")
    for k, v in sorted(group.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):5d} x {sum(v)/len(v):10.1f} us  (share {sum(v)/tot:5.1%})  {k}")
