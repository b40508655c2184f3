"""Refresh profiles/<round>_traffic.json (DRAM bytes per launch) from the
ncu --set full captures under profiles/ (run here, no GPU).

    python tools/make_traffic.py r2
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
# kernel key -> (capture, note, algorithmic bytes or None)
REPS = {
    "k_gram2<0>": ("gram_raw", "C2: frames read once (1.07 GB) + int32 upper-triangle Gram (1.07 GB)", 2147745792),
    "k_ingest": ("ingest", "C2: raster read + ring-major write", 2147483648),
    "k_project": ("project", "C2 k=64", None),
    "k_gram2<1>": ("gram_cmp", "C2 k=64: f32 C~ upper triangle + bf16 planes", 1124335616),
    "k_stream_sparse": ("stream_sparse", "C3 single push at depth 8200: nnz x t history bytes", None),
    "k_stream_events": ("stream_events", "C3 push_many: one K5e launch (16 frames x 64 rings x the level's segments)", None),
    "k_stream_cmp_tc": ("stream_cmp_tc", "C3 push_many k=128: every coefficient row read once for 16 frames (3xTF32 mma)", None),
    "k_gram2<0> C4": ("c4_gram", "C4: T=16384, 1024^2, Q=100", None),
    "k_ingest C5": ("c5_ingest", "C5 chunk of 4096 frames", None),
    "k_project C5": ("c5_project", "C5 chunk of 4096 frames, k=64", None),
}


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "ms": 1e3,
             "msecond": 1e3}
    got = {}
    for k, u, x in zip(h, units, v):
        if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            got[k] = float(x.replace(",", "")) * scale.get(u, 1)
    return got


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r2"
    res = {"source": f"profiles/{rnd}_*.ncu-rep (ncu --set full --import-source on --clock-control "
                     f"none, one launch each; tools/capture_profiles.sh {rnd})"}
    for key, (name, note, alg) in REPS.items():
        rep = os.path.join(PROF, f"{rnd}_{name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        m = metrics(rep)
        e = {"dram_read_bytes": m["dram__bytes_read.sum"], "dram_write_bytes": m["dram__bytes_write.sum"],
             "kernel_us": m["gpu__time_duration.sum"], "note": note}
        if alg:
            e["algorithmic_bytes"] = alg
        res[key] = e
    with open(os.path.join(PROF, f"{rnd}_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
