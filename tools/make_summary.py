"""Regenerate profiles/<round>_summary.txt from the
ncu reports and launch list committed under profiles/ (run here, no GPU).

    python tools/make_summary.py r1
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def run(*args):
    return subprocess.run([sys.executable, *args], capture_output=True, text=True,
                          cwd=ROOT).stdout


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r2"
    lines = [f"# {rnd} launch list: ncu --metrics gpu__time_duration.sum --clock-control none "
             "(cold, serialised; compare SHARES)",
             "# command: python bench.py --steps 3 --warmup 3 --only 1 --no-cpu-baseline --no-e2e "
             "(tools/capture_profiles.sh): the device-resident raw C2 step",
             run("tools/launches.py", os.path.join(PROF, f"{rnd}_launches.csv")).rstrip(), ""]
    c3 = os.path.join(PROF, f"{rnd}_c3_launches.csv")
    if os.path.exists(c3):
        lines += ["# C3 streaming launch list: push_many (batches of 16) at history depth ~19000,",
                  "# raw photon-event + k=128 compressed columns (tools/time_batch.py DEPTH=18960 K=128,",
                  "# the timed window's launches; cold, serialised: the raw and compressed chains",
                  "# overlap on two streams live)",
                  run("tools/launches.py", c3).rstrip(), ""]
    for name in ("ingest", "gram_raw", "project", "gram_cmp", "stream_dense", "stream_sparse",
                 "stream_cmp", "stream_events", "stream_cmp_tc", "c4_gram", "c5_ingest",
                 "c5_project"):
        rep = os.path.join(PROF, f"{rnd}_{name}.ncu-rep")
        if not os.path.exists(rep):
            continue
        lines.append(f"# {rnd}_{name}.ncu-rep (ncu --set full --import-source on)")
        lines.append(run("tools/ncu_summary.py", rep).rstrip())
        lines.append("")
    open(os.path.join(PROF, f"{rnd}_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
