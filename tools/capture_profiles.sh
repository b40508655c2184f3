#!/bin/bash
# Round-end measurement captures (run on the GPU box from the repo root, e.g.
#   gpurun -- 'bash tools/capture_profiles.sh r1'), results into gpurun_out/,
# then copied to profiles/ and summarised with tools/make_summary.py.
# Every ncu command runs only after the same program exited 0 without ncu.
R=${1:-r1}
O=gpurun_out
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err || exit 1
python tools/time_gram.py > $O/time_gram.log 2>&1 || exit 1
python tools/time_cmp.py > $O/time_cmp.log 2>&1 || exit 1
DEPTH=8192 K=128 python tools/time_stream.py > $O/time_stream.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-stream --no-compressed --no-e2e \
    > /dev/null 2>&1
$NCU -k regex:"k_ingest" -s 2 -c 1 -o $O/${R}_ingest python tools/time_gram.py > /dev/null 2>&1
$NCU -k regex:"k_gram2" -c 1 -o $O/${R}_gram_raw python tools/time_gram.py > /dev/null 2>&1
$NCU -k regex:"k_project" -c 1 -o $O/${R}_project python tools/time_cmp.py > /dev/null 2>&1
$NCU -k regex:"k_gram2" -c 1 -o $O/${R}_gram_cmp python tools/time_cmp.py > /dev/null 2>&1
# streaming: skip the history fill (3 kernels per sparse push + 3 compressed)
DEPTH=8192 K=128 $NCU --cache-control none --kernel-name-base function -k k_stream_sparse --launch-skip 8000 \
    --launch-count 1 -o $O/${R}_stream_sparse python tools/time_stream.py > /dev/null 2>&1
DEPTH=8192 K=128 $NCU --cache-control none -k regex:"k_stream_cmp" --launch-skip 8000 \
    --launch-count 1 -o $O/${R}_stream_cmp python tools/time_stream.py > /dev/null 2>&1
ls -la $O
