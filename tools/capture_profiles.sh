#!/bin/bash
# Round-end measurement captures (run on the GPU box from the repo root, e.g.
#   gpurun -- 'bash tools/capture_profiles.sh r2'), results into gpurun_out/,
# then copied to profiles/ and summarised with tools/make_summary.py.
# Every ncu command runs only after the same program exited 0 without ncu.
R=${1:-r2}
O=gpurun_out
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err || exit 1
python tools/prof_r2.py c2 > $O/${R}_p_c2.log 2>&1 || exit 1
python tools/prof_r2.py c2cmp > $O/${R}_p_c2cmp.log 2>&1 || exit 1
python tools/prof_r2.py c3push > $O/${R}_p_c3.log 2>&1 || exit 1
python tools/prof_r2.py c4 > $O/${R}_p_c4.log 2>&1 || exit 1
python tools/prof_r2.py c5 64 > $O/${R}_p_c5.log 2>&1 || exit 1
# launch list of the headline step (cold, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --only 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# full captures of the kernel each workload is about
$NCU -k regex:"k_ingest" -s 1 -c 1 -o $O/${R}_ingest python tools/prof_r2.py c2 > /dev/null 2>&1
$NCU -k regex:"k_gram2" -s 1 -c 1 -o $O/${R}_gram_raw python tools/prof_r2.py c2 > /dev/null 2>&1
ONLY="store+fused g2" $NCU -k regex:"k_gram2" -s 5 -c 1 -o $O/${R}_gram_cmp python tools/prof_r2.py c2cmp > /dev/null 2>&1
ONLY="store+fused g2" $NCU -k regex:"k_project" -c 1 -o $O/${R}_project python tools/prof_r2.py c2cmp > /dev/null 2>&1
# C3 streaming at history depth ~19000, raw + k=128 (push_many batches): launch list of
# the timed window, the level-1 event walk (K5e), the batched compressed columns (K6c),
# and the dense-history K5s of the single-push path (depth 8192)
DEPTH=18960 K=128 ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 9000 -c 300 \
    --log-file $O/${R}_c3_launches.csv python tools/time_batch.py > /dev/null 2>&1
DEPTH=18960 $NCU -k regex:"k_stream_events" -s 1500 -c 1 -o $O/${R}_stream_events python tools/time_batch.py > /dev/null 2>&1
DEPTH=18960 K=128 RAW=0 $NCU -k regex:"k_stream_cmp_tc" -s 1190 -c 1 -o $O/${R}_stream_cmp_tc python tools/time_batch.py > /dev/null 2>&1
$NCU -k regex:"k_stream_sparse" -s 8200 -c 1 -o $O/${R}_stream_sparse python tools/prof_r2.py c3single > /dev/null 2>&1
$NCU -k regex:"k_gram2" -s 1 -c 1 -o $O/${R}_c4_gram python tools/prof_r2.py c4 > /dev/null 2>&1
$NCU -k regex:"k_ingest" -s 2 -c 1 -o $O/${R}_c5_ingest python tools/prof_r2.py c5 64 > /dev/null 2>&1
$NCU -k regex:"k_project" -s 2 -c 1 -o $O/${R}_c5_project python tools/prof_r2.py c5 64 > /dev/null 2>&1
ls -la $O | grep $R
