#!/bin/bash
# Round-end refresh after the streaming work: GPU tests, the bench line, the C3
# launch list and the K5e / K6 captures (results into gpurun_out/, then
# copied to profiles/ and summarised with tools/make_summary.py).
R=r2
O=gpurun_out
NCU="ncu --set full --import-source on --clock-control none"
python -m pytest tests -m gpu -x -q > $O/t_gpu.log 2>&1; echo pytest=$? >> $O/t_gpu.log
python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err
DEPTH=18960 K=128 ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 9000 -c 300 --log-file $O/${R}_c3_launches.csv python tools/time_batch.py > /dev/null 2>&1
DEPTH=18960 $NCU -k regex:"k_stream_events" -s 1500 -c 1 -o $O/${R}_stream_events python tools/time_batch.py > /dev/null 2>&1
DEPTH=18960 K=128 RAW=0 $NCU -k regex:"k_stream_cmp_tc" -s 1190 -c 1 -o $O/${R}_stream_cmp_tc python tools/time_batch.py > /dev/null 2>&1
echo all-done
