#!/bin/bash
# A/B of library variants on one box: variant V is paper_2407_20356_b200/
# libxpcs_b200_V.so (built with `make -C .../csrc OUT=... OBJDIR=... XG_EXTRA=-D...`),
# "base" is the in-tree build.  Each variant runs the C2 headline + compressed
# bench twice, interleaved; prints step / compressed step / K3 / K4 times.
set -u
P=paper_2407_20356_b200
cp $P/libxpcs_b200.so /tmp/v_base.so
VARS="base"
for f in $P/libxpcs_b200_*.so; do v=${f#$P/libxpcs_b200_}; v=${v%.so}; cp $f /tmp/v_$v.so; VARS="$VARS $v"; done
for rep in 1 2; do
  for v in $VARS; do
    cp /tmp/v_$v.so $P/libxpcs_b200.so
    timeout 300 python bench.py --no-stream --no-large --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/ab_$v.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));c=d['compressed'];print('$v', round(d['ms_per_step'],4), round(c['ms_per_step'],4), 'K3', round(c['projection']['ms'],4), c['projection']['frac'], 'K4', round(c['gram']['ms'],4))"
  done
done
cp /tmp/v_base.so $P/libxpcs_b200.so
