set -u
P=paper_2407_20356_b200
cp $P/libxpcs_b200.so /tmp/A.so; cp $P/libxpcs_b200_B.so /tmp/B.so
for v in A B A B; do
  cp /tmp/$v.so $P/libxpcs_b200.so
  timeout 300 python bench.py --no-stream --no-large --no-cpu-baseline --no-e2e --steps 40 > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', d['ms_per_step'], d['compressed']['ms_per_step'], d['compressed']['gram']['ms'], d['compressed']['gram']['frac'])"
done
cp /tmp/B.so $P/libxpcs_b200.so
timeout 600 python -m pytest -q -m gpu tests/test_gpu_compressed.py tests/test_gpu_baseline_sizes.py 2>&1 | tail -2
