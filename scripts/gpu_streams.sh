mkdir -p gpurun_out
for s in 1 2 3 4 8; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-other --no-pageable --streams $s > gpurun_out/s.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/s.json').read().strip().splitlines()[-1]); print('streams $s', round(d['value']/1e9,3), 'G', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'])"
done
