mkdir -p gpurun_out
bash scripts/cmp_variants.sh
echo "== FFCA_K1=p"
FFCA_K1=p timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-other --no-pageable > gpurun_out/k1p.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/k1p.json').read().strip().splitlines()[-1]); print(d['value']/1e9, d['ms_per_step'], d['roofline']['kernel_ms_avg'])"
echo "== C4"
bash scripts/cmp_variants.sh --config 4
echo "== C2"
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-cpu --no-pageable > gpurun_out/c2.json 2>&1; tail -c 1500 gpurun_out/c2.json
python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t_par.log 2>&1; tail -2 gpurun_out/t_par.log
