mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
for c in 2 4; do echo "== config $c"; bash scripts/cmp_variants.sh --config $c; done
echo "== config 2 fca"; bash scripts/cmp_variants.sh --config 2 --engine fca
