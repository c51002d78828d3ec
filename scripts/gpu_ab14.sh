mkdir -p gpurun_out
python scripts/gpu_plans.py 2>&1 | grep "^2 fast"
python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
echo "== config 2"; bash scripts/cmp_variants.sh --config 2
echo "== config 2 c64"; bash scripts/cmp_variants.sh --config 2 --dtype c64
