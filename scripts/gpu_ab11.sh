mkdir -p gpurun_out
python scripts/gpu_plans.py 2>&1 | grep "^[34] fast c128"
python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
bash scripts/cmp_variants.sh
bash scripts/cmp_variants.sh --config 4
bash scripts/cmp_variants.sh --config 1
bash scripts/cmp_variants.sh --config 0
