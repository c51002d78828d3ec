mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
bash scripts/cmp_variants.sh
bash scripts/cmp_variants.sh
bash scripts/cmp_variants.sh --config 4
