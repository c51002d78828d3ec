mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
for c in 0 1 2 3 4; do echo "== config $c"; bash scripts/cmp_variants.sh --config $c; done
