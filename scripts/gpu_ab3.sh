mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -k "fca or image or config" > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
bash scripts/cmp_variants.sh --engine fca
bash scripts/cmp_variants.sh --engine fca --config 4
bash scripts/cmp_variants.sh --engine fca --config 2
