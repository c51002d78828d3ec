mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -x -k "singular or degenerate or silent or determin" > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
bash scripts/cmp_variants.sh
bash scripts/cmp_variants.sh
bash scripts/cmp_variants.sh --config 4
