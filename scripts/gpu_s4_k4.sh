# K4 sweep-inverse A/B: FCA parity tests, then config 3 / 4 / 1 FCA on the shipped library and the variants
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -m gpu -k "fca or FCA or conventional or determin or stage" > gpurun_out/s4_k4_tests.log 2>&1; tail -3 gpurun_out/s4_k4_tests.log
for c in 3 4; do echo "== config $c fca"; bash scripts/cmp_variants.sh --config $c --engine fca; done
