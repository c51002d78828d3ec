mkdir -p gpurun_out
for c in 3; do echo "== config $c fca"; bash scripts/cmp_variants.sh --config $c --engine fca; done
python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "fca or FCA or conventional" > gpurun_out/s4_k4_tests.log 2>&1; tail -3 gpurun_out/s4_k4_tests.log
