# KP (persistent EM kernel): tests, then configs 0 / 1 with and without it
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "persistent or determin or bitwise" > gpurun_out/s4_kp_tests.log 2>&1; tail -5 gpurun_out/s4_kp_tests.log
for minf in 32 16; do
  echo "== persist on, MINF $minf"; FFCA_PERSIST=1 FFCA_PERSIST_MINF=$minf timeout 300 python profiles/all_configs.py --steps 5 --configs 0,1 --engines fast 2>&1 | cut -c1-260
done
echo "== persist off"; timeout 300 python profiles/all_configs.py --steps 5 --configs 0,1 --engines fast 2>&1 | cut -c1-260
