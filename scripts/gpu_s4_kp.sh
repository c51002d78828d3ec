# KP (persistent EM kernel): tests, then configs 0 / 1 with and without it
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "persistent" > gpurun_out/s4_kp_tests.log 2>&1; tail -5 gpurun_out/s4_kp_tests.log
for lib in paper_1805_06572_b200/lib/libfastfca_b200.so paper_1805_06572_b200/lib/var_*.so; do
for minf in 32 16; do
  echo "== persist on, $lib MINF $minf"; FFCA_LIBRARY=$lib FFCA_PERSIST_MINF=$minf timeout 300 python profiles/all_configs.py --steps 5 --configs 0,1 --engines fast 2>&1 | cut -c1-260
done; done
echo "== persist off"; FFCA_PERSIST=0 timeout 300 python profiles/all_configs.py --steps 5 --configs 0,1 --engines fast 2>&1 | cut -c1-260
