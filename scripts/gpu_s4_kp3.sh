mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "persistent or determin or bitwise" 2>&1 | tail -2
for lar in 1 0; do
echo "== LAR $lar"; FFCA_PERSIST_LAR=$lar FFCA_PERSIST=1 timeout 300 python profiles/all_configs.py --steps 5 --configs 0,1 --engines fast 2>&1 | cut -c1-200
done
echo "== plain"; FFCA_PERSIST=0 timeout 300 python profiles/all_configs.py --steps 5 --configs 0,1 --engines fast 2>&1 | cut -c1-200
