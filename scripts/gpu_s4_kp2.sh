mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "persistent or determin or bitwise" 2>&1 | tail -2
timeout 300 python profiles/all_configs.py --steps 5 --configs 0,1 --engines fast 2>&1 | cut -c1-200
FFCA_PERSIST=1 timeout 300 python profiles/all_configs.py --steps 5 --configs 0 --engines fast 2>&1 | cut -c1-200
