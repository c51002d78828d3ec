for lib in paper_1805_06572_b200/lib/libfastfca_b200.so paper_1805_06572_b200/lib/var_fcaminb1.so; do echo "== $lib"; FFCA_LIBRARY=$lib python profiles/all_configs.py --steps 5 --configs 0,1 --engines fca 2>&1 | cut -c1-330; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -m gpu -k "fca or FCA or conventional" 2>&1 | tail -2
