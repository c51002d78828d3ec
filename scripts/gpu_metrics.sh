mkdir -p gpurun_out
python -m pytest tests/test_gpu_metrics.py tests/test_gpu_parity.py -q -x -k "metric or sdr or sweep or pairing or silent or shape or scale or delay or perfect or orthogonal or determin" > gpurun_out/t_metrics.log 2>&1; tail -15 gpurun_out/t_metrics.log
