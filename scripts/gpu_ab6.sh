mkdir -p gpurun_out
python scripts/gpu_plans.py
timeout 900 python bench.py --steps 5 --warmup 3 --no-pageable > gpurun_out/bench_c3.json 2>&1; tail -c 2500 gpurun_out/bench_c3.json
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-pageable > gpurun_out/bench_c4.json 2>&1; tail -c 1800 gpurun_out/bench_c4.json
bash scripts/gpu_sanitize.sh
