mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4g_bench_c3.json 2> gpurun_out/s4g_bench_c3.err; tail -c 300 gpurun_out/s4g_bench_c3.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s4g_ref_c3.json 2>&1
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu --no-extras > gpurun_out/s4g_bench_c4.json 2>&1; tail -c 300 gpurun_out/s4g_bench_c4.json
timeout 600 python bench.py --engine fca --steps 5 --warmup 3 --no-cpu --no-e2e --no-pageable --no-other --no-extras > gpurun_out/s4g_bench_c3_fca.json 2>&1
timeout 900 python profiles/all_configs.py --steps 5 > gpurun_out/s4g_allcfg.jsonl 2>&1; cut -c1-200 gpurun_out/s4g_allcfg.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4g_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-other --no-pageable --no-extras > gpurun_out/s4g_ncu_launch.log 2>&1
