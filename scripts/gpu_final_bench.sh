mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/final_bench_c3.json 2> gpurun_out/final_bench_c3.err; tail -c 3500 gpurun_out/final_bench_c3.json
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref_c3.json 2>&1; tail -c 1200 gpurun_out/final_ref_c3.json
python bench.py --config 4 --steps 5 --warmup 3 --no-cpu > gpurun_out/final_bench_c4.json 2>&1; tail -c 2500 gpurun_out/final_bench_c4.json
python bench.py --dtype c64 --steps 5 --warmup 3 --no-cpu --no-e2e --no-pageable > gpurun_out/final_bench_c3_c64.json 2>&1; tail -c 1500 gpurun_out/final_bench_c3_c64.json
python profiles/all_configs.py --steps 5 > gpurun_out/final_allcfg.jsonl 2>&1; cut -c1-220 gpurun_out/final_allcfg.jsonl
