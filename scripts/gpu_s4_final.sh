# session-4 final evidence: bench lines (both arms), all configs, KP ncu capture, launch list
mkdir -p gpurun_out/ncu
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4f_bench_c3.json 2> gpurun_out/s4f_bench_c3.err; tail -c 400 gpurun_out/s4f_bench_c3.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s4f_ref_c3.json 2>&1; tail -c 300 gpurun_out/s4f_ref_c3.json
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu > gpurun_out/s4f_bench_c4.json 2>&1; tail -c 300 gpurun_out/s4f_bench_c4.json
timeout 600 python bench.py --engine fca --steps 5 --warmup 3 --no-cpu --no-e2e --no-pageable --no-other --no-extras > gpurun_out/s4f_bench_c3_fca.json 2>&1
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu --no-extras > gpurun_out/s4f_bench_c1.json 2>&1; tail -c 300 gpurun_out/s4f_bench_c1.json
timeout 900 python profiles/all_configs.py --steps 5 > gpurun_out/s4f_allcfg.jsonl 2>&1; cut -c1-200 gpurun_out/s4f_allcfg.jsonl
N="ncu --set full --clock-control none --import-source on -f"
cap() {  # name kernel-regex skip cmd...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 $N -k regex:$kre --launch-skip $skip -c 1 -o gpurun_out/ncu/$name "$@" > gpurun_out/ncu/$name.log 2>&1
  ncu -i gpurun_out/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>/dev/null
  python profiles/ncu_lines.py gpurun_out/ncu/$name.ncu-rep 25 > gpurun_out/ncu/${name}_lines.txt 2>/dev/null
  rm -f gpurun_out/ncu/$name.ncu-rep
}
PR="python profiles/prof_run.py"
cap s4f_kp_c1 fast_persist_kernel 0 $PR --config 1 --engine fast --iters 12
cap s4f_k4_c3 fca_em_kernel 1 $PR --config 3 --engine fca
cap s4f_k3p_c2 fast_par_kernel 2 $PR --config 2 --engine fast
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4f_launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-other --no-pageable --no-extras > gpurun_out/s4f_ncu_launch.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/s4f_launches_c1.csv python profiles/prof_run.py --config 1 --engine fast --iters 50 > gpurun_out/s4f_ncu_launch_c1.log 2>&1
ls gpurun_out/ncu | grep s4f
