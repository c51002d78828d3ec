# session-4 checkpoint: full GPU suite, default bench (both arms), K4 ncu captures
mkdir -p gpurun_out/ncu
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4_gputest_full.log 2>&1; tail -3 gpurun_out/s4_gputest_full.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4_bench_c3.json 2> gpurun_out/s4_bench_c3.err; tail -c 3000 gpurun_out/s4_bench_c3.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s4_ref_c3.json 2>&1; tail -c 800 gpurun_out/s4_ref_c3.json
timeout 600 python bench.py --engine fca --steps 5 --warmup 3 --no-cpu --no-e2e --no-pageable --no-other --no-extras > gpurun_out/s4_bench_c3_fca.json 2>&1; tail -c 1500 gpurun_out/s4_bench_c3_fca.json
N="ncu --set full --clock-control none --import-source on -f"
cap() {  # name kernel-regex skip cmd...
  local name=$1 kre=$2 skip=$3; shift 3
  timeout 600 $N -k regex:$kre --launch-skip $skip -c 1 -o gpurun_out/ncu/$name "$@" > gpurun_out/ncu/$name.log 2>&1
  ncu -i gpurun_out/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>/dev/null
  python profiles/ncu_lines.py gpurun_out/ncu/$name.ncu-rep 25 > gpurun_out/ncu/${name}_lines.txt 2>/dev/null
  rm -f gpurun_out/ncu/$name.ncu-rep
}
PR="python profiles/prof_run.py"
cap s4_k4_c3 fca_em_kernel 1 $PR --config 3 --engine fca
cap s4_k4img_c3 fca_em_kernel 2 $PR --config 3 --engine fca
cap s4_k3_c3 fast_em2_kernel 1 $PR --config 3 --engine fast
ls gpurun_out/ncu | tail
