# Final evidence: ncu captures (summaries only), launch list, SDR bench
mkdir -p gpurun_out/ncu
N="ncu --set full --clock-control none --import-source on -f"
cap() {  # name kernel-regex skip cmd...
  local name=$1 kre=$2 skip=$3; shift 3
  $N -k regex:$kre --launch-skip $skip -c 1 -o gpurun_out/ncu/$name "$@" > gpurun_out/ncu/$name.log 2>&1
  ncu -i gpurun_out/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>/dev/null
  python profiles/ncu_lines.py gpurun_out/ncu/$name.ncu-rep 25 > gpurun_out/ncu/${name}_lines.txt 2>/dev/null
  rm -f gpurun_out/ncu/$name.ncu-rep
}
PR="python profiles/prof_run.py"
cap k3_c3 fast_em2_kernel 1 $PR --config 3 --engine fast
cap k3img_c3 fast_em2_kernel 2 $PR --config 3 --engine fast
cap k1_c3 pencil_update_kernel 1 $PR --config 3 --engine fast
cap k3_c4 fast_em2_kernel 1 $PR --config 4 --engine fast
cap k1p_c4 pencil_par_kernel 1 $PR --config 4 --engine fast
cap k3p_c2 fast_par_kernel 1 $PR --config 2 --engine fast
cap k1p_c2 pencil_par_kernel 1 $PR --config 2 --engine fast
cap k4_c3 fca_em_kernel 1 $PR --config 3 --engine fca
cap k4img_c3 fca_em_kernel 2 $PR --config 3 --engine fca
cap k4b_c3 fca_bin_par_kernel 1 $PR --config 3 --engine fca
cap k4p_c2 fca_par_kernel 1 $PR --config 2 --engine fca
cap k8_stats sdr_stats_kernel 1 python profiles/sdr_bench.py --pairs 256 --reps 1
cap k8_resid sdr_resid_kernel 1 python profiles/sdr_bench.py --pairs 256 --reps 1
python profiles/sdr_bench.py > gpurun_out/sdr_bench.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-other --no-pageable > gpurun_out/ncu_launch.log 2>&1
du -sh gpurun_out
