# ncu captures of the hot kernels, summarised on the box (reports are large):
# raw metrics CSV + CUDA-source CSV per capture; only reports < 12 MB are kept
mkdir -p gpurun_out/ncu
N="ncu --set full --clock-control none --import-source on -f"
cap() {  # name kernel-regex skip args...
  local name=$1 kre=$2 skip=$3; shift 3
  $N -k regex:$kre --launch-skip $skip -c 1 -o gpurun_out/ncu/$name python profiles/prof_run.py "$@" > gpurun_out/ncu/$name.log 2>&1
  ncu -i gpurun_out/ncu/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu/$name.ncu-rep --page source --csv --print-source cuda > gpurun_out/ncu/${name}_src.csv 2>/dev/null
  ncu -i gpurun_out/ncu/$name.ncu-rep --page details > gpurun_out/ncu/${name}_details.txt 2>/dev/null
  sz=$(stat -c %s gpurun_out/ncu/$name.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -gt 12000000 ]; then rm -f gpurun_out/ncu/$name.ncu-rep; fi
}
cap k3p_c2 fast_par_kernel 1 --config 2 --engine fast
cap k1p_c2 pencil_par_kernel 1 --config 2 --engine fast
cap k4_c3 fca_em_kernel 1 --config 3 --engine fca
cap k1_c3 pencil_update_kernel 1 --config 3 --engine fast
cap k3img_c3 fast_em2_kernel 2 --config 3 --engine fast
cap k3_c3 fast_em2_kernel 1 --config 3 --engine fast
cap k3_c4 fast_em2_kernel 1 --config 4 --engine fast
cap k1p_c4 pencil_par_kernel 1 --config 4 --engine fast
cap k4p_c2 fca_par_kernel 1 --config 2 --engine fca
du -sh gpurun_out/ncu; ls -la gpurun_out/ncu | head -50
