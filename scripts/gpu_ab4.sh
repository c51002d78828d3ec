mkdir -p gpurun_out/ncu
bash scripts/cmp_variants.sh
echo "== 1 stream"
bash scripts/cmp_variants.sh --streams 1
N="ncu --set full --clock-control none --import-source on -f"
$N -k regex:fca_em_kernel --launch-skip 2 -c 1 -o gpurun_out/ncu/k4img_c3 python profiles/prof_run.py --config 3 --engine fca > gpurun_out/ncu/k4img.log 2>&1
ncu -i gpurun_out/ncu/k4img_c3.ncu-rep --page raw --csv > gpurun_out/ncu/k4img_c3_raw.csv 2>/dev/null
$N -k regex:fca_em_kernel --launch-skip 1 -c 1 -o gpurun_out/ncu/k4_c3 python profiles/prof_run.py --config 3 --engine fca > gpurun_out/ncu/k4.log 2>&1
ncu -i gpurun_out/ncu/k4_c3.ncu-rep --page raw --csv > gpurun_out/ncu/k4_c3_raw.csv 2>/dev/null
ls -la gpurun_out/ncu/
