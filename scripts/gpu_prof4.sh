mkdir -p gpurun_out/ncu
N="ncu --set full --clock-control none --import-source on -f"
$N -k regex:pencil_update_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu/k1_c1 python profiles/prof_run.py --config 1 --engine fast --iters 5 > gpurun_out/ncu/k1c1.log 2>&1
ncu -i gpurun_out/ncu/k1_c1.ncu-rep --page raw --csv > gpurun_out/ncu/k1_c1_raw.csv 2>/dev/null
$N -k regex:fast_em2_kernel --launch-skip 3 -c 1 -o gpurun_out/ncu/k3_c1 python profiles/prof_run.py --config 1 --engine fast --iters 5 > gpurun_out/ncu/k3c1.log 2>&1
ncu -i gpurun_out/ncu/k3_c1.ncu-rep --page raw --csv > gpurun_out/ncu/k3_c1_raw.csv 2>/dev/null


ls -la gpurun_out/ncu/k1_c1* gpurun_out/ncu/k3_c1* gpurun_out/ncu/k1_c3*
find gpurun_out -name "*.ncu-rep" -size +20M -delete; du -sh gpurun_out
