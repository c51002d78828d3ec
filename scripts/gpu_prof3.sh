mkdir -p gpurun_out/ncu
for c in 0 1 2; do python profiles/timeline.py --config $c > gpurun_out/tl_c$c.txt 2>&1; tail -1 gpurun_out/tl_c$c.txt | cut -c1-1500; done
N="ncu --set full --clock-control none --import-source on -f"
$N -k regex:pencil_par_kernel --launch-skip 1 -c 1 -o gpurun_out/ncu/k1p_c2 python profiles/prof_run.py --config 2 --engine fast > gpurun_out/ncu/k1p.log 2>&1
ncu -i gpurun_out/ncu/k1p_c2.ncu-rep --page raw --csv > gpurun_out/ncu/k1p_c2_raw.csv 2>/dev/null
$N -k regex:fast_par_kernel --launch-skip 1 -c 1 -o gpurun_out/ncu/k3p_c2 python profiles/prof_run.py --config 2 --engine fast > gpurun_out/ncu/k3p.log 2>&1
ncu -i gpurun_out/ncu/k3p_c2.ncu-rep --page raw --csv > gpurun_out/ncu/k3p_c2_raw.csv 2>/dev/null
ls -la gpurun_out/ncu
