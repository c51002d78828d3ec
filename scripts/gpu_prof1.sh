# GPU session: full GPU tests, all-config throughput, C2 timeline, ncu captures
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
python profiles/all_configs.py --steps 3 > gpurun_out/allcfg.jsonl 2>&1; tail -c 600 gpurun_out/allcfg.jsonl
python profiles/timeline.py --config 2 > gpurun_out/tl_c2.txt 2>&1; tail -20 gpurun_out/tl_c2.txt
N="ncu --set full --clock-control none --import-source on -f"
$N -k regex:fast_par_kernel --launch-skip 1 -c 1 -o gpurun_out/k3p_c2 python profiles/prof_run.py --config 2 --engine fast > gpurun_out/ncu1.log 2>&1
$N -k regex:pencil_par_kernel --launch-skip 1 -c 1 -o gpurun_out/k1p_c2 python profiles/prof_run.py --config 2 --engine fast > gpurun_out/ncu2.log 2>&1
$N -k regex:fca_em_kernel --launch-skip 1 -c 1 -o gpurun_out/k4_c3 python profiles/prof_run.py --config 3 --engine fca > gpurun_out/ncu3.log 2>&1
$N -k regex:pencil_update_kernel --launch-skip 1 -c 1 -o gpurun_out/k1_c3 python profiles/prof_run.py --config 3 --engine fast > gpurun_out/ncu4.log 2>&1
$N -k regex:fast_em2_kernel --launch-skip 2 -c 1 -o gpurun_out/k3img_c3 python profiles/prof_run.py --config 3 --engine fast > gpurun_out/ncu5.log 2>&1
$N -k regex:fast_em2_kernel --launch-skip 1 -c 1 -o gpurun_out/k3_c4 python profiles/prof_run.py --config 4 --engine fast > gpurun_out/ncu6.log 2>&1
$N -k regex:pencil_par_kernel --launch-skip 1 -c 1 -o gpurun_out/k1p_c4 python profiles/prof_run.py --config 4 --engine fast > gpurun_out/ncu7.log 2>&1
$N -k regex:fca_par_kernel --launch-skip 1 -c 1 -o gpurun_out/k4p_c2 python profiles/prof_run.py --config 2 --engine fca > gpurun_out/ncu8.log 2>&1
ls -la gpurun_out/*.ncu-rep
