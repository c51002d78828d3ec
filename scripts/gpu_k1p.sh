for c in 0 1; do
  for m in default p; do
    if [ $m = p ]; then export FFCA_K1=p; else unset FFCA_K1; fi
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu --no-pageable > gpurun_out/k1_$c_$m.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/k1_$c_$m.json').read().strip().splitlines()[-1]); print('config $c K1=$m', round(d['value']/1e9,2), 'G', round(d['ms_per_step'],4), 'ms', 'pass', d['roofline']['kernel_ms_avg'], 'iter', d['roofline']['iteration_ms_avg'], 'fca', round(d['fca']['value']/1e9,2))"
  done
done
