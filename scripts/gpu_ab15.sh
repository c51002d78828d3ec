mkdir -p gpurun_out
for c in 3 1 0; do echo "== config $c"; bash scripts/cmp_variants.sh --config $c; done
