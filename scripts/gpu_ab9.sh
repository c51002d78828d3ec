mkdir -p gpurun_out
for c in 0 1; do echo "== config $c"; bash scripts/cmp_variants.sh --config $c; done
