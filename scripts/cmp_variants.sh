# A/B the shipped library against variant builds (paper_1805_06572_b200/lib/var_*.so)
# on the bench workload: value, update-pass ms, image-pass ms, SM clock.
# usage: bash scripts/cmp_variants.sh [bench args...]
mkdir -p gpurun_out
for v in paper_1805_06572_b200/lib/libfastfca_b200.so paper_1805_06572_b200/lib/var_*.so; do
  [ -f "$v" ] || continue
  FFCA_LIBRARY=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-other --no-pageable "$@" > gpurun_out/var.json 2> gpurun_out/var.err || tail -3 gpurun_out/var.err
  python - "$v" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/var.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1].split("/")[-1], round(d["value"] / 1e9, 3), "G", round(d["ms_per_step"], 3), "ms/run",
      "pass", r["kernel_ms_avg"], "frac", r["frac"], "img", r["last_pass_with_images_ms"],
      "mhz", d["clocks"]["sm_mhz"], flush=True)
PY
done
