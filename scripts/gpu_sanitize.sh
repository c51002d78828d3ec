# compute-sanitizer memcheck / racecheck / synccheck over the EM kernels
# (small configs, both engines, I = 2 / 4 / 8, c128 + c64, images + likelihood)
mkdir -p gpurun_out/sanitizer
run() {  # tool name args...
  local tool=$1 name=$2; shift 2
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python profiles/prof_run.py "$@" > gpurun_out/sanitizer/${tool}_${name}.log 2>&1
  echo "$tool $name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitizer/${tool}_${name}.log | tail -1)"
}
for tool in memcheck racecheck synccheck; do
  run $tool c0_fast --config 0 --engine fast --iters 2 --likelihood
  run $tool c0_fca --config 0 --engine fca --iters 2 --likelihood
  run $tool c3_fast --config 3 --engine fast --iters 2 --mixtures 2
  run $tool c3_fca --config 3 --engine fca --iters 2 --mixtures 2
  run $tool c3_fast_c64 --config 3 --engine fast --iters 2 --mixtures 2 --dtype c64
  run $tool c2_fast --config 2 --engine fast --iters 2
  run $tool c2_fca --config 2 --engine fca --iters 2
done
