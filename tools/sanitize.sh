# compute-sanitizer over small device-resident solves (B200): memcheck,
# racecheck (shared memory hazards), synccheck (barrier misuse) and initcheck
# (reads of uninitialised global memory); c0 (64^2, 4 levels), c1 with two
# x-slabs on one device, and the optimizer's first outer iterations
o=gpurun_out/sanitize; mkdir -p $o
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool args...
  n=$1; tool=$2; shift 2
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 "$@" > $o/$n.$tool.log 2>&1
  echo "$n $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $o/$n.$tool.log | tail -1)"
}
for t in memcheck racecheck synccheck initcheck; do
  run c0 $t python tools/step.py --config c0 --solves 2
done
for t in memcheck racecheck; do
  run c1slab2 $t python tools/step.py --config c1 --slabs 2 --solves 1
done
run opt memcheck python tools/sanitize_opt.py
