# A/B of the OC exchange over builds and CTAs per SM (under gpurun):
#   bash tools/ab_oc.sh "LIB:CTAS LIB:CTAS ..." [rounds]
for r in $(seq ${2:-2}); do
  for lc in $1; do
    lib=${lc%%:*}; c=${lc##*:}
    echo -n "$lib ctas=$c: "
    TMG_OC_CTAS=$c TMG_LIB_PATH=$PWD/$lib python tools/bench_oc.py --reps 3 2>gpurun_out/oc_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['device_ms'], round(d['roofline']['frac'],3))"
  done
done
