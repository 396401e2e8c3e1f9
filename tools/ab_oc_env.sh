# A/B of the OC exchange over environment settings (under gpurun):
#   bash tools/ab_oc_env.sh "VAR=V VAR=V ..." [rounds]
for r in $(seq ${2:-2}); do
  for kv in $1; do
    echo -n "$kv: "
    env $kv python tools/bench_oc.py --reps 3 2>gpurun_out/oc_err.txt | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['device_ms'], d['bisection_steps'], round(d['roofline']['frac'],3))"
  done
done
