# A/B timing of one build under two values of an environment switch, in one
# GPU session (alternating runs of tools/step.py):
#   bash tools/ab_env.sh VAR valA valB [config] [rounds]
var=$1; cfg=${4:-c4}; n=${5:-3}
for i in $(seq $n); do
  for v in "$2" "$3"; do
    echo -n "$var=$v: "; env $var=$v python tools/step.py --config $cfg --solves 2 2>&1 | tail -1
  done
done
