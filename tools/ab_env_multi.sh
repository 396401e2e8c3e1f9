# A/B of an environment switch over several values and configs (alternating):
#   bash tools/ab_env_multi.sh VAR "v1 v2 ..." "cfg1 cfg2 ..." [rounds]
var=$1; vals=$2; cfgs=$3; n=${4:-2}
for cfg in $cfgs; do
  for i in $(seq $n); do
    for v in $vals; do
      echo -n "$var=$v: "; env $var=$v python tools/step.py --config $cfg --solves 3 2>&1 | tail -1
    done
  done
done
