# A/B timing of two builds of libtmg_gpu.so on several configs, alternating:
#   bash tools/ab_multi.sh libA.so libB.so "c4 c3 c1" [rounds]
for i in $(seq ${4:-2}); do
  for cfg in $3; do
    for lib in "$1" "$2"; do
      echo -n "$lib $cfg: "; TMG_LIB_PATH=$PWD/$lib python tools/step.py --config $cfg --solves 3 2>&1 | tail -1
    done
  done
done
