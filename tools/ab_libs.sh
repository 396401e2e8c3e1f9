# A/B timing of several builds of libtmg_gpu.so on several configs, alternating:
#   bash tools/ab_libs.sh "libA.so libB.so ..." "c4 c2" [rounds]
for i in $(seq ${3:-2}); do
  for cfg in $2; do
    for lib in $1; do
      echo -n "$lib $cfg: "; TMG_LIB_PATH=$PWD/$lib python tools/step.py --config $cfg --solves 3 2>&1 | tail -1
    done
  done
done
