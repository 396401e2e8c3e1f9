# A/B timing of two builds of libtmg_gpu.so in one GPU session (alternating):
#   bash tools/ab_step.sh libA.so libB.so [config]
cfg=${3:-c4}
for i in 1 2 3; do
  for lib in "$1" "$2"; do
    echo -n "$lib: "; TMG_LIB_PATH=$PWD/$lib python tools/step.py --config $cfg --solves 2 2>&1 | tail -1
  done
done
