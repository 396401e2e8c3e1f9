# Same-box A/B of two builds (TMG_LIB_PATH), alternating, plus bitwise hashes:
#   bash tools/ab_two.sh libA.so libB.so "c4 c1 c3"
A=$1; B=$2; cfgs=${3:-c4}
for c in $cfgs; do
  for lib in $A $B; do echo -n "$c $lib hash: "; TMG_LIB_PATH=$PWD/$lib python tools/hash_solve.py --config $c 2>&1 | tail -1; done
  for i in 1 2 3; do for lib in $A $B; do
    echo -n "$c $lib: "; TMG_LIB_PATH=$PWD/$lib python tools/step.py --config $c --solves 3 2>&1 | tail -1 | sed 's/.*pcg=/pcg=/'
  done; done
done
