# Same-box A/B of several builds (TMG_LIB_PATH), alternating, with hashes:
#   bash tools/ab_libs3.sh "c3 c1 c4" libA.so libB.so ...
cfgs=$1; shift
for c in $cfgs; do
  for lib in "$@"; do echo -n "$c $lib hash: "; TMG_LIB_PATH=$PWD/$lib python tools/hash_solve.py --config $c 2>&1 | tail -1; done
  for i in 1 2; do for lib in "$@"; do
    echo -n "$c $lib: "; TMG_LIB_PATH=$PWD/$lib python tools/step.py --config $c --solves 3 2>&1 | tail -1 | sed 's/.*pcg=/pcg=/'
  done; done
done
