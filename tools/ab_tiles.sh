# Tile-size A/B on the small-mesh configs: per-iteration times and solution
# hashes for the 1-/2-/4-/8-node tiles (TMG_STILE_TC{1,2,4}_NODES)
for c in c0 c1 c3; do
  for v in "0 0 0" "0 1089 16641" "289 1089 16641" "1089 4225 16641" "0 4225 16641" "0 0 0"; do
    set -- $v
    echo "== $c tc1<=$1 tc2<=$2 tc4<=$3"
    TMG_STILE_TC1_NODES=$1 TMG_STILE_TC2_NODES=$2 TMG_STILE_TC4_NODES=$3 python tools/step.py --config $c --solves 4 | tail -1 | sed 's/.*pcg=/pcg=/'
    TMG_STILE_TC1_NODES=$1 TMG_STILE_TC2_NODES=$2 TMG_STILE_TC4_NODES=$3 python tools/hash_solve.py --config $c | tail -1
  done
done
