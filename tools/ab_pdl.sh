# PDL of the bottom kernels and small tiles: hashes (bitwise) and per-iteration times
for c in c0 c1 c3 c2; do
  for env in "TMG_NO_PDL=0" "TMG_NO_PDL=1" "TMG_NO_PDL=1 TMG_STILE_TC2_NODES=0 TMG_STILE_TC4_NODES=0" "TMG_NO_PDL=0"; do
    echo "== $c $env"
    env $env python tools/step.py --config $c --solves 3 | tail -1 | sed 's/.*pcg=/pcg=/'
    env $env python tools/hash_solve.py --config $c | tail -1
  done
done
