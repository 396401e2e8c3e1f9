# strip-width model's nominal resident CTAs per SM (TMG_STRIP_SLOTS), alternating
for c in c3 c1 c2 c4; do for i in 1 2; do for s in 3 4; do
  echo -n "$c slots=$s: "; TMG_STRIP_SLOTS=$s python tools/step.py --config $c --solves 3 2>&1 | tail -1 | sed 's/.*pcg=/pcg=/'
done; done; done
