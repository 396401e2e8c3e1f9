# DSMEM cluster bottom (tmg_vbottom.cuh): bitwise hashes against the per-level
# launches (TMG_VBOTTOM=0) and per-iteration times, alternating
for c in c0 c1 c3; do
  for v in 0 1; do echo -n "$c VBOTTOM=$v hash: "; TMG_VBOTTOM=$v timeout 120 python tools/hash_solve.py --config $c 2>&1 | tail -1; done
done
for c in c0 c1 c3 c4; do for i in 1 2; do for v in 0 1; do
  echo -n "$c VBOTTOM=$v: "; TMG_VBOTTOM=$v timeout 120 python tools/step.py --config $c --solves 3 2>&1 | tail -1 | sed 's/.*pcg=/pcg=/'
done; done; done
