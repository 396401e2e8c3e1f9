# per-PCG-iteration cost of the x-slab machinery on one B200 (LocalComm: N
# slabs on concurrent per-slab streams, halo copies and the partial-array
# reductions), c4 and c2, alternating
for c in c4 c2; do for i in 1 2; do for n in 1 2 4 8; do
  echo -n "$c slabs=$n: "; python tools/step.py --config $c --solves 2 --slabs $n 2>&1 | tail -1 | sed 's/.*pcg=/pcg=/'
done; done; done
