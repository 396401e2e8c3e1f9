for c in c4 c3 c2 c1; do for i in 1 2; do for lim in 66049 263169; do
  echo -n "$c lim=$lim: "; TMG_STILE_MAX_NODES=$lim python tools/step.py --config $c --solves 3 2>&1 | tail -1 | sed 's/.*pcg=/pcg=/'
done; done; done
