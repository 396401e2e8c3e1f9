for s in 3 4 5 6; do echo -n "c3 slots=$s: "; TMG_STRIP_SLOTS=$s python tools/step.py --config c3 --solves 3 | tail -1 | sed 's/.*pcg=/pcg=/'; echo -n "c1 slots=$s: "; TMG_STRIP_SLOTS=$s python tools/step.py --config c1 --solves 3 | tail -1 | sed 's/.*pcg=/pcg=/'; done
python tools/bench_optimize.py > gpurun_out/bench_optimize.json 2> gpurun_out/bench_optimize.err
