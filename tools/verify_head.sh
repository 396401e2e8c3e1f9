o=gpurun_out/v1; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q -x > $o/gputest.log 2>&1; echo gputest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke=$?
python bench.py --steps 20 --warmup 5 > $o/bench_c4.json 2> $o/bench_c4.err; echo bench=$?
python bench.py --config c1 --steps 400 --warmup 20 --no-cpu-baseline > $o/bench_c1.json 2>&1; echo c1=$?
python bench.py --config c3 --steps 200 --warmup 10 --no-cpu-baseline > $o/bench_c3_mesh.json 2>&1; echo c3=$?
tail -3 $o/gputest.log; cat $o/bench_c4.json | head -c 600
