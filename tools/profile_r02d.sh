# Round-2 end-state measurement set (after the large-coarsest path, the OC load schedule and the reduction tail):
# the GPU test suite and smoke(), bench lines of every solve config with
# clock samples (small configs with enough steps for the 100 ms nvidia-smi
# sampler), the reference arm with the driver's step counts, the optimizer
# bench, the ncu launch list of a short bench run, `ncu --set full` of one c4
# PCG iteration's fine and coarse passes, and warm-cache launch lists of c1
# and c3. ncu runs use TMG_NO_COND_NODES=1 (ncu cannot profile kernels inside
# graphs with conditional nodes; the kernels are identical).
set -x
o=gpurun_out/r02d; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/gputest.log 2>&1; echo gputest=$?
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke=$?
python bench.py --steps 20 --warmup 5 > $o/bench_c4.json 2> $o/bench_c4.err; echo bench=$?
python bench.py --impl reference --steps 20 --warmup 5 > $o/bench_ref.json 2> $o/bench_ref.err; echo ref=$?
python bench.py --config c1 --steps 400 --warmup 20 --no-cpu-baseline > $o/bench_c1.json 2>&1; echo c1=$?
python bench.py --config c3 --steps 200 --warmup 10 --no-cpu-baseline > $o/bench_c3_mesh.json 2>&1; echo c3=$?
python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline > $o/bench_c2.json 2>&1; echo c2=$?
python bench.py --config weak --steps 40 --warmup 5 --no-cpu-baseline > $o/bench_weak_n1.json 2>&1; echo weak=$?
python tools/bench_optimize.py > $o/bench_optimize.json 2> $o/bench_optimize.err; echo opt=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/bench_small.json 2>&1 && TMG_NO_COND_NODES=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/ncu_bench.log 2>&1; echo ncu1=$?
python tools/step.py --config c4 --solves 1 > $o/plain.log 2>&1 && TMG_NO_COND_NODES=1 ncu --set full --clock-control none --import-source on -k regex:"k_smarch2" -s 16 -c 16 -o $o/full_coarse python tools/step.py --config c4 --solves 1 > $o/ncu_full_c.log 2>&1; echo ncu2=$?
TMG_NO_COND_NODES=1 ncu --set full --clock-control none --import-source on -k regex:"k_march" -s 5 -c 5 -o $o/full_fine python tools/step.py --config c4 --solves 1 > $o/ncu_full_f.log 2>&1; echo ncu3=$?
python tools/step.py --config c1 --solves 1 > $o/plain_c1.log 2>&1 && TMG_NO_COND_NODES=1 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $o/launches_c1_warm.csv python tools/step.py --config c1 --solves 2 > $o/ncu_c1.log 2>&1; echo ncu4=$?
TMG_NO_COND_NODES=1 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $o/launches_c3_warm.csv python tools/step.py --config c3 --solves 2 > $o/ncu_c3.log 2>&1; echo ncu5=$?
python tools/bench_oc.py > $o/bench_oc.json 2> $o/bench_oc.err; echo oc=$?
python tools/bench_poisson.py > $o/bench_poisson.json 2> $o/bench_poisson.err; echo poisson=$?
bash tools/large_coarsest_check.sh > $o/large_coarsest.txt 2>&1; echo lc=$?
