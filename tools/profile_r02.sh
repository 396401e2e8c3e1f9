# The round's measurement set (run under gpurun from the repo root): the
# default bench.py line, the reference arm, the ncu launch list of a short
# bench run (after the same command exited 0 without ncu) and an
# `ncu --set full` capture of the c4 fine and coarse passes.
#   python tools/ncu_summary.py gpurun_out/full_r02.ncu-rep profiles/r02/ncu.csv profiles/ncu_traffic.json
set -x
# ncu cannot profile kernels inside graphs that contain conditional nodes, so
# the ncu runs use the plain iteration graphs (identical kernels; only the
# device-side skip of the converging iteration's speculative tail is off)
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench=$?
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && TMG_NO_COND_NODES=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo ncu1=$?
python tools/step.py --config c4 --solves 1 > gpurun_out/plain.log 2>&1 && TMG_NO_COND_NODES=1 ncu --set full --clock-control none --import-source on -k regex:"k_smarch" -s 12 -c 12 -o gpurun_out/full_r02 python tools/step.py --config c4 --solves 1 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?; TMG_NO_COND_NODES=1 ncu --set full --clock-control none --import-source on -k regex:"k_march" -s 5 -c 5 -o gpurun_out/full_r02f python tools/step.py --config c4 --solves 1 > gpurun_out/ncu_full_f.log 2>&1; echo ncu3=$?
