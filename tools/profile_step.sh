# Step timing on the GPU box plus the launch list of one c4 PCG stretch
# (run under gpurun from the repo root; results in gpurun_out/):
#   /usr/local/graft/bin/gpurun -- bash tools/profile_step.sh
#   python tools/launches.py gpurun_out/launches_c4h.csv 12
python tools/step.py --config c4 --solves 2 && python tools/step.py --config c4 --solves 1 > gpurun_out/plain.log 2>&1 && TMG_NO_COND_NODES=1 ncu --metrics gpu__time_duration.sum --clock-control none -s 130 -c 100 --csv --log-file gpurun_out/launches_c4h.csv python tools/step.py --config c4 --solves 1 > gpurun_out/ncu1.log 2>&1; echo ncu=$?
