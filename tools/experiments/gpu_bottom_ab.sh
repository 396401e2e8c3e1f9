# (archived experiment, see tools/experiments/tmg_bottom_cluster.cuh)
# A/B of the cluster bottom kernel's size limit (TMG_BOTTOM_MAX_NODES) on the
# small-mesh configs, plus its bitwise tests
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster_bottom" > gpurun_out/t_bot.log 2>&1; echo test=$?
for c in c0 c1 c3; do for lim in 0 1089 4225 16641; do echo "== $c lim=$lim"; TMG_BOTTOM_MAX_NODES=$lim python tools/step.py --config $c --solves 4 | tail -1; done; done > gpurun_out/step_bot.log 2>&1
tail -3 gpurun_out/t_bot.log
