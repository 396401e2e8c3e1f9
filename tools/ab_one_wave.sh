# single-wave strip rule (TMG_STRIP_ONE_WAVE): per-iteration times, alternating
for c in c3 c1 c2; do for i in 1 2; do for v in 0 1; do
  echo -n "$c one_wave=$v: "; TMG_STRIP_ONE_WAVE=$v python tools/step.py --config $c --solves 3 2>&1 | tail -1 | sed 's/.*pcg=/pcg=/'
done; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slabs.py tests/test_gpu_optimize.py -q -x > gpurun_out/t_ow.log 2>&1; tail -1 gpurun_out/t_ow.log
python tools/bench_optimize.py --configs c3 > gpurun_out/opt_c3.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/opt_c3.json').read().splitlines()[-1]); print('c3 optimizer', d['value'], d['seconds'])"
