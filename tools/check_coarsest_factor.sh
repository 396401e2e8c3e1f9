# coarsest banded Cholesky: bitwise tests against the dense kernel, solve
# hashes and the factor's launch times (ncu)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "banded or errors_mirror or singular" 2>&1 | tail -1
for c in c0 c1 c3 c4; do python tools/hash_solve.py --config $c | tail -1; done
python tools/step.py --config c1 --solves 1 > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cholesky|k_lower|k_gram" --csv python tools/step.py --config c1 --solves 1 2>/dev/null | grep -E "k_cholesky|k_lower|k_gram" | awk -F'","' '{print $5, $NF}'
