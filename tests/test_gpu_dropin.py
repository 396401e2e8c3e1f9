"""C++ drop-in check: the reference optimizer's designs solved, and their OC
pair sweep applied, by the reference and by include/topmg_gpu.hpp
(tests/cpp/dropin_check.cpp)."""
import pathlib
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = pathlib.Path(__file__).resolve().parent / "cpp" / "dropin_check"


@pytest.mark.skipif(not BIN.exists(), reason="dropin_check is built where /root/reference exists")
def test_cpp_dropin_matches_reference_on_optimizer_designs():
    p = subprocess.run([str(BIN), "64", "6"], capture_output=True, text=True, timeout=600)
    lines = [l.split() for l in p.stdout.strip().splitlines()]
    assert len(lines) == 7, p.stdout + p.stderr
    # the same designs served again as one pipelined stream (PcgmgGpu::solve_many)
    assert lines[-1] == ["many", "6", "0"], p.stdout
    for k, it_ref, it_gpu, eu, ec, es, ef, eoc in lines[:-1]:
        assert abs(int(it_ref) - int(it_gpu)) <= 2
        assert float(eu) <= 1e-8 and float(ec) <= 1e-9
        assert float(es) <= 1e-8 and float(ef) <= 1e-8
        # the OC pair sweep (mto.cpp:312-323) through topmg_gpu.hpp
        assert float(eoc) <= 1e-12
    assert p.returncode == 0, p.stdout + p.stderr
