"""bench.py's workloads against BASELINE.json (host-only checks)."""
import json
import pathlib

import bench

ROOT = pathlib.Path(__file__).resolve().parent.parent


def test_configs_follow_baseline():
    base = json.loads((ROOT / "BASELINE.json").read_text())["configs"]
    # (mesh, levels) quoted in each BASELINE config
    want = {"c1": (512, 7), "c2": (2048, 9), "c4": (8192, 11)}
    for name, (n, levels) in want.items():
        nx, ny, nc, recipe, seed, _ = bench.CONFIGS[name]
        assert (nx, ny, nc + 1) == (n, n, levels)
        text = base[int(name[1])]
        assert f"{n}×{n}" in text and f"{levels} levels" in text
    assert bench.CONFIGS["c2"][3] == "checker" and bench.CONFIGS["c4"][3:5] == ("iid", 1)
    assert bench.CONFIGS["c1"][3:5] == ("iid", 0)
    # c4 is the largest single-GPU configuration the metric is quoted on
    assert max(c[0] * c[1] for c in bench.CONFIGS.values()) == 8192 * 8192


def test_weak_scaling_mesh_grows_with_the_ranks():
    for ws in (1, 2, 4, 8):
        nx, ny, nc, *_ = bench.config_of("weak", ws)
        assert (nx, ny, nc) == (1024 * ws, 8192, 10)
        assert nx % (1 << nc) == 0 and ny % (1 << nc) == 0
    assert bench.config_of("c4", 8)[:2] == (8192, 8192)  # strong scaling: fixed mesh


def test_reference_arm_uses_every_core():
    assert bench.host_cores() >= 1


def test_gpus_flag_launches_one_rank_per_gpu():
    """bench.py --gpus N outside torchrun starts N ranks itself (rank 0 prints
    the line). On a GPU-less host both ranks get up to device init."""
    import subprocess
    import sys

    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("host has a GPU: the bench itself covers the launch")
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c0", "--steps", "1",
                        "--warmup", "3", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600)
    err = p.stderr
    assert "launching 2 ranks" in err
    assert "rank 0/2" in err and "rank 1/2" in err


def test_multi_rank_watchdog_ends_a_stuck_rank():
    """A rank with no result after TMG_BENCH_WATCHDOG_S exits 124 with a message
    (bench.arm_watchdog, armed for every rank of an N > 1 run)."""
    import os
    import subprocess
    import sys

    code = ("import sys, time; sys.path.insert(0, %r); import bench; bench.arm_watchdog(); time.sleep(30)"
            % str(ROOT))
    env = dict(os.environ, TMG_BENCH_WATCHDOG_S="0.5", RANK="1")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=60, env=env)
    assert p.returncode == 124
    assert "rank 1: no result after" in p.stderr
