"""Output writers of the Python mirror, byte for byte against the reference's
own writers (report.cpp:34-97, 153-168), run through
oracle/_ref. Pure host code: no GPU needed."""
import numpy as np
import pytest

import paper_2301_07457_b200 as P
from oracle import pyoracle as po

needs_ref = pytest.mark.skipif(not po.available("ref"), reason="oracle/_ref not built")


def report(n=7, seed=0):
    rng = np.random.default_rng(seed)
    hist = [float(v) for v in rng.uniform(0, 200, n)]
    hist[2] = 1.0 / 3.0
    hist[3] = 1e-300
    return P.OptimReport(np.zeros((1, 1)), hist, [float(v) for v in rng.uniform(0, 1, n)],
                         [int(v) for v in rng.integers(1, 900, n)], [float(v) for v in rng.exponential(0.3, n)], n,
                         0, 1.0, False)


def density(nx, ny, nph, seed=0):
    rng = np.random.default_rng(seed)
    a = rng.uniform(0, 1, (nx * ny, nph))
    a /= a.sum(1, keepdims=True)
    a[0] = [0.5 / 255.0] + [0.0] * (nph - 2) + [1.0 - 0.5 / 255.0]  # exact rounding ties
    a[1] = [2.5 / 255.0] + [0.0] * (nph - 2) + [1.0 - 2.5 / 255.0]
    return a


@needs_ref
def test_history_and_residual_csv_bytes(tmp_path):
    r = report()
    P.write_history_csv(r, tmp_path / "mine.csv")
    po.ref_write_history_csv(r, tmp_path / "ref.csv")
    assert (tmp_path / "mine.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
    hist = [1.0, 0.5, 1.0 / 3.0, 2.2250738585072014e-308, 0.0]
    P.write_residual_csv(P.SolveReport(np.zeros(1), 4, hist[-1], True, 0.0, hist), tmp_path / "r_mine.csv")
    po.ref_write_residual_csv(hist, tmp_path / "r_ref.csv")
    assert (tmp_path / "r_mine.csv").read_bytes() == (tmp_path / "r_ref.csv").read_bytes()


@needs_ref
@pytest.mark.parametrize("nx,ny,nph", [(16, 9, 4), (5, 12, 2), (8, 8, 6)])
def test_density_images_bytes(tmp_path, nx, ny, nph):
    a = density(nx, ny, nph)
    (tmp_path / "ref").mkdir()
    po.ref_write_density_images(nx, ny, a, tmp_path / "ref")
    rep = P.OptimReport(a, [], [], [], [], 0, 0, 0.0, False)
    P.emit_outputs(rep, P.GridLevel(nx, ny), tmp_path / "mine", images=True, csv=False)
    for i in range(nph):
        assert (tmp_path / "mine" / f"phase_{i + 1}.pgm").read_bytes() == \
            (tmp_path / "ref" / f"phase_{i + 1}.pgm").read_bytes()
    assert (tmp_path / "mine" / "composite.ppm").read_bytes() == (tmp_path / "ref" / "composite.ppm").read_bytes()
