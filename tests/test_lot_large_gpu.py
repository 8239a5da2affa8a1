"""LOT at orders wider than one CTA's registers: cluster-split rows (DSMEM row
combine).  Checked against the CPU oracle on the same G with a bounded sweep count."""
import numpy as np
import pytest

import paper_2111_05366_b200 as gb
from oracle import goat_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,precision", [(4501, "fp32"), (5000, "fp32"), (7000, "fp32"), (10000, "fp32"), (17000, "fp32"), (5000, "fp64")])
def test_lot_cluster_split_matches_oracle(n, precision):
    rng = np.random.default_rng(n)
    # structured costs (rank-2 degree products + noise), like a barycenter gradient
    d1 = rng.integers(50, 150, n).astype(float)
    d2 = rng.integers(50, 150, n).astype(float)
    M = np.outer(d1, d2) / n + rng.random((n, n))
    params = gb.SinkhornParams(max_sweeps=30)
    res = gb.lot(M, "maximize", params, precision=precision)
    Q, conv, sweeps, dev = O.lot(M, "maximize", 100.0, 30, 1e-8)
    assert res.sweeps == sweeps and res.converged == conv
    tol = 1e-3 if precision == "fp32" else 1e-5
    assert np.abs(res.matrix - Q).max() < tol
    assert res.deviation == pytest.approx(dev, rel=1e-2 if precision == "fp32" else 1e-6)


@pytest.mark.parametrize("n", [10000, 20000])
def test_fixed_shift_redo_path(n, monkeypatch):
    """Wide fp32 rows use the previous row LSE as the exponent shift; a sweep with a
    row outside the window is recomputed with the max shift.  Forcing every sweep
    through the redo (GOAT_SK_RES=3) must give exactly the max-shift run
    (GOAT_SK_RES=2), and the default run must agree with both to fp32 accuracy."""
    rng = np.random.default_rng(n)
    d1 = rng.integers(50, 150, n).astype(float)
    d2 = rng.integers(50, 150, n).astype(float)
    M = np.outer(d1, d2) / n + rng.random((n, n))
    params = gb.SinkhornParams(max_sweeps=12)
    out = {}
    for mode in ("2", "3", "1"):
        monkeypatch.setenv("GOAT_SK_RES", mode)
        out[mode] = gb.lot(M, "maximize", params, precision="fp32")
    assert np.array_equal(out["3"].matrix, out["2"].matrix)
    assert out["3"].sweeps == out["2"].sweeps and out["3"].deviation == out["2"].deviation
    assert np.abs(out["1"].matrix - out["2"].matrix).max() < 1e-5
    assert out["1"].sweeps == out["2"].sweeps


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 33, 127, 255, 257, 511, 1001, 1999])
@pytest.mark.parametrize("sense", ["maximize", "minimize"])
def test_lot_small_orders_tile_kernel(n, sense):
    """Orders served by the shared-memory tile kernel (2- and 4-CTA clusters, ragged
    last row group and slice), fp64: the oracle's sweep count, flag and iterate."""
    rng = np.random.default_rng(n + (sense == "minimize"))
    M = rng.random((n, n)) * rng.integers(1, 50)
    params = gb.SinkhornParams(max_sweeps=200)
    res = gb.lot(M, sense, params, precision="fp64")
    Q, conv, sweeps, dev = O.lot(M, sense, 100.0, 200, 1e-8)
    assert res.sweeps == sweeps and res.converged == conv
    assert np.abs(res.matrix - Q).max() < 1e-9
