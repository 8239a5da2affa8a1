"""Exact LAP for n >= 256: eps-scaling auction front end + certified repair by
warm-started augmenting paths.  Must return scipy's (unique) optimum, including
on hub-dominated matrices like the final gradients of failed GOAT runs."""
import numpy as np
import pytest

import paper_2111_05366_b200 as gb
from oracle import goat_oracle as O

pytestmark = pytest.mark.gpu


def _hub(n, rng):
    # rank-1 degree products + a few hub columns + noise: most rows share argmaxes
    d1 = rng.gamma(2.0, 1.0, n)
    d2 = rng.gamma(2.0, 1.0, n)
    M = np.outer(d1, d2)
    M[:, rng.choice(n, 5, replace=False)] += 3.0 * d1[:, None]
    return M + 1e-3 * rng.random((n, n))


@pytest.mark.parametrize("n", [300, 1000, 2500])
@pytest.mark.parametrize("kind", ["uniform", "hub"])
@pytest.mark.parametrize("sense", ["maximize", "minimize"])
def test_auction_lap_matches_scipy(n, kind, sense):
    rng = np.random.default_rng(n + (kind == "hub"))
    M = rng.random((n, n)) if kind == "uniform" else _hub(n, rng)
    p, v = O.lap(M, sense)
    for precision in ("fp64", "fp32"):
        Mp = M if precision == "fp64" else M.astype(np.float32).astype(np.float64)
        pp, vp = (p, v) if precision == "fp64" else O.lap(Mp, sense)
        sol = gb.solve_lap(Mp, sense, precision=precision)
        assert sol.objective == vp  # exact optimum, always
        if not np.array_equal(sol.assignment, pp):
            # a different optimal permutation is only allowed on an exact tie
            # (seen on the fp32-rounded hub matrix): same objective, valid bijection
            gb.as_permutation(sol.assignment)
            assert Mp[np.arange(n), sol.assignment].sum() == Mp[np.arange(n), pp].sum()


@pytest.mark.parametrize("n", [700, 3000])
@pytest.mark.parametrize("kind", ["uniform", "hub"])
@pytest.mark.parametrize("sense", ["maximize", "minimize"])
def test_cluster_repair_matches_scipy(n, kind, sense, monkeypatch):
    """The cluster-split augmenting-path repair (used once the single-CTA state
    outgrows shared memory, n >~ 7000) forced at smaller n: scipy's optimum."""
    monkeypatch.setenv("GOAT_LAP_CLUSTER", "2")
    rng = np.random.default_rng(7 * n + (kind == "hub"))
    M = rng.random((n, n)) if kind == "uniform" else _hub(n, rng)
    p, v = O.lap(M, sense)
    sol = gb.solve_lap(M, sense, precision="fp64")
    assert sol.objective == v
    gb.as_permutation(sol.assignment)
    if not np.array_equal(sol.assignment, p):
        assert M[np.arange(n), sol.assignment].sum() == M[np.arange(n), p].sum()


@pytest.mark.parametrize("kind", ["uniform", "tied"])
def test_large_order_bidder_list_paths(kind):
    """n = 7500: beyond the single-CTA repair (cluster solver by default) and with more
    bidders than warps in the first rounds of a phase, so the auction's bidder-list
    splits (1, 2 and 4 rows per warp) and the level-wise cluster repair all run.
    `uniform` is checked against scipy.  `tied` is a rank-1 product of small integer
    degree vectors -- exact ties everywhere, the shape of FAQ's first gradient; scipy
    needs minutes on it, but its optimum is known in closed form (rearrangement
    inequality: sort both vectors)."""
    n = 7500
    rng = np.random.default_rng(75 + (kind == "tied"))
    if kind == "uniform":
        M = rng.random((n, n)).astype(np.float32).astype(np.float64)
        v = O.lap(M, "maximize")[1]
    else:
        d1 = rng.integers(1, 21, n).astype(np.float64)
        d2 = rng.integers(1, 21, n).astype(np.float64)
        M = np.outer(d1, d2)
        v = float(np.dot(np.sort(d1), np.sort(d2)))
    sol = gb.solve_lap(M, "maximize", precision="fp32")
    gb.as_permutation(sol.assignment)
    assert sol.objective == v


def test_order_12000_four_rows_per_warp_path_matches_scipy():
    """n = 12000: the first rounds of every auction phase have more than three bidders
    per warp, so the 4-rows-per-warp split with shared-memory price tiles runs (the
    only other order that reaches it in the suite is config 5, which has no scipy
    reference).  Both handle precisions on the same fp32-representable matrix."""
    n = 12000
    rng = np.random.default_rng(120)
    M = rng.random((n, n)).astype(np.float32).astype(np.float64)
    v = O.lap(M, "maximize")[1]
    for precision in ("fp32", "fp64"):
        sol = gb.solve_lap(M, "maximize", precision=precision)
        gb.as_permutation(sol.assignment)
        assert sol.objective == v, precision
