"""BASELINE config 5 (sparse correlated ER, undirected) scaled to n = 4000 against
the recorded oracle run (tests/golden/make_c5_golden.py): the full device GOAT
iteration -- tcgen05 gradient, persistent Sinkhorn, line search, auction + exact
repair LAP -- must return the oracle's permutation, objective and step sizes."""
import os

import numpy as np
import pytest

from paper_2111_05366_b200 import engine, graphs
from paper_2111_05366_b200.records import MatchOptions

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "c5_n4000.npz")


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c5_n4000_matches_oracle(precision):
    g = np.load(GOLD)
    A, Bs, truth = graphs.config_pair(5, 0, n=4000)
    opts = MatchOptions(step_solver="lot", max_iters=4, precision=precision)
    a, hist, iters, conv, diag = engine.fw_core(A.to_dense(), Bs.to_dense(), None, None, opts)
    assert iters == int(g["iterations"]) and conv == bool(g["converged"])
    np.testing.assert_array_equal(a, g["assignment"])
    assert diag["objective"] == float(g["objective"])
    np.testing.assert_allclose([h[2] for h in hist[1:]], g["alpha"], atol=1e-6)
    if precision == "fp64":
        assert diag["lot_sweeps"] == g["sweeps"].tolist()
