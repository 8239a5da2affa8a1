"""tcgen05 gradient (fp32 mode) against a float64 numpy reference."""
import numpy as np
import pytest

import paper_2111_05366_b200 as gb
from paper_2111_05366_b200 import graphs

pytestmark = pytest.mark.gpu


def _ref(A, B, P):
    return A @ P @ B.T + A.T @ P @ B


@pytest.mark.parametrize("n", [17, 64, 130, 300, 1000])
@pytest.mark.parametrize("kind", ["directed01", "sym01", "weighted"])
def test_tc_gradient_matches_fp64(n, kind):
    rng = np.random.default_rng(n)
    if kind == "directed01":
        A = (rng.random((n, n)) < 0.3).astype(float)
        B = (rng.random((n, n)) < 0.3).astype(float)
    elif kind == "sym01":
        A = np.triu((rng.random((n, n)) < 0.3).astype(float), 1); A = A + A.T
        B = np.triu((rng.random((n, n)) < 0.3).astype(float), 1); B = B + B.T
    else:
        A = rng.lognormal(0, 1, (n, n)) * (rng.random((n, n)) < 0.3)
        B = rng.lognormal(0, 1, (n, n)) * (rng.random((n, n)) < 0.3)
    P = gb.random_doubly_stochastic(n, rng)
    G32 = gb.gradient(A, B, P, precision="fp32")
    G = _ref(A, B, P)
    err = np.abs(G32 - G).max() / np.abs(G).max()
    assert err < 2e-6, err


def test_tc_gradient_config2_scale():
    A, Bs, _ = graphs.config_pair(2, 0, n=1000)
    P = np.full((1000, 1000), 1e-3)
    P[np.arange(1000), np.arange(1000)] += 0.5
    G32 = gb.gradient(A, Bs, P, precision="fp32")
    G = _ref(A, Bs, P)
    assert np.abs(G32 - G).max() / np.abs(G).max() < 2e-6
