"""CSR adjacency path (goat_fw_core_csr / goat_gradient_csr): the gradient by
SpMM and the whole GOAT iteration on sparse inputs, against the CPU oracle and
the dense device path on the same seeded inputs."""
import ctypes
import os

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2111_05366_b200 as gb
from oracle import goat_oracle as O
from paper_2111_05366_b200 import _lib, engine, graphs
from paper_2111_05366_b200.records import MatchOptions, SeedSet

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "c5_n4000.npz")


def _gradient_csr(A, B, P, precision):
    A = engine.as_csr(A)
    B = engine.as_csr(B)
    aa, ba = engine._csr_arrays(A), engine._csr_arrays(B)
    ca, cb = _lib.csr_struct(*aa), _lib.csr_struct(*ba)
    n = A.shape[0]
    P = np.ascontiguousarray(P, dtype=np.float64)
    G = np.empty((n, n))
    h = _lib.handle(0, precision)
    with h.lock:
        _lib.check(_lib.load().goat_gradient_csr(h.ptr, n, ctypes.byref(ca), ctypes.byref(cb), _lib.dptr(P), n,
                                                 _lib.dptr(G), n))
    return G


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("kind", ["sym01", "directed01", "weighted"])
@pytest.mark.parametrize("n", [37, 300, 1000])
def test_gradient_csr_matches_oracle(precision, kind, n):
    rng = np.random.default_rng(n)
    A = (rng.random((n, n)) < 0.05).astype(float)
    B = (rng.random((n, n)) < 0.05).astype(float)
    np.fill_diagonal(A, 0)
    if kind == "sym01":
        A = np.triu(A, 1); A = A + A.T
        B = np.triu(B, 1); B = B + B.T
    elif kind == "weighted":
        A = A * rng.lognormal(0, 1, (n, n))
        B = B * rng.lognormal(0, 1, (n, n))
    P = rng.random((n, n))
    P /= P.sum(1, keepdims=True)
    G = _gradient_csr(sp.csr_matrix(A), sp.csr_matrix(B), P, precision)
    ref = O.qap_gradient(A, B, P)
    tol = 1e-12 if precision == "fp64" else 2e-6
    assert np.abs(G - ref).max() <= tol * np.abs(ref).max()


def test_gradient_csr_empty_rows_and_graph():
    n = 50
    A = np.zeros((n, n)); A[3, 7] = 1; A[7, 3] = 1
    B = np.zeros((n, n))
    P = np.full((n, n), 1.0 / n)
    G = _gradient_csr(sp.csr_matrix(A), sp.csr_matrix(B), P, "fp64")
    assert np.array_equal(G, np.zeros((n, n)))
    G = _gradient_csr(sp.csr_matrix(A), sp.csr_matrix(A), P, "fp64")
    np.testing.assert_allclose(G, O.qap_gradient(A, A, P), rtol=0, atol=1e-15)


def test_csr_rejects_bad_structure():
    n = 4
    indptr = np.array([0, 2, 2, 2, 2], dtype=np.int64)
    bad = np.array([3, 1], dtype=np.int32)  # not increasing
    ok = np.array([1, 3], dtype=np.int32)
    h = _lib.handle(0, "fp64")
    P = np.full((n, n), 0.25)
    G = np.empty((n, n))
    cbad, cok = _lib.csr_struct(indptr, bad), _lib.csr_struct(indptr, ok)
    with pytest.raises(ValueError):
        _lib.check(_lib.load().goat_gradient_csr(h.ptr, n, ctypes.byref(cbad), ctypes.byref(cok), _lib.dptr(P), n,
                                                 _lib.dptr(G), n))
    big = np.array([1, 4], dtype=np.int32)  # out of range
    cbig = _lib.csr_struct(indptr, big)
    with pytest.raises(ValueError):
        _lib.check(_lib.load().goat_gradient_csr(h.ptr, n, ctypes.byref(cok), ctypes.byref(cbig), _lib.dptr(P), n,
                                                 _lib.dptr(G), n))


@pytest.mark.parametrize("replicate", [0, 1])
def test_c1_sparse_equals_oracle(replicate):
    """Config 1 (fp64) through frank_wolfe_match on scipy CSR inputs: the
    oracle's permutation, objective, iterations and history."""
    A, Bs, truth = graphs.config_pair(1, replicate)
    opts = MatchOptions(step_solver="lot", fw_tol=0.03, precision="fp64")
    res = gb.frank_wolfe_match(sp.csr_matrix(A), sp.csr_matrix(Bs), opts)
    align, obj, iters, hist, conv = O.run_seeded(A, Bs, np.empty((0, 2)), fw_tol=0.03)
    np.testing.assert_array_equal(res.alignment, align)
    assert res.objective == obj and res.iterations == iters and res.converged == conv
    np.testing.assert_allclose([h[1] for h in res.iterate_history], [h[1] for h in hist], rtol=1e-9)


def test_weighted_sparse_seeded_equals_dense_path():
    """c4-like weighted directed pair with seeds and shuffling: CSR path == dense path."""
    A, Bs, truth = graphs.config_pair(4, 0, n=300)
    seeds = SeedSet(np.stack([np.arange(5), truth[:5]], axis=1))
    opts = MatchOptions(step_solver="lot", precision="fp64", shuffle_input=True, max_iters=8)
    dense = gb.seeded_match(A, Bs, seeds, opts)
    sparse = gb.seeded_match(sp.csr_matrix(A), sp.csr_matrix(Bs), seeds, opts)
    np.testing.assert_array_equal(sparse.alignment, dense.alignment)
    assert sparse.objective == pytest.approx(dense.objective, rel=1e-12)
    assert sparse.iterations == dense.iterations


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_c5_n4000_csr_matches_oracle(precision):
    """Config 5 scaled to n = 4000, CSR end to end (SpMM gradient, CSR degrees and
    objective): the oracle's permutation, objective and step sizes."""
    g = np.load(GOLD)
    A, Bs, truth = graphs.config_pair(5, 0, n=4000)
    opts = MatchOptions(step_solver="lot", max_iters=4, precision=precision)
    a, hist, iters, conv, diag = engine.fw_core_csr(A, Bs, None, None, opts)
    assert iters == int(g["iterations"]) and conv == bool(g["converged"])
    np.testing.assert_array_equal(a, g["assignment"])
    assert diag["objective"] == float(g["objective"])
    np.testing.assert_allclose([h[2] for h in hist[1:]], g["alpha"], atol=1e-6)
    if precision == "fp64":
        assert diag["lot_sweeps"] == g["sweeps"].tolist()
