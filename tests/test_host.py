"""CPU tests of the host-side mirror of the reference interface."""
import numpy as np
import pytest

import paper_2111_05366_b200 as gb
from paper_2111_05366_b200 import graphs


def test_option_validation_matches_reference():
    # matcher.py:52-66, sinkhorn.py:34-40
    with pytest.raises(ValueError):
        gb.MatchOptions(step_solver="hungarian")
    with pytest.raises(ValueError):
        gb.MatchOptions(max_iters=0)
    with pytest.raises(ValueError):
        gb.MatchOptions(fw_tol=0.0)
    with pytest.raises(ValueError):
        gb.MatchOptions(init="identity")
    with pytest.raises(ValueError):
        gb.MatchOptions(precision="fp16")
    for kw in (dict(lam=0), dict(tol=-1), dict(max_sweeps=0)):
        with pytest.raises(ValueError):
            gb.SinkhornParams(**kw)
    assert gb.MatchOptions() == gb.MatchOptions()
    assert gb.MatchOptions().step_solver == "exact_lap"  # reference default is FAQ


def test_seedset_validation():
    with pytest.raises(ValueError, match="duplicate"):
        gb.SeedSet(np.array([[0, 1], [0, 2]]))
    assert gb.SeedSet(np.empty((0, 2), dtype=int)).count == 0


def test_permutation_helpers():
    rng = np.random.default_rng(0)
    p = rng.permutation(9)
    inv = gb.invert_permutation(p)
    assert np.array_equal(p[inv], np.arange(9))
    B = rng.random((9, 9))
    Bp = gb.permute_matrix(B, p)
    assert np.allclose(Bp[np.ix_(p, p)], B)
    with pytest.raises(ValueError):
        gb.as_permutation([0, 0, 1])
    with pytest.raises(ValueError, match="finite"):
        gb.as_square_matrix([[1.0, np.inf], [0.0, 1.0]])
    with pytest.raises(ValueError, match="square"):
        gb.as_square_matrix(np.zeros((2, 3)))


def test_generators_are_seeded_and_well_formed():
    A, Bs, truth = graphs.config_pair(2, 0, n=200)
    assert np.array_equal(A, graphs.config_pair(2, 0, n=200)[0])
    assert not np.array_equal(A, A.T)  # directed
    assert (np.diag(A) == 0).all() and set(np.unique(A)) <= {0.0, 1.0}
    B = Bs[np.ix_(truth, truth)]
    agree = (A == B).mean()
    assert agree > 0.9
    A, Bs, truth = graphs.config_pair(4, 0, n=150)
    B = Bs[np.ix_(truth, truth)]
    assert (A > 0).sum() == pytest.approx((B > 0).sum(), rel=0.02)
    A, Bs, truth = graphs.config_pair(3, 0, n=300)
    assert np.array_equal(A, A.T)


def test_sparse_generator_symmetric_hollow():
    A, B, perm = graphs.sparse_er_pair_csr(600, 0.05, 0.9, config=5, replicate=0, block_rows=128)
    Ad = A.to_dense()
    Bd = B.to_dense()
    assert np.array_equal(Ad, Ad.T) and np.array_equal(Bd, Bd.T)
    assert np.trace(Ad) == 0
    # planted: B relabelled by perm agrees with A on most slots
    assert (Ad == Bd[np.ix_(perm, perm)]).mean() > 0.99


def test_product_path_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    A = np.zeros((4, 4))
    with pytest.raises(RuntimeError):
        gb.frank_wolfe_match(A, A, gb.MatchOptions(step_solver="lot"))


def test_as_csr_validation_and_canonical_form():
    import scipy.sparse as sp

    from paper_2111_05366_b200 import engine, graphs
    M = sp.coo_matrix((np.array([1.0, 2.0, 3.0]), (np.array([0, 0, 1]), np.array([2, 2, 0]))), shape=(3, 3))
    C = engine.as_csr(M)
    assert C.has_sorted_indices and C.nnz == 2 and C[0, 2] == 3.0  # duplicates summed
    with pytest.raises(ValueError):
        engine.as_csr(sp.csr_matrix(np.ones((2, 3))))
    with pytest.raises(ValueError):
        engine.as_csr(sp.csr_matrix(np.array([[0.0, np.inf], [1.0, 0.0]])))
    A, B, truth = graphs.config_pair(5, 0, n=300)
    assert engine.is_sparse(A) and not engine.is_sparse(A.to_dense())
    np.testing.assert_array_equal(engine.as_csr(A).toarray(), A.to_dense())
    ip, ix, v = engine._csr_arrays(engine.as_csr(A))
    assert v is None and ip.dtype == np.int64 and ix.dtype == np.int32
