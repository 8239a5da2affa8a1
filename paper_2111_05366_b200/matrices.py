"""Host-side validation and permutation helpers (reference core.py semantics).

These run on the host because they are O(n) bookkeeping or input
validation around the device path, not part of it: the validation semantics
of ``as_square_matrix`` (core.py:17-27) are the boundary's error contract,
and the permutation utilities are what ``_run_seeded`` uses to relabel inputs
(core.py:64-93, 152-163).  The QAP objective on a permutation (core.py:120-124)
is evaluated on the device.
"""

from __future__ import annotations

import numpy as np

from . import _lib

DS_TOL = 1e-8


def as_square_matrix(M, name: str = "matrix", check_finite: bool = True) -> np.ndarray:
    """core.py:17-27.  ``check_finite=False`` is for inputs whose finiteness the
    library checks itself while uploading them (goat_fw_core raises the same
    ValueError from the device conversion)."""
    M = np.asarray(M, dtype=float)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError(f"{name} must be square, got shape {M.shape}")
    if check_finite and not np.all(np.isfinite(M)):
        raise ValueError(f"{name} contains non-finite entries")
    return M


def as_permutation(p, name: str = "permutation") -> np.ndarray:
    p = np.asarray(p)
    if p.ndim != 1:
        raise ValueError(f"{name} must be a 1-D index vector, got shape {p.shape}")
    if p.size and not np.issubdtype(p.dtype, np.integer):
        if not np.array_equal(p, p.astype(np.intp)):
            raise ValueError(f"{name} has non-integer entries")
    p = p.astype(np.intp)
    if not np.array_equal(np.sort(p), np.arange(p.size)):
        raise ValueError(f"{name} is not a bijection of [0, {p.size})")
    return p


def as_doubly_stochastic(P, tol: float = DS_TOL, name: str = "matrix") -> np.ndarray:
    P = as_square_matrix(P, name)
    if P.size and P.min() < -tol:
        raise ValueError(f"{name} has negative entries (min {P.min():.3e})")
    rdev = np.abs(P.sum(axis=1) - 1.0).max(initial=0.0)
    cdev = np.abs(P.sum(axis=0) - 1.0).max(initial=0.0)
    if rdev > tol or cdev > tol:
        raise ValueError(f"{name} is not doubly stochastic at tol {tol:g} "
                         f"(row dev {rdev:.3e}, col dev {cdev:.3e})")
    return P


def permutation_matrix(p) -> np.ndarray:
    p = as_permutation(p)
    out = np.zeros((p.size, p.size))
    out[np.arange(p.size), p] = 1.0
    return out


def invert_permutation(p) -> np.ndarray:
    p = as_permutation(p)
    inv = np.empty_like(p)
    inv[p] = np.arange(p.size)
    return inv


def compose_permutations(p, q) -> np.ndarray:
    p = as_permutation(p)
    q = as_permutation(q)
    if p.size != q.size:
        raise ValueError(f"length mismatch: {p.size} vs {q.size}")
    return q[p]


def barycenter(n: int) -> np.ndarray:
    if n < 1:
        raise ValueError("order must be positive")
    return np.full((n, n), 1.0 / n)


def permute_matrix(B, p) -> np.ndarray:
    """out[p[i], p[j]] = B[i, j] (core.py:152-163)."""
    B = as_square_matrix(B, "B")
    p = as_permutation(p)
    if p.size != B.shape[0]:
        raise ValueError(f"order mismatch: {[B.shape[0], p.size]}")
    inv = invert_permutation(p)
    return B[np.ix_(inv, inv)]


def match_ratio(found, truth) -> float:
    found = as_permutation(found, "found")
    truth = as_permutation(truth, "truth")
    if found.size != truth.size:
        raise ValueError(f"length mismatch: {found.size} vs {truth.size}")
    return float(np.mean(found == truth))


def edge_disagreements(A, B, p) -> float:
    """||A - P B P^T||_F^2 = ||A||^2 + ||B||^2 - 2 qap(A, B, p) (core.py:130-140)."""
    A = as_square_matrix(A, "A")
    B = as_square_matrix(B, "B")
    p = as_permutation(p)
    if not (A.shape[0] == B.shape[0] == p.size):
        raise ValueError(f"order mismatch: {[A.shape[0], B.shape[0], p.size]}")
    return float(((A - B[np.ix_(p, p)]) ** 2).sum())


def qap_objective(A, B, P, *, device=0) -> float:
    """trace(A^T P B P^T) for a permutation vector or a dense matrix (core.py:111-127).

    Both forms run on the device: the permutation form as an fp64 gather-reduce
    (exact for integer graphs), the dense form as <M(P), P> with M(P) = A^T P B.
    """
    A = as_square_matrix(A, "A")
    B = as_square_matrix(B, "B")
    arr = np.asarray(P)
    if arr.ndim == 1:
        p = as_permutation(arr)
        if not (A.shape[0] == B.shape[0] == p.size):
            raise ValueError(f"order mismatch: {[A.shape[0], B.shape[0], p.size]}")
        h = _lib.handle(device, "fp64")
        out = np.zeros(1)
        A_ = _lib.f64(A)
        B_ = _lib.f64(B)
        p64 = np.ascontiguousarray(p, dtype=np.int64)
        with h.lock:
            _lib.check(_lib.load().goat_qap_objective_perm(
                h.ptr, p.size, _lib.dptr(A_), _lib.ld_of(A_), _lib.dptr(B_), _lib.ld_of(B_),
                p64.ctypes.data_as(_lib._c_i64_p), _lib.dptr(out)))
        return float(out[0])
    Pd = as_square_matrix(arr, "P")
    if not (A.shape[0] == B.shape[0] == Pd.shape[0]):
        raise ValueError(f"order mismatch: {[A.shape[0], B.shape[0], Pd.shape[0]]}")
    from .ops import gradient
    # <G(P), P> = 2 trace(A^T P B P^T)
    return float((gradient(A, B, Pd, device=device) * Pd).sum() / 2.0)
