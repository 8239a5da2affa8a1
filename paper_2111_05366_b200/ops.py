"""Device implementations of the functions ``_fw_core`` calls.

Each public function keeps the reference's name, arguments, return type and
ValueError behaviour, and runs on the GPU through libgoat.so:

  gradient            matcher.py:100-107   -> goat_gradient
  exact_line_search   matcher.py:138-154   -> goat_line_search_coeffs + _optimal_alpha
  lot                 sinkhorn.py:103-130  -> goat_lot
  sinkhorn_knopp      sinkhorn.py:60-85    -> goat_sinkhorn_knopp
  solve_lap           lap.py:48-58         -> goat_lap

``precision`` selects the device arithmetic ("fp64" = the reference's float64,
the default; "fp32" = the fast mode).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .matrices import as_square_matrix, barycenter
from .records import SENSES, LapSolution, SinkhornParams, SinkhornResult

__all__ = ["gradient", "exact_line_search", "optimal_alpha", "lot", "sinkhorn_knopp",
           "solve_lap", "random_doubly_stochastic", "randomized_blend_init"]


def _h(device, precision):
    return _lib.handle(device, precision)


def _sense_code(sense):
    if sense not in SENSES:
        raise ValueError(f"sense must be one of {SENSES}, got {sense!r}")
    return _lib.GOAT_MAXIMIZE if sense == "maximize" else _lib.GOAT_MINIMIZE


def gradient(A, B, P, *, device=0, precision="fp64") -> np.ndarray:
    """A P B^T + A^T P B on the device."""
    A = as_square_matrix(A, "A")
    B = as_square_matrix(B, "B")
    P = as_square_matrix(P, "P")
    if not (A.shape == B.shape == P.shape):
        raise ValueError(f"order mismatch: {A.shape[0]}, {B.shape[0]}, {P.shape[0]}")
    n = A.shape[0]
    A_, B_, P_ = _lib.f64(A), _lib.f64(B), _lib.f64(P)
    G = np.empty((n, n))
    h = _h(device, precision)
    with h.lock:
        _lib.check(_lib.load().goat_gradient(h.ptr, n, _lib.dptr(A_), _lib.ld_of(A_), _lib.dptr(B_),
                                             _lib.ld_of(B_), _lib.dptr(P_), _lib.ld_of(P_),
                                             _lib.dptr(G), n))
    return G


def optimal_alpha(c2: float, c1: float, sense: str) -> float:
    """Exact optimiser of c2 a^2 + c1 a on [0, 1] (matcher.py:125-135)."""
    if c2 != 0.0:
        crit = -c1 / (2.0 * c2)
        concave = c2 < 0 if sense == "maximize" else c2 > 0
        if concave and 0.0 <= crit <= 1.0:
            return crit
    gain = c2 + c1
    if sense == "maximize":
        return 1.0 if gain >= 0.0 else 0.0
    return 1.0 if gain <= 0.0 else 0.0


def line_search_coeffs(A, B, L, P, Q, *, device=0, precision="fp64"):
    """(c2, c1) of g(a) = f(aP + (1-a)Q) (matcher.py:110-122), on the device."""
    n = A.shape[0]
    A_, B_, P_, Q_ = (_lib.f64(x) for x in (A, B, P, Q))
    L_ = _lib.f64(L) if L is not None else None
    c2 = ctypes.c_double()
    c1 = ctypes.c_double()
    h = _h(device, precision)
    with h.lock:
        _lib.check(_lib.load().goat_line_search_coeffs(
            h.ptr, n, _lib.dptr(A_), _lib.ld_of(A_), _lib.dptr(B_), _lib.ld_of(B_),
            _lib.dptr(L_) if L_ is not None else None, _lib.ld_of(L_) if L_ is not None else n,
            _lib.dptr(P_), _lib.ld_of(P_), _lib.dptr(Q_), _lib.ld_of(Q_),
            ctypes.byref(c2), ctypes.byref(c1)))
    return c2.value, c1.value


def exact_line_search(A, B, P, Q, sense: str = "maximize", *, device=0, precision="fp64") -> float:
    A = as_square_matrix(A, "A")
    B = as_square_matrix(B, "B")
    P = as_square_matrix(P, "P")
    Q = as_square_matrix(Q, "Q")
    if not (A.shape == B.shape == P.shape == Q.shape):
        raise ValueError("order mismatch in line search")
    if sense not in SENSES:
        raise ValueError(f"sense must be one of {SENSES}")
    c2, c1 = line_search_coeffs(A, B, None, P, Q, device=device, precision=precision)
    return optimal_alpha(c2, c1, sense)


def _run_sinkhorn(fn, M, sense_code, params, device, precision, *extra):
    n = M.shape[0]
    M_ = _lib.f64(M)
    Q = np.empty((n, n))
    conv = ctypes.c_int32()
    sweeps = ctypes.c_int32()
    dev = ctypes.c_double()
    h = _h(device, precision)
    with h.lock:
        if sense_code is None:
            rc = fn(h.ptr, n, _lib.dptr(M_), _lib.ld_of(M_), params.max_sweeps, params.tol,
                    _lib.dptr(Q), n, ctypes.byref(conv), ctypes.byref(sweeps), ctypes.byref(dev))
        else:
            rc = fn(h.ptr, n, _lib.dptr(M_), _lib.ld_of(M_), sense_code, params.lam,
                    params.max_sweeps, params.tol, _lib.dptr(Q), n, ctypes.byref(conv),
                    ctypes.byref(sweeps), ctypes.byref(dev))
        _lib.check(rc)
    return SinkhornResult(Q, bool(conv.value), int(sweeps.value), float(dev.value))


def lot(M, sense: str = "minimize", params: SinkhornParams = SinkhornParams(), *, device=0,
        precision="fp64") -> SinkhornResult:
    """Relaxed LAP: Sinkhorn balancing of exp(-lam * unit-range cost), on the device."""
    M = as_square_matrix(M, "M")
    if sense not in SENSES:
        raise ValueError(f"sense must be minimize or maximize, got {sense!r}")
    return _run_sinkhorn(_lib.load().goat_lot, M, _sense_code(sense), params, device, precision)


def sinkhorn_knopp(K, params: SinkhornParams = SinkhornParams(), *, device=0,
                   precision="fp64") -> SinkhornResult:
    """Balance a strictly positive matrix to doubly stochastic form, on the device."""
    K = as_square_matrix(K, "K")
    if K.min() <= 0:
        raise ValueError("sinkhorn_knopp requires strictly positive entries")
    return _run_sinkhorn(_lib.load().goat_sinkhorn_knopp, K, None, params, device, precision)


def solve_lap(M, sense: str = "minimize", *, device=0, precision="fp64") -> LapSolution:
    """Exact LAP on the device (certificate fast path, else exact augmenting paths)."""
    M = as_square_matrix(M, "M")
    code = _sense_code(sense)
    n = M.shape[0]
    M_ = _lib.f64(M)
    out = np.empty(n, dtype=np.int64)
    obj = ctypes.c_double()
    cert = ctypes.c_int32()
    h = _h(device, precision)
    with h.lock:
        _lib.check(_lib.load().goat_lap(h.ptr, n, _lib.dptr(M_), _lib.ld_of(M_), code,
                                        out.ctypes.data_as(_lib._c_i64_p), ctypes.byref(obj),
                                        ctypes.byref(cert)))
    p = out.astype(np.intp)
    # objective exactly as lap.py:57 evaluates it
    return LapSolution(assignment=p, objective=float(M[np.arange(n), p].sum()))


def relaxed_objective(A, B, L, P, *, device=0, precision="fp64") -> float:
    """f(P) = sum(A^T P B * P) (+ <L, P>) (matcher.py:170-174) = <G(P), P> / 2 with the
    gradient formed on the device."""
    P = np.asarray(P, dtype=np.float64)
    G = gradient(A, B, P, device=device, precision=precision)
    val = 0.5 * float((G * P).sum())
    if L is not None:
        val += float((np.asarray(L, dtype=np.float64) * P).sum())
    return val


#: largest order accepted by the exhaustive tie enumeration (lap.py:22)
TIE_SET_MAX_N = 10


def lap_tie_set(M, sense: str = "minimize", atol: float = 1e-9, *, device=0, precision="fp64") -> list:
    """Every permutation within ``atol`` of the LAP optimum (lap.py:61-80): the
    optimum from the device solver, then exhaustive enumeration (n <= 10)."""
    import itertools

    M = as_square_matrix(M, "M")
    if sense not in SENSES:
        raise ValueError(f"sense must be one of {SENSES}, got {sense!r}")
    n = M.shape[0]
    if n > TIE_SET_MAX_N:
        raise ValueError(f"lap_tie_set is exhaustive; n = {n} exceeds {TIE_SET_MAX_N}")
    best = solve_lap(M, sense, device=device, precision=precision).objective
    rows = np.arange(n)
    out = []
    for cand in itertools.permutations(range(n)):
        q = np.array(cand, dtype=np.intp)
        if abs(float(M[rows, q].sum()) - best) <= atol:
            out.append(q)
    return out


def random_doubly_stochastic(n: int, rng: np.random.Generator, *, device=0,
                             precision="fp64") -> np.ndarray:
    """Uniform(0,1) matrix (host RNG stream) balanced on the device (matcher.py:157-162)."""
    if n < 1:
        raise ValueError("order must be positive")
    K = rng.uniform(size=(n, n))
    return sinkhorn_knopp(K, device=device, precision=precision).matrix


def randomized_blend_init(n: int, rng: np.random.Generator, *, device=0,
                          precision="fp64") -> np.ndarray:
    """Half barycenter, half random doubly stochastic (matcher.py:165-167)."""
    return 0.5 * (barycenter(n) + random_doubly_stochastic(n, rng, device=device, precision=precision))
