"""CPU oracle for the GOAT iteration -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm (``otmatch``,
arXiv 2111.05366) for the one hot path this repository accelerates: the
Frank-Wolfe engine ``_fw_core`` with the LOT (Sinkhorn) step direction, plus
the pieces it calls.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as a checker or a timed CPU baseline -- never as the product path.
The product (``paper_2111_05366_b200``) fails loudly when its CUDA library
is missing; it never routes through this file.

Parity pinning: ``tests/golden/make_golden.py`` runs the unmodified
reference (imported from /root/reference in the build container) on seeded
inputs and stores its outputs under ``tests/golden/``; ``tests/test_oracle.py``
checks this restatement against those fixtures bit-for-bit (alignment,
iterations, sweep counts) and to 1e-12 (objectives, alpha sequence).

All arithmetic is float64, as in the reference (``core.py:22``).  Each
function cites the reference ``file:line`` it restates.  The exact LAP is
``scipy.optimize.linear_sum_assignment`` (scipy 1.18.1 in this image), which is
what the reference itself calls (``lap.py:55``); ``oracle/lsap.c`` restates
that solver's published shortest-augmenting-path algorithm (Crouse 2016) in C
and is checked against scipy by ``tests/test_oracle.py``.
"""

from __future__ import annotations

import numpy as np

__all__ = [
    "qap_gradient", "line_coeffs", "best_alpha", "relaxed_objective",
    "balance", "balance_log", "lot", "lap", "fw_core", "run_seeded",
    "qap_objective_perm", "TIE_MATRIX",
]

# 4x4 matrix whose minimum LAP has a two-way tie at 172 (max = 183);
# known-answer values from the reference test-suite (test_lap.py:11-20,32-40).
TIE_MATRIX = np.array(
    [[40.0, 50.0, 60.0, 65.0],
     [30.0, 38.0, 46.0, 48.0],
     [25.0, 33.0, 41.0, 43.0],
     [39.0, 45.0, 51.0, 59.0]]
)


def _square(M):
    # core.py:17-27 -- float cast + square + finite check
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError(f"must be square, got shape {M.shape}")
    if not np.all(np.isfinite(M)):
        raise ValueError("contains non-finite entries")
    return M


def qap_gradient(A, B, P):
    """matcher.py:100-107: A P B^T + A^T P B, evaluated left to right."""
    return A @ P @ B.T + A.T @ P @ B


def line_coeffs(A, B, L, P, Q):
    """matcher.py:110-122: (c2, c1) of g(a) = f(aP + (1-a)Q) - const."""
    D = P - Q
    ADB = A.T @ D @ B
    c2 = float((ADB * D).sum())
    c1 = float((ADB * Q).sum() + (A.T @ Q @ B * D).sum())
    if L is not None:
        c1 += float((L * D).sum())
    return c2, c1


def best_alpha(c2, c1, sense):
    """matcher.py:125-135: exact maximiser/minimiser of c2 a^2 + c1 a on [0,1]."""
    if c2 != 0.0:
        crit = -c1 / (2.0 * c2)
        ok = (c2 < 0) if sense == "maximize" else (c2 > 0)
        if ok and 0.0 <= crit <= 1.0:
            return crit
    end = c2 + c1
    if sense == "maximize":
        return 1.0 if end >= 0.0 else 0.0
    return 1.0 if end <= 0.0 else 0.0


def relaxed_objective(A, B, L, P):
    """matcher.py:170-174: trace(A^T P B P^T) (+ <L, P>)."""
    val = float((A.T @ P @ B * P).sum())
    if L is not None:
        val += float((L * P).sum())
    return val


def _marginal_dev(P):
    # sinkhorn.py:53-57
    return max(np.abs(P.sum(axis=1) - 1.0).max(), np.abs(P.sum(axis=0) - 1.0).max())


def balance(K, max_sweeps=1000, tol=1e-8):
    """sinkhorn.py:60-85 (standard-domain Sinkhorn-Knopp).

    Returns (matrix, converged, sweeps, deviation).
    """
    K = _square(K)
    if K.min() <= 0:
        raise ValueError("sinkhorn_knopp requires strictly positive entries")
    dev = _marginal_dev(K)
    if dev < tol:
        return K, True, 0, dev
    v = np.ones(K.shape[0])
    Kv = K @ v
    for sweep in range(1, max_sweeps + 1):
        u = 1.0 / Kv
        v = 1.0 / (K.T @ u)
        Kv = K @ v
        dev = float(np.abs(u * Kv - 1.0).max())
        if dev < tol:
            return u[:, None] * K * v[None, :], True, sweep, dev
    return u[:, None] * K * v[None, :], False, max_sweeps, dev


def _lse(X, axis):
    # scipy.special.logsumexp restated (max-shifted), as used at sinkhorn.py:94-95
    m = X.max(axis=axis, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    s = np.log(np.exp(X - m).sum(axis=axis, keepdims=True)) + m
    return np.squeeze(s, axis=axis)


def balance_log(E, max_sweeps=1000, tol=1e-8):
    """sinkhorn.py:88-100 (log-domain fallback; no 0-sweep pre-check)."""
    n = E.shape[0]
    f = np.zeros(n)
    g = np.zeros(n)
    P = None
    dev = np.inf
    for sweep in range(1, max_sweeps + 1):
        f = -_lse(E + g[None, :], axis=1)
        g = -_lse(E + f[:, None], axis=0)
        P = np.exp(E + f[:, None] + g[None, :])
        dev = _marginal_dev(P)
        if dev < tol:
            return P, True, sweep, dev
    return P, False, max_sweeps, dev


def lot(M, sense="minimize", lam=100.0, max_sweeps=1000, tol=1e-8):
    """sinkhorn.py:103-130: relaxed LAP by Sinkhorn on the unit-range Gibbs kernel."""
    M = _square(M)
    shifted = (M.max() - M) if sense == "maximize" else (M - M.min())
    scale = shifted.max()
    n = M.shape[0]
    if scale == 0.0:
        return np.full((n, n), 1.0 / n), True, 0, 0.0
    E = (-lam / scale) * shifted
    K = np.exp(E)
    if K.min() <= 0.0:
        return balance_log(E, max_sweeps, tol)
    return balance(K, max_sweeps, tol)


def lap(M, sense="minimize"):
    """lap.py:48-58: exact LAP through the reference's own dependency."""
    from scipy.optimize import linear_sum_assignment

    M = _square(M)
    rows, cols = linear_sum_assignment(M, maximize=(sense == "maximize"))
    p = np.empty(M.shape[0], dtype=np.intp)
    p[rows] = cols
    return p, float(M[rows, cols].sum())


def qap_objective_perm(A, B, p):
    """core.py:120-124: sum_ij A_ij B_{p(i) p(j)}."""
    return float((A * B[np.ix_(p, p)]).sum())


def fw_core(A, B, L, P0, *, step_solver="lot", sense="maximize", lam=100.0,
            max_sweeps=1000, sk_tol=1e-8, max_iters=30, fw_tol=1e-2, trace=None):
    """matcher.py:177-212: one Frank-Wolfe run.

    Returns (assignment, history, iterations, converged).  When ``trace`` is a
    dict it receives per-iteration diagnostics the reference computes but
    discards (LOT sweeps / converged / deviation, step norms, Q snapshots).
    """
    P = P0
    history = [(0, relaxed_objective(A, B, L, P), None)]
    converged = False
    iterations = 0
    if trace is not None:
        trace.setdefault("sweeps", []); trace.setdefault("lot_converged", [])
        trace.setdefault("lot_dev", []); trace.setdefault("step", [])
        trace.setdefault("Q", [])
    for i in range(1, max_iters + 1):
        G = qap_gradient(A, B, P)
        if L is not None:
            G = G + L
        if step_solver == "exact_lap":
            p, _ = lap(G, sense)
            Q = np.zeros_like(G)
            Q[np.arange(G.shape[0]), p] = 1.0
            sw, cv, dv = 0, True, 0.0
        else:
            Q, cv, sw, dv = lot(G, sense, lam, max_sweeps, sk_tol)
        c2, c1 = line_coeffs(A, B, L, P, Q)
        alpha = best_alpha(c2, c1, sense)
        P_new = alpha * P + (1.0 - alpha) * Q
        history.append((i, relaxed_objective(A, B, L, P_new), alpha))
        iterations = i
        step = float(np.linalg.norm(P_new - P))
        if trace is not None:
            trace["sweeps"].append(sw); trace["lot_converged"].append(cv)
            trace["lot_dev"].append(dv); trace["step"].append(step)
            trace["Q"].append(Q)
        P = P_new
        if step < fw_tol:
            converged = True
            break
    G = qap_gradient(A, B, P)
    if L is not None:
        G = G + L
    assignment, _ = lap(G, sense)
    if trace is not None:
        trace["G_final"] = G
        trace["P_final"] = P
    return assignment, history, iterations, converged


def _sinkhorn_uniform(n, rng):
    # matcher.py:157-167 (random_doubly_stochastic / randomized_blend_init)
    K = rng.uniform(size=(n, n))
    return balance(K)[0]


def run_seeded(A, B, seeds, *, step_solver="lot", sense="maximize", lam=100.0,
               max_sweeps=1000, sk_tol=1e-8, max_iters=30, fw_tol=1e-2,
               init="barycenter", n_restarts=1, shuffle_input=False, rng_seed=0,
               trace=None):
    """matcher.py:230-295: seed reduction + restarts around ``fw_core``.

    Returns (alignment, objective, iterations, history, converged).
    """
    A = _square(A)
    B = _square(B)
    if A.shape != B.shape:
        raise ValueError("order mismatch")
    n = A.shape[0]
    seeds = np.asarray(seeds, dtype=np.intp).reshape(-1, 2)
    m = seeds.shape[0]
    if m >= n:
        raise ValueError("seed count must be less than order")
    free1 = np.setdiff1d(np.arange(n), seeds[:, 0]) if m else np.arange(n)
    free2 = np.setdiff1d(np.arange(n), seeds[:, 1]) if m else np.arange(n)
    o1 = np.concatenate([seeds[:, 0], free1]).astype(np.intp)
    o2 = np.concatenate([seeds[:, 1], free2]).astype(np.intp)
    Ar = A[np.ix_(o1, o1)]
    Br = B[np.ix_(o2, o2)]
    nf = n - m
    best = None
    for r in range(n_restarts):
        rng = np.random.default_rng([rng_seed, r])
        shuf = rng.permutation(nf).astype(np.intp) if (shuffle_input and nf > 1) \
            else np.arange(nf, dtype=np.intp)
        inv = np.empty_like(shuf)
        inv[shuf] = np.arange(nf)
        B22 = Br[m:, m:][np.ix_(inv, inv)]
        B12 = Br[:m, m:][:, inv]
        B21 = Br[m:, :m][inv, :]
        A22 = Ar[m:, m:]
        L = (Ar[m:, :m] @ B21.T + Ar[:m, m:].T @ B12) if m else None
        if nf == 1:
            p22 = np.zeros(1, dtype=np.intp)
            hist = [(0, relaxed_objective(A22, B22, L, np.ones((1, 1))), None)]
            iters, conv = 0, True
        else:
            if isinstance(init, str):
                if init == "barycenter":
                    P0 = np.full((nf, nf), 1.0 / nf)
                else:
                    P0 = 0.5 * (np.full((nf, nf), 1.0 / nf) + _sinkhorn_uniform(nf, rng))
            else:
                P0 = _square(init)
            p22, hist, iters, conv = fw_core(
                A22, B22, L, P0, step_solver=step_solver, sense=sense, lam=lam,
                max_sweeps=max_sweeps, sk_tol=sk_tol, max_iters=max_iters,
                fw_tol=fw_tol, trace=trace)
        p22 = inv[p22]
        align = np.empty(n, dtype=np.intp)
        align[o1[:m]] = o2[:m]
        align[o1[m:]] = o2[m + p22]
        obj = qap_objective_perm(A, B, align)
        better = best is None or ((obj > best[1]) if sense == "maximize" else (obj < best[1]))
        if better:
            best = (align, obj, iters, hist, conv)
    return best
