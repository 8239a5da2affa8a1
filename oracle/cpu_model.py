"""Extrapolated CPU cost of the reference GOAT iteration at config 5 -- TEST /
BENCH INFRASTRUCTURE ONLY (imported by bench.py's ``cpu_baseline`` and
``--impl reference`` legs, never by the product).

Config 5 (n = 40000) cannot run through the reference on a host: the reference
densifies its inputs (core.py:22) and one float64 n x n buffer is 12.8 GB, with
~10 of them live, and one outer iteration is ~1.3e15 flop of dgemm.
§8(d) therefore asks for an EXTRAPOLATED per-iteration time, anchored on live
measurements of the same float64 numpy/OpenBLAS operations the reference
performs, on this host:

  one outer iteration of matcher.py:187-204 =
      10 dense n x n x n products (gradient :107 four, line search :118-119 four,
      objective :171 two)                      -> 10 * 2 n^3 / R_gemm
    + one LOT (sinkhorn.py:103-130): S sweeps of two n x n gemv
      (K @ v and K.T @ u, :78-80)              -> S * t_sweep(n)
    + the elementwise n^2 passes around them (shift/scale/exp of the LOT, the
      returned diag(u) K diag(v), D = P - Q, three Hadamard-sum reductions, the
      convex update and the step norm)         -> E * n^2 / R_elem
  with R_gemm, t_sweep and R_elem measured here on bounded samples at the
  config-5 row length.  The final LAP is excluded (the metric is outer
  iterations/s), which favours the reference.

``validate()`` predicts a small config (default c2, n = 1000) with the same
model and compares it with a live run of the oracle port.
"""

from __future__ import annotations

import os
import time

import numpy as np

ELEMENTWISE_PASSES = 16  # counted from matcher.py:187-204 and sinkhorn.py:103-130 (see module doc)


def _best(fn, reps):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def anchors(n=40000, band=2000, gemm=4096, reps=3, seed=0):
    """Live float64 rates on this host: dgemm GFLOP/s at a square gemm x gemm
    product, the two-gemv Sinkhorn sweep on a band x n slab (scaled to n rows),
    and an elementwise pass rate (GB/s of one read + one write)."""
    rng = np.random.default_rng(seed)
    X = rng.random((gemm, gemm))
    Y = rng.random((gemm, gemm))
    X @ Y  # first BLAS call of a process is slow (thread pool start)
    t_mm = _best(lambda: X @ Y, reps)
    r_gemm = 2.0 * gemm ** 3 / t_mm
    del X, Y
    K = rng.random((band, n)) + 0.5
    v = np.ones(n)
    u = np.ones(band)

    def sweep():
        Kv = K @ v
        w = 1.0 / Kv
        return K.T @ w

    t_sw = _best(sweep, reps) * (n / band)  # two gemv over an n x n K
    t_el = _best(lambda: np.exp(K, out=K), reps)
    r_elem = K.nbytes * 2 / t_el  # bytes moved per second (read + write)
    del K, v, u
    return {"gemm_gflops": r_gemm / 1e9, "sweep_s_at_n": t_sw, "elem_gbs": r_elem / 1e9,
            "n": n, "band": band, "gemm_order": gemm}


def iteration_seconds(n, sweeps, a):
    """Model time of one outer iteration of order n with ``sweeps`` LOT sweeps,
    using rates ``a`` measured by ``anchors`` (the sweep time scales as n^2)."""
    t_gemm = 10 * 2.0 * n ** 3 / (a["gemm_gflops"] * 1e9)
    t_sweep = a["sweep_s_at_n"] * (n / a["n"]) ** 2
    t_elem = ELEMENTWISE_PASSES * n * n * 8 * 2 / (a["elem_gbs"] * 1e9)
    return t_gemm + sweeps * t_sweep + t_elem, {"gemm": t_gemm, "lot": sweeps * t_sweep, "elementwise": t_elem}


def validate(a, config=2, max_solves=2):
    """Live oracle solve of a small config vs the model's prediction with the
    oracle's own sweep counts (the model's accuracy, reported beside the estimate)."""
    from oracle import goat_oracle as O
    from paper_2111_05366_b200 import graphs
    A, B, _ = graphs.config_pair(config, 0)
    n = A.shape[0]
    best = None
    for _ in range(max_solves):
        tr = {}
        t0 = time.perf_counter()
        P0 = np.full((n, n), 1.0 / n)
        _, hist, it, _ = O.fw_core(A, B, None, P0, trace=tr)
        t_iter = time.perf_counter() - t0  # includes the final LAP (small at c2)
        best = t_iter if best is None else min(best, t_iter)
    pred = sum(iteration_seconds(n, s, a)[0] for s in tr["sweeps"])
    return {"config": config, "n": n, "iterations": it, "sweeps": tr["sweeps"],
            "measured_s": best, "model_s": pred, "model_over_measured": pred / best}


def host_cores():
    return len(os.sched_getaffinity(0))
