"""Generate golden fixtures by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``otmatch`` from /root/reference/pkg/src, runs it on seeded inputs
and writes ``tests/golden/*.npz``.  Observe-only wrappers record the per-LOT
diagnostics the reference computes but discards (sweeps / converged /
deviation, matcher.py:194).  The fixtures pin ``oracle/goat_oracle.py``
(tests/test_oracle.py) and are the parity targets for the CUDA path
(tests/test_parity_gpu.py).  0/1 matrices are stored bit-packed.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import otmatch  # noqa: E402  (the reference)
import otmatch.matcher as ref_matcher  # noqa: E402
from paper_2111_05366_b200 import graphs  # noqa: E402


def pack(M):
    M = np.asarray(M, dtype=np.float64)
    if np.isin(M, (0.0, 1.0)).all():
        return {"bits": np.packbits(M.astype(np.uint8).ravel()), "n": np.int64(M.shape[0])}
    return {"dense": M}


def put(store, prefix, key, M):
    for k, v in pack(M).items():
        store[f"{prefix}/{key}.{k}"] = v


class LotRecorder:
    def __init__(self):
        self.log = []
        self.keep_q = False

    def __call__(self, M, sense="minimize", params=otmatch.SinkhornParams()):
        res = otmatch.sinkhorn.lot(M, sense, params)
        self.log.append(res)
        return res


def run_fw(store, name, A, B, opts, seeds=None, keep_q=False, truth=None):
    rec = LotRecorder()
    orig = ref_matcher.lot
    ref_matcher.lot = rec
    try:
        if seeds is None:
            res = otmatch.frank_wolfe_match(A, B, opts)
        else:
            res = otmatch.seeded_match(A, B, otmatch.SeedSet(seeds), opts)
    finally:
        ref_matcher.lot = orig
    put(store, name, "A", A)
    put(store, name, "B", B)
    if seeds is not None:
        store[f"{name}/seeds"] = np.asarray(seeds, dtype=np.int64).reshape(-1, 2)
    if truth is not None:
        store[f"{name}/truth"] = np.asarray(truth, dtype=np.int64)
    o = opts
    store[f"{name}/opts"] = np.array([
        o.max_iters, o.fw_tol, o.sinkhorn.lam, o.sinkhorn.max_sweeps, o.sinkhorn.tol,
        o.n_restarts, float(o.shuffle_input), o.rng_seed,
        1.0 if o.objective_sense == "maximize" else 0.0,
        1.0 if o.step_solver == "lot" else 0.0,
    ])
    store[f"{name}/init"] = np.array(o.init if isinstance(o.init, str) else "matrix")
    store[f"{name}/alignment"] = np.asarray(res.alignment, dtype=np.int64)
    store[f"{name}/objective"] = np.float64(res.objective)
    store[f"{name}/iterations"] = np.int64(res.iterations)
    store[f"{name}/converged"] = np.bool_(res.converged)
    store[f"{name}/hist_obj"] = np.array([h[1] for h in res.iterate_history])
    store[f"{name}/hist_alpha"] = np.array(
        [np.nan if h[2] is None else h[2] for h in res.iterate_history])
    store[f"{name}/lot_sweeps"] = np.array([r.sweeps for r in rec.log], dtype=np.int64)
    store[f"{name}/lot_converged"] = np.array([r.converged for r in rec.log])
    store[f"{name}/lot_dev"] = np.array([r.deviation for r in rec.log])
    if keep_q:
        store[f"{name}/Q"] = np.stack([r.matrix for r in rec.log])
    print(f"{name}: n={A.shape[0]} iters={res.iterations} obj={res.objective} "
          f"sweeps={[r.sweeps for r in rec.log]} wall={res.wall_time:.2f}s", flush=True)


def lot_opts(**kw):
    sk = {k: kw.pop(k) for k in ("lam", "max_sweeps", "tol") if k in kw}
    return otmatch.MatchOptions(step_solver="lot", sinkhorn=otmatch.SinkhornParams(**sk), **kw)


def fw_cases():
    store = {}
    # Config 1 (n=100), replicates 0..4: reference sampler == ours, checked here.
    for r in range(5):
        rng = np.random.default_rng([1, r])
        A, B = otmatch.sample_er_pair(100, 0.5, 0.9, rng)
        Bs, truth = otmatch.shuffle_pair(B, rng)
        A2, Bs2, t2 = graphs.config_pair(1, r)
        assert np.array_equal(A, A2) and np.array_equal(Bs, Bs2) and np.array_equal(truth, t2)
        run_fw(store, f"c1_r{r}", A, Bs, lot_opts(fw_tol=0.03), keep_q=(r == 0), truth=truth)
    # Config 2 (n=1000, directed), replicates 0..1.
    for r in range(2):
        A, Bs, truth = graphs.config_pair(2, r)
        run_fw(store, f"c2_r{r}", A, Bs, lot_opts(), truth=truth)
    # Config 3 scaled to n=600 (same block proportions / probabilities / rho).
    rng = np.random.default_rng([3, 0])
    spec = otmatch.SbmSpec((240, 240, 120), np.array([[.3, .05, .05], [.05, .3, .05], [.05, .05, .3]]), 0.7)
    A, B = otmatch.sample_sbm_pair(spec, rng)
    Bs, truth = otmatch.shuffle_pair(B, rng)
    A2, Bs2, _ = graphs.config_pair(3, 0, n=600)
    assert np.array_equal(A, A2) and np.array_equal(Bs, Bs2)
    run_fw(store, "c3s_r0", A, Bs, lot_opts(), truth=truth)
    # Config 4 scaled to n=200 (weighted directed).
    A, Bs, truth = graphs.config_pair(4, 0, n=200)
    run_fw(store, "c4s_r0", A, Bs, lot_opts(), truth=truth)
    # Config-5 proxy: sparse undirected ER at the same mean degree as the
    # survey's n=2000 proxy (20), scaled to n=1500.
    rng = np.random.default_rng([5, 0])
    A, B = otmatch.sample_er_pair(1500, 20.0 / 1500, 0.9, rng)
    Bs, truth = otmatch.shuffle_pair(B, rng)
    run_fw(store, "c5p_r0", A, Bs, lot_opts(), truth=truth)
    # FAQ (exact_lap step) on config-1 input: the §8f "next" row.
    A = store["c1_r0/A.bits"]
    rng = np.random.default_rng([1, 0])
    A, B = otmatch.sample_er_pair(100, 0.5, 0.9, rng)
    Bs, truth = otmatch.shuffle_pair(B, rng)
    run_fw(store, "faq_c1_r0", A, Bs, otmatch.MatchOptions(step_solver="exact_lap", fw_tol=0.03))
    # Seeded SBM (m=10 of 60), GOAT.
    spec = otmatch.SbmSpec((20, 20, 20), np.array([[.7, .3, .4], [.3, .7, .3], [.4, .3, .7]]), 0.9)
    rng = np.random.default_rng([16, 0])
    A, B = otmatch.sample_sbm_pair(spec, rng)
    Bs, truth = otmatch.shuffle_pair(B, rng)
    g1 = rng.choice(60, size=10, replace=False)
    run_fw(store, "seeded_sbm60", A, Bs, lot_opts(), seeds=np.stack([g1, truth[g1]], axis=1), truth=truth)
    # Randomized-blend init + restarts + input shuffling (host RNG streams).
    rng = np.random.default_rng(8)
    A = (rng.random((15, 15)) < 0.3).astype(float)
    B = (rng.random((15, 15)) < 0.3).astype(float)
    run_fw(store, "blend15", A, B, lot_opts(init="randomized_blend", n_restarts=3,
                                            shuffle_input=True, rng_seed=99))
    # Minimisation on dense float matrices.
    rng = np.random.default_rng(7)
    A = rng.random((12, 12)); B = rng.random((12, 12))
    run_fw(store, "min12", A, B, lot_opts(objective_sense="minimize"))
    # Planted isomorphic ER at n=200, p=log n/n (acceptance criterion 4).
    master = np.random.default_rng(0)
    for r in range(3):
        A, B = otmatch.sample_er_pair(200, np.log(200) / 200, 1.0, master)
        Bs, truth = otmatch.shuffle_pair(B, master)
        run_fw(store, f"iso200_r{r}", A, Bs, lot_opts(), truth=truth)
    np.savez_compressed(os.path.join(HERE, "fw_cases.npz"), **store)


def unit_cases():
    store = {}
    rng = np.random.default_rng(2024)
    lots = []
    lots.append(("tie_min", otmatch.lap.__dict__.get("TIE", None) or np.array(
        [[40.0, 50.0, 60.0, 65.0], [30.0, 38.0, 46.0, 48.0],
         [25.0, 33.0, 41.0, 43.0], [39.0, 45.0, 51.0, 59.0]]), "minimize", {}))
    lots.append(("unif50", rng.uniform(100.0, 150.0, (50, 50)), "minimize", {}))
    lots.append(("unif120_max", rng.uniform(100.0, 150.0, (120, 120)), "maximize", {}))
    lots.append(("rand8_1sweep", rng.uniform(0.5, 2.0, (8, 8)), "minimize", {"max_sweeps": 1, "tol": 1e-14}))
    lots.append(("rand30_lam10", rng.random((30, 30)), "maximize", {"lam": 10.0}))
    lots.append(("logpath5", rng.random((5, 5)), "minimize", {"lam": 5e4, "max_sweeps": 5000}))
    M = np.full((5, 5), 100.0) + rng.random((5, 5)); np.fill_diagonal(M, rng.random(5))
    lots.append(("sharp5", M, "minimize", {}))
    lots.append(("const4", np.full((4, 4), 2.0), "minimize", {}))
    perm = rng.permutation(7); Pm = np.zeros((7, 7)); Pm[np.arange(7), perm] = 1.0
    lots.append(("perm7_0sweeps", Pm * 3.0, "maximize", {}))
    lots.append(("rand200_max", rng.random((200, 200)), "maximize", {"max_sweeps": 300}))
    names = []
    for name, M, sense, kw in lots:
        res = otmatch.lot(M, sense, otmatch.SinkhornParams(**kw))
        store[f"lot/{name}/M"] = M
        store[f"lot/{name}/sense"] = np.array(sense)
        store[f"lot/{name}/params"] = np.array([kw.get("lam", 100.0), kw.get("max_sweeps", 1000), kw.get("tol", 1e-8)])
        store[f"lot/{name}/Q"] = res.matrix
        store[f"lot/{name}/converged"] = np.bool_(res.converged)
        store[f"lot/{name}/sweeps"] = np.int64(res.sweeps)
        store[f"lot/{name}/dev"] = np.float64(res.deviation)
        names.append(name)
        print(f"lot {name}: sweeps={res.sweeps} conv={res.converged} dev={res.deviation:.3e}")
    store["lot/names"] = np.array(names)
    sk = []
    sk.append(("ones5", np.ones((5, 5)), {}))
    sk.append(("ds4", np.full((4, 4), 0.25), {}))
    sk.append(("two", np.array([[2.0, 1.0], [1.0, 2.0]]), {}))
    sk.append(("unif6", rng.uniform(0.5, 2.0, (6, 6)), {}))
    sk.append(("unif40", rng.uniform(size=(40, 40)), {}))
    names = []
    for name, K, kw in sk:
        res = otmatch.sinkhorn_knopp(K, otmatch.SinkhornParams(**kw))
        store[f"sk/{name}/K"] = K
        store[f"sk/{name}/Q"] = res.matrix
        store[f"sk/{name}/converged"] = np.bool_(res.converged)
        store[f"sk/{name}/sweeps"] = np.int64(res.sweeps)
        store[f"sk/{name}/dev"] = np.float64(res.deviation)
        names.append(name)
    store["sk/names"] = np.array(names)
    laps = []
    laps.append(("rand50", rng.random((50, 50))))
    laps.append(("int30", rng.integers(0, 3, size=(30, 30)).astype(float)))
    laps.append(("int8", rng.integers(0, 3, size=(8, 8)).astype(float)))
    laps.append(("const6", np.full((6, 6), 1.5)))
    laps.append(("zeros5", np.zeros((5, 5))))
    laps.append(("rand300", rng.random((300, 300))))
    names = []
    for name, M in laps:
        for sense in ("minimize", "maximize"):
            sol = otmatch.solve_lap(M, sense)
            store[f"lap/{name}/M"] = M
            store[f"lap/{name}/{sense}/assignment"] = np.asarray(sol.assignment, dtype=np.int64)
            store[f"lap/{name}/{sense}/objective"] = np.float64(sol.objective)
        names.append(name)
    store["lap/names"] = np.array(names)
    # gradient + line search + objective on small dense inputs
    for k in range(3):
        n = [5, 9, 33][k]
        A = rng.random((n, n)); B = rng.random((n, n))
        P = otmatch.random_doubly_stochastic(n, rng)
        Q = otmatch.random_doubly_stochastic(n, rng)
        store[f"grad/{k}/A"] = A; store[f"grad/{k}/B"] = B
        store[f"grad/{k}/P"] = P; store[f"grad/{k}/Q"] = Q
        store[f"grad/{k}/G"] = otmatch.gradient(A, B, P)
        c2, c1 = ref_matcher._line_search_coeffs(A, B, None, P, Q)
        store[f"grad/{k}/c2c1"] = np.array([c2, c1])
        store[f"grad/{k}/alpha_max"] = np.float64(otmatch.exact_line_search(A, B, P, Q, "maximize"))
        store[f"grad/{k}/alpha_min"] = np.float64(otmatch.exact_line_search(A, B, P, Q, "minimize"))
        store[f"grad/{k}/objP"] = np.float64(ref_matcher._objective(A, B, None, P))
        p = rng.permutation(n)
        store[f"grad/{k}/perm"] = p.astype(np.int64)
        store[f"grad/{k}/qap_perm"] = np.float64(otmatch.qap_objective(A, B, p))
    np.savez_compressed(os.path.join(HERE, "unit_cases.npz"), **store)


if __name__ == "__main__":
    unit_cases()
    fw_cases()
