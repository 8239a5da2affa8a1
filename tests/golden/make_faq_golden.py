"""FAQ (step_solver="exact_lap") goldens on tie-free inputs: the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_faq_golden.py

FAQ's trajectory is discontinuous in the gradient: every step is an exact LAP
(matcher.py:191-192, lap.py:48-58), so on 0/1 graphs -- where gradients tie
exactly -- the chosen permutation depends on scipy's tie order and on last-bit
rounding.  Weighted graphs (config 4's law: lognormal weights, directed) have no
ties at any iterate, so the whole trajectory is pinned: these cases are the
exact-parity targets for the device LAP step (tests/test_parity_gpu.py) and pin
the oracle's FAQ branch (tests/test_oracle.py).

Inputs are ``graphs.config_pair(4, r, n=...)``; the fixture stores their
SHA-256 (the tests regenerate them), the reference's MatchResult, and the
smallest gap between the best and second-best row-wise reduced costs is not
needed: uniqueness is evidenced by the reference and the device agreeing.
Writes ``tests/golden/faq_cases.npz``.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import otmatch  # noqa: E402  (the reference)
from paper_2111_05366_b200 import graphs  # noqa: E402

# name -> (replicate, n, objective_sense, max_iters)
CASES = {
    "faq_w150": (0, 150, "maximize", 30),      # n < 256: scipy-order shortest augmenting paths
    "faq_w150_min": (1, 150, "minimize", 30),
    "faq_w300": (2, 300, "maximize", 30),      # n >= 256: auction + certified repair
    "faq_w700": (3, 700, "maximize", 12),
}


def digest(M):
    return hashlib.sha256(np.ascontiguousarray(M, dtype=np.float64).tobytes()).hexdigest()


def main():
    store = {}
    for name, (rep, n, sense, mi) in CASES.items():
        A, Bs, truth = graphs.config_pair(4, rep, n=n)
        opts = otmatch.MatchOptions(step_solver="exact_lap", objective_sense=sense, max_iters=mi)
        res = otmatch.frank_wolfe_match(A, Bs, opts)
        store[f"{name}/spec"] = np.array([rep, n, 1 if sense == "maximize" else 0, mi], dtype=np.int64)
        store[f"{name}/sha_A"] = np.array(digest(A))
        store[f"{name}/sha_B"] = np.array(digest(Bs))
        store[f"{name}/alignment"] = np.asarray(res.alignment, dtype=np.int64)
        store[f"{name}/objective"] = np.float64(res.objective)
        store[f"{name}/iterations"] = np.int64(res.iterations)
        store[f"{name}/converged"] = np.bool_(res.converged)
        store[f"{name}/hist_obj"] = np.array([h[1] for h in res.iterate_history])
        store[f"{name}/hist_alpha"] = np.array([np.nan if h[2] is None else h[2] for h in res.iterate_history])
        print(f"{name}: n={n} {sense} iters={res.iterations} conv={res.converged} obj={res.objective!r} "
              f"alpha={[h[2] for h in res.iterate_history[1:]]} match={np.mean(res.alignment == truth):.3f}",
              flush=True)
    np.savez_compressed(os.path.join(HERE, "faq_cases.npz"), **store)


if __name__ == "__main__":
    main()
