"""at n = 40000 the CPU reference cannot run, so the GPU
fp64 mode (bit-compatible with the reference at every size it can run) is the
oracle for the fp32 path on the seeded config-5 input graphs.config_pair(5, 0).

Prints one JSON line: permutation / objective / alpha / sweep agreement of the two
full solves through the public API, and max |Q32 - Q64| of one LOT on the same
fp32-representable gradient (the 1e-3 fp32 bar of BASELINE.json).

usage: python scripts/c5_fp64_oracle.py [n] [max_iters]
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import torch

import paper_2111_05366_b200 as gb
from paper_2111_05366_b200 import _lib, graphs

n_arg = int(sys.argv[1]) if len(sys.argv) > 1 else None
max_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
A, Bs, truth = graphs.config_pair(5, 0, n=n_arg)
n = A.n


def to_scipy(g):
    return sp.csr_matrix((np.ones(g.indices.size), g.indices, g.indptr), shape=(g.n, g.n))


sA, sB = to_scipy(A), to_scipy(Bs)
out = {"n": n, "max_iters": max_iters}
runs = {}
for prec in ("fp64", "fp32"):
    t0 = time.perf_counter()
    r = gb.frank_wolfe_match(sA, sB, gb.MatchOptions(step_solver="lot", precision=prec, max_iters=max_iters))
    dt = time.perf_counter() - t0
    runs[prec] = r
    out[prec] = {"solve_s": dt, "iterations": r.iterations, "converged": r.converged, "objective": r.objective,
                 "alpha": [h[2] for h in r.iterate_history[1:]], "hist_obj": [h[1] for h in r.iterate_history],
                 "lot_sweeps": r.diagnostics["lot_sweeps"], "lot_fp64_from": r.diagnostics.get("lot_fp64_from"),
                 "lot_deviation": r.diagnostics["lot_deviation"],
                 "match_ratio": float(np.mean(r.alignment == truth)),
                 "phase_ms": {k: round(v, 1) for k, v in r.diagnostics["time_ms"].items()}}
    _lib.release_handles()
    torch.cuda.empty_cache()
r64, r32 = runs["fp64"], runs["fp32"]
out["same_permutation"] = bool(np.array_equal(r64.alignment, r32.alignment))
out["permutation_agreement"] = float(np.mean(r64.alignment == r32.alignment))
out["same_objective"] = r64.objective == r32.objective
out["same_iterations"] = r64.iterations == r32.iterations
m = min(r64.iterations, r32.iterations)
a64 = np.array(out["fp64"]["alpha"][:m]); a32 = np.array(out["fp32"]["alpha"][:m])
out["alpha_max_abs_diff"] = float(np.max(np.abs(a64 - a32))) if m else 0.0
h64 = np.array(out["fp64"]["hist_obj"][:m + 1]); h32 = np.array(out["fp32"]["hist_obj"][:m + 1])
out["hist_obj_max_rel_diff"] = float(np.max(np.abs(h64 - h32) / np.maximum(1.0, np.abs(h64))))
print(json.dumps(out), flush=True)
