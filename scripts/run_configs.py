"""End-to-end GOAT solves for BASELINE configs on the GPU (fp32 unless noted):
time-to-converge, iterations, phase split, LOT sweeps, certificate, match ratio."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2111_05366_b200 as gb
from paper_2111_05366_b200 import graphs

cfgs = [int(c) for c in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "4", "3"])]
for c in cfgs:
    spec = graphs.CONFIGS[c]
    n = spec["n"] if len(sys.argv) <= 2 else int(sys.argv[2])
    A, Bs, truth = graphs.config_pair(c, 0, n=n)
    opts = gb.MatchOptions(step_solver="lot", precision=spec["precision"], fw_tol=spec["fw_tol"])
    gb.frank_wolfe_match(A[:50, :50], Bs[:50, :50], opts)  # warm
    t0 = time.perf_counter()
    r = gb.frank_wolfe_match(A, Bs, opts)
    dt = time.perf_counter() - t0
    d = r.diagnostics
    print(json.dumps({"config": c, "n": n, "precision": spec["precision"], "wall_s": round(dt, 3),
                      "iterations": r.iterations, "converged": r.converged, "objective": r.objective,
                      "match_ratio": float(np.mean(r.alignment == truth)),
                      "lap_certified": d["lap_certified"], "lot_sweeps": d["lot_sweeps"],
                      "phase_ms": {k: round(v, 2) for k, v in d["time_ms"].items()}}), flush=True)
