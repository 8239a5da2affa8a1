"""fp32-mode status against the reference goldens (GPU; prints one JSON line per case).

Full-size c3/c4 (tests/golden/full_cases.npz) and the scaled fw_cases goldens that
the fp32 parity test does not list (c3s_r0, c5p_r0): permutation / objective /
sweeps / alpha vs the unmodified reference, for DESIGN.md §4's fp32 statement.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2111_05366_b200 as gb  # noqa: E402
from golden_io import Fixture  # noqa: E402
from paper_2111_05366_b200 import graphs  # noqa: E402

precisions = sys.argv[1].split(",") if len(sys.argv) > 1 else ["fp32"]
FULL = np.load(os.path.join(ROOT, "tests", "golden", "full_cases.npz"))
FW = Fixture("fw_cases.npz")


def report(name, res, ref_align, ref_obj, ref_sweeps, ref_alpha, precision, dt):
    al = [h[2] for h in res.iterate_history[1:]]
    print(json.dumps({
        "case": name, "precision": precision, "same_perm": bool(np.array_equal(res.alignment, ref_align)),
        "perm_agree": float(np.mean(res.alignment == ref_align)), "objective": res.objective,
        "ref_objective": float(ref_obj), "iterations": res.iterations, "sweeps": res.diagnostics["lot_sweeps"],
        "ref_sweeps": [int(x) for x in ref_sweeps], "alpha": al, "ref_alpha": [float(x) for x in ref_alpha],
        "lot_dev": res.diagnostics["lot_deviation"], "solve_s": dt}), flush=True)


for precision in precisions:
    for cfg in (4, 3):
        A, B, _ = graphs.config_pair(cfg, 0)
        k = f"c{cfg}_full"
        gb.frank_wolfe_match(A[:64, :64], B[:64, :64], gb.MatchOptions(step_solver="lot", precision=precision))
        t0 = time.perf_counter()
        r = gb.frank_wolfe_match(A, B, gb.MatchOptions(step_solver="lot", precision=precision))
        report(k, r, FULL[f"{k}/alignment"], FULL[f"{k}/objective"], FULL[f"{k}/lot_sweeps"],
               FULL[f"{k}/hist_alpha"][1:], precision, time.perf_counter() - t0)
    for case in ("c3s_r0", "c5p_r0"):
        A, B = FW.matrix(case, "A"), FW.matrix(case, "B")
        t0 = time.perf_counter()
        r = gb.frank_wolfe_match(A, B, gb.MatchOptions(step_solver="lot", precision=precision))
        report(case, r, FW[f"{case}/alignment"], FW[f"{case}/objective"], FW[f"{case}/lot_sweeps"],
               FW[f"{case}/hist_alpha"][1:], precision, time.perf_counter() - t0)
