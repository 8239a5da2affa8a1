"""Pin the CPU oracle (oracle/goat_oracle.py, oracle/lsap.c) to the reference.

The fixtures under tests/golden/ were produced by the unmodified reference
(tests/golden/make_golden.py).  These tests are CPU-only.
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

from golden_io import Fixture
from oracle import goat_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FW = Fixture("fw_cases.npz")
UNIT = Fixture("unit_cases.npz")
FAST_CASES = [c for c in FW.cases() if not c.startswith(("c3s", "c5p", "c2_r1"))]


@pytest.mark.parametrize("case", FAST_CASES)
def test_oracle_fw_matches_reference(case):
    A = FW.matrix(case, "A")
    B = FW.matrix(case, "B")
    o = FW.opts(case)
    seeds = FW[f"{case}/seeds"] if FW.has(f"{case}/seeds") else np.empty((0, 2), dtype=np.int64)
    trace = {}
    align, obj, iters, hist, conv = O.run_seeded(
        A, B, seeds, step_solver=o["step_solver"], sense=o["sense"], lam=o["lam"],
        max_sweeps=o["max_sweeps"], sk_tol=o["sk_tol"], max_iters=o["max_iters"],
        fw_tol=o["fw_tol"], init=o["init"], n_restarts=o["n_restarts"],
        shuffle_input=o["shuffle_input"], rng_seed=o["rng_seed"], trace=trace)
    np.testing.assert_array_equal(align, FW[f"{case}/alignment"])
    assert obj == FW[f"{case}/objective"]
    assert iters == int(FW[f"{case}/iterations"])
    assert conv == bool(FW[f"{case}/converged"])
    np.testing.assert_allclose([h[1] for h in hist], FW[f"{case}/hist_obj"], rtol=1e-12)
    alphas = np.array([np.nan if h[2] is None else h[2] for h in hist])
    np.testing.assert_allclose(alphas, FW[f"{case}/hist_alpha"], rtol=1e-12, atol=1e-15)
    if o["step_solver"] == "lot":
        np.testing.assert_array_equal(trace["sweeps"], FW[f"{case}/lot_sweeps"])
    if FW.has(f"{case}/Q"):
        for q_o, q_r in zip(trace["Q"], FW[f"{case}/Q"]):
            np.testing.assert_allclose(q_o, q_r, atol=1e-14)


FAQ = Fixture("faq_cases.npz")


@pytest.mark.parametrize("case", ["faq_w150", "faq_w150_min", "faq_w300"])
def test_oracle_faq_matches_reference(case):
    """FAQ branch (exact LAP steps, matcher.py:191-192) on tie-free weighted graphs
    (tests/golden/make_faq_golden.py): the oracle follows the reference exactly."""
    import hashlib

    from paper_2111_05366_b200 import graphs
    rep, n, smax, mi = (int(x) for x in FAQ[f"{case}/spec"])
    A, B, _ = graphs.config_pair(4, rep, n=n)
    for M, tag in ((A, "A"), (B, "B")):
        assert hashlib.sha256(np.ascontiguousarray(M).tobytes()).hexdigest() == str(FAQ[f"{case}/sha_{tag}"])
    align, obj, iters, hist, conv = O.run_seeded(
        A, B, np.empty((0, 2), dtype=np.int64), step_solver="exact_lap",
        sense="maximize" if smax else "minimize", max_iters=mi)
    np.testing.assert_array_equal(align, FAQ[f"{case}/alignment"])
    assert obj == FAQ[f"{case}/objective"]
    assert iters == int(FAQ[f"{case}/iterations"]) and conv == bool(FAQ[f"{case}/converged"])
    alphas = np.array([np.nan if h[2] is None else h[2] for h in hist])
    np.testing.assert_allclose(alphas, FAQ[f"{case}/hist_alpha"], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("name", list(UNIT["lot/names"]))
def test_oracle_lot_matches_reference(name):
    M = UNIT[f"lot/{name}/M"]
    lam, ms, tol = UNIT[f"lot/{name}/params"]
    Q, conv, sweeps, dev = O.lot(M, str(UNIT[f"lot/{name}/sense"]), lam, int(ms), tol)
    assert sweeps == int(UNIT[f"lot/{name}/sweeps"])
    assert conv == bool(UNIT[f"lot/{name}/converged"])
    np.testing.assert_allclose(Q, UNIT[f"lot/{name}/Q"], atol=1e-13)
    np.testing.assert_allclose(dev, UNIT[f"lot/{name}/dev"], rtol=1e-6, atol=1e-15)


@pytest.mark.parametrize("name", list(UNIT["sk/names"]))
def test_oracle_sinkhorn_matches_reference(name):
    Q, conv, sweeps, dev = O.balance(UNIT[f"sk/{name}/K"])
    assert sweeps == int(UNIT[f"sk/{name}/sweeps"])
    np.testing.assert_allclose(Q, UNIT[f"sk/{name}/Q"], atol=1e-14)


def test_oracle_gradient_linesearch_objective():
    for k in range(3):
        A, B, P, Q = (UNIT[f"grad/{k}/{x}"] for x in "ABPQ")
        np.testing.assert_allclose(O.qap_gradient(A, B, P), UNIT[f"grad/{k}/G"], rtol=1e-13)
        c2, c1 = O.line_coeffs(A, B, None, P, Q)
        np.testing.assert_allclose([c2, c1], UNIT[f"grad/{k}/c2c1"], rtol=1e-12)
        assert O.best_alpha(c2, c1, "maximize") == pytest.approx(float(UNIT[f"grad/{k}/alpha_max"]), abs=1e-12)
        assert O.best_alpha(c2, c1, "minimize") == pytest.approx(float(UNIT[f"grad/{k}/alpha_min"]), abs=1e-12)
        assert O.relaxed_objective(A, B, None, P) == pytest.approx(float(UNIT[f"grad/{k}/objP"]), rel=1e-13)
        p = UNIT[f"grad/{k}/perm"]
        assert O.qap_objective_perm(A, B, p) == pytest.approx(float(UNIT[f"grad/{k}/qap_perm"]), rel=1e-13)


def test_known_answers():
    # reference test_lap.py:32-40 and test_sinkhorn.py:36-40 / :30-34
    p, v = O.lap(O.TIE_MATRIX, "minimize")
    assert v == 172.0 and p.tolist() in ([0, 1, 3, 2], [0, 3, 1, 2])
    assert O.lap(O.TIE_MATRIX, "maximize")[1] == 183.0
    Q, conv, sweeps, _ = O.balance(np.array([[2.0, 1.0], [1.0, 2.0]]))
    np.testing.assert_allclose(Q, [[2 / 3, 1 / 3], [1 / 3, 2 / 3]], atol=1e-7)
    assert O.balance(np.full((4, 4), 0.25))[2] == 0


def _lsap_lib():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_build", "liblsap_oracle.so"))
    lib.oracle_lsap_min.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
    return lib


def test_c_lsap_restatement_matches_scipy_and_fixtures():
    lib = _lsap_lib()
    for name in UNIT["lap/names"]:
        M = UNIT[f"lap/{name}/M"]
        for sense in ("minimize", "maximize"):
            C = np.ascontiguousarray(-M if sense == "maximize" else M)
            out = np.empty(M.shape[0], dtype=np.int64)
            assert lib.oracle_lsap_min(M.shape[0], C.ctypes.data, out.ctypes.data) == 0
            np.testing.assert_array_equal(out, UNIT[f"lap/{name}/{sense}/assignment"])
    from scipy.optimize import linear_sum_assignment
    rng = np.random.default_rng(0)
    for t in range(200):
        n = int(rng.integers(1, 40))
        M = rng.integers(0, 3, size=(n, n)).astype(float) if t % 2 else rng.random((n, n))
        r, c = linear_sum_assignment(M)
        out = np.empty(n, dtype=np.int64)
        C = np.ascontiguousarray(M)
        lib.oracle_lsap_min(n, C.ctypes.data, out.ctypes.data)
        np.testing.assert_array_equal(out[r], c)


def test_generators_match_fixtures():
    from paper_2111_05366_b200 import graphs
    A, Bs, truth = graphs.config_pair(1, 0)
    np.testing.assert_array_equal(A, FW.matrix("c1_r0", "A"))
    np.testing.assert_array_equal(Bs, FW.matrix("c1_r0", "B"))
    A, Bs, truth = graphs.config_pair(2, 1)
    np.testing.assert_array_equal(Bs, FW.matrix("c2_r1", "B"))
    np.testing.assert_array_equal(truth, FW["c2_r1/truth"])
