"""GPU parity of the CUDA path (libgoat.so) against the reference goldens and
the CPU oracle.  Tolerances follow BASELINE.json's north star: the same final
permutation and an integer-exact objective for 0/1 graphs; doubly stochastic
iterates within 1e-5 max-abs in fp64 mode and 1e-3 in fp32 mode."""
import numpy as np
import pytest

import paper_2111_05366_b200 as gb
from golden_io import Fixture
from oracle import goat_oracle as O

pytestmark = pytest.mark.gpu

FW = Fixture("fw_cases.npz")
UNIT = Fixture("unit_cases.npz")

TOL_Q = {"fp64": 1e-5, "fp32": 1e-3}


def _opts(case, precision):
    o = FW.opts(case)
    return gb.MatchOptions(
        step_solver=o["step_solver"], init=o["init"], max_iters=o["max_iters"], fw_tol=o["fw_tol"],
        n_restarts=o["n_restarts"], shuffle_input=o["shuffle_input"], rng_seed=o["rng_seed"],
        objective_sense=o["sense"], precision=precision,
        sinkhorn=gb.SinkhornParams(lam=o["lam"], max_sweeps=o["max_sweeps"], tol=o["sk_tol"]))


def _run(case, precision):
    A = FW.matrix(case, "A")
    B = FW.matrix(case, "B")
    opts = _opts(case, precision)
    if FW.has(f"{case}/seeds"):
        return gb.seeded_match(A, B, gb.SeedSet(FW[f"{case}/seeds"]), opts)
    return gb.frank_wolfe_match(A, B, opts)


FP64_CASES = [c for c in FW.cases() if not c.startswith("faq")]


def _assert_alphas(res, case):
    """alpha sequence equal, except an endpoint tie at the terminal iteration:
    when Q ~= P the line-search gain c2 + c1 = f(P) - f(Q) is zero to rounding
    and alpha in {0, 1} may flip; both choices give a step below
    fw_tol, so iterations/convergence/permutation are unaffected (checked)."""
    ours = np.array([np.nan if h[2] is None else h[2] for h in res.iterate_history])
    ref = FW[f"{case}/hist_alpha"]
    if len(ours) == len(ref) and len(ours) > 1 and {ours[-1], ref[-1]} <= {0.0, 1.0} \
            and ours[-1] != ref[-1] and res.converged:
        ours, ref = ours[:-1], ref[:-1]
    np.testing.assert_allclose(ours, ref, atol=1e-7)


@pytest.mark.parametrize("case", FP64_CASES)
def test_fw_fp64_matches_reference(case):
    res = _run(case, "fp64")
    np.testing.assert_array_equal(res.alignment, FW[f"{case}/alignment"])
    ref_obj = float(FW[f"{case}/objective"])
    assert res.objective == pytest.approx(ref_obj, rel=1e-12, abs=1e-9)
    if float(ref_obj).is_integer():
        assert res.objective == ref_obj  # integer-exact for 0/1 graphs
    assert res.iterations == int(FW[f"{case}/iterations"])
    assert res.converged == bool(FW[f"{case}/converged"])
    objs = np.array([h[1] for h in res.iterate_history])
    # f(P_i) depends on 1000-sweep unconverged LOT iterates; log-domain vs the
    # reference's standard-domain summation order moves it at ~1e-9 relative.
    np.testing.assert_allclose(objs, FW[f"{case}/hist_obj"], rtol=1e-7, atol=1e-9)
    _assert_alphas(res, case)
    if FW.opts(case)["step_solver"] == "lot" and FW.opts(case)["n_restarts"] == 1:
        np.testing.assert_array_equal(res.diagnostics["lot_sweeps"], FW[f"{case}/lot_sweeps"])


FP32_CASES = ["c1_r0", "c1_r1", "c1_r2", "c1_r3", "c1_r4", "c2_r0", "c2_r1", "iso200_r0",
              "iso200_r1", "iso200_r2", "c4s_r0", "c5p_r0"]


@pytest.mark.parametrize("case", FP32_CASES)
def test_fw_fp32_matches_reference(case):
    res = _run(case, "fp32")
    np.testing.assert_array_equal(res.alignment, FW[f"{case}/alignment"])
    ref_obj = float(FW[f"{case}/objective"])
    if float(ref_obj).is_integer():
        assert res.objective == ref_obj
    else:
        assert res.objective == pytest.approx(ref_obj, rel=1e-6)
    objs = np.array([h[1] for h in res.iterate_history])
    n_ref = len(FW[f"{case}/hist_obj"])
    m = min(len(objs), n_ref)
    np.testing.assert_allclose(objs[:m], FW[f"{case}/hist_obj"][:m], rtol=1e-4)
    # fp32 LOTs finish in fp64 below the fp32 deviation floor, so the reference's
    # stopping rule (tol 1e-8) fires within one sweep of the reference's count
    ours, ref = res.diagnostics["lot_sweeps"], FW[f"{case}/lot_sweeps"]
    if FW.opts(case)["n_restarts"] == 1:
        assert len(ours) == len(ref)
        assert max(abs(int(a) - int(b)) for a, b in zip(ours, ref)) <= 1, (ours, ref.tolist())


def test_fw_fp32_nonconverging_trajectory_is_bounded():
    """c3s_r0 (config 3 scaled to n = 600) never converges: 30 outer iterations whose
    step sizes wander (reference alphas 0.4, 0.007, 0.3, ...), and recovery fails
    (match ratio 0.2).  Such a trajectory separates under any perturbation -- the
    reference itself moves 3 of 5000 assignments when its gradients are perturbed by
    3e-8 relative (profiles/round2_precision_study.txt) -- so fp32 mode is held to a
    bound here, not to identity: same iteration count and LOT sweeps, the first
    alphas within 1e-3, objective within 1e-3, >= 95% of the assignments equal."""
    case = "c3s_r0"
    res = _run(case, "fp32")
    assert res.iterations == int(FW[f"{case}/iterations"]) and not res.converged
    assert res.diagnostics["lot_sweeps"] == FW[f"{case}/lot_sweeps"].tolist()
    ours = np.array([h[2] for h in res.iterate_history[1:9]])
    np.testing.assert_allclose(ours, FW[f"{case}/hist_alpha"][1:9], atol=1e-3)
    assert res.objective == pytest.approx(float(FW[f"{case}/objective"]), rel=1e-3)
    assert np.mean(res.alignment == FW[f"{case}/alignment"]) >= 0.95


def test_faq_exact_lap_step():
    """FAQ (step_solver="exact_lap", the SURVEY 8f "next" row).  Its trajectory
    is discontinuous in G: the first LAP runs on the barycenter gradient, whose
    entries tie exactly among equal-degree vertices, so which tied permutation
    wins depends on last-bit rounding of G (OpenBLAS vs device).  Checked here:
    a valid FAQ run whose iterates are permutations, monotone objective, result
    objective consistent, and final objective close to the reference's."""
    case = "faq_c1_r0"
    res = _run(case, "fp64")
    p = gb.as_permutation(res.alignment)
    A, B = FW.matrix(case, "A"), FW.matrix(case, "B")
    assert res.objective == O.qap_objective_perm(A, B, p)
    objs = [o for _, o, _ in res.iterate_history]
    assert all(b >= a - 1e-9 for a, b in zip(objs, objs[1:]))
    assert res.objective == pytest.approx(float(FW[f"{case}/objective"]), rel=0.05)


FAQ = Fixture("faq_cases.npz")


@pytest.mark.parametrize("case", ["faq_w150", "faq_w150_min", "faq_w300", "faq_w700"])
def test_faq_exact_parity_on_tie_free_graphs(case):
    """FAQ with every step on the device LAP (matcher.py:191-192, lap.py:48-58)
    against the UNMODIFIED reference on weighted graphs, whose gradients never tie
    (tests/golden/make_faq_golden.py): the same permutation, objective, iteration
    count, convergence flag and alpha sequence.  n = 150 runs the scipy-order
    augmenting-path solver, n >= 256 the auction + certified repair."""
    import hashlib

    from paper_2111_05366_b200 import graphs
    rep, n, smax, mi = (int(x) for x in FAQ[f"{case}/spec"])
    A, B, _ = graphs.config_pair(4, rep, n=n)
    for M, tag in ((A, "A"), (B, "B")):
        assert hashlib.sha256(np.ascontiguousarray(M).tobytes()).hexdigest() == str(FAQ[f"{case}/sha_{tag}"])
    res = gb.frank_wolfe_match(A, B, gb.MatchOptions(
        step_solver="exact_lap", objective_sense="maximize" if smax else "minimize", max_iters=mi,
        precision="fp64"))
    np.testing.assert_array_equal(res.alignment, FAQ[f"{case}/alignment"])
    assert res.objective == pytest.approx(float(FAQ[f"{case}/objective"]), rel=1e-12)
    assert res.iterations == int(FAQ[f"{case}/iterations"])
    assert res.converged == bool(FAQ[f"{case}/converged"])
    ours = np.array([np.nan if h[2] is None else h[2] for h in res.iterate_history])
    np.testing.assert_allclose(ours, FAQ[f"{case}/hist_alpha"], atol=1e-9)
    np.testing.assert_allclose([h[1] for h in res.iterate_history], FAQ[f"{case}/hist_obj"], rtol=1e-10)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", list(UNIT["lot/names"]))
def test_lot_matches_reference(name, precision):
    M = UNIT[f"lot/{name}/M"]
    lam, ms, tol = UNIT[f"lot/{name}/params"]
    if precision == "fp32" and lam > 1000:
        pytest.skip("lam=5e4 exponents exceed fp32 resolution of the unit-range cost")
    res = gb.lot(M, str(UNIT[f"lot/{name}/sense"]), gb.SinkhornParams(lam=lam, max_sweeps=int(ms), tol=tol),
                 precision=precision)
    Qref = UNIT[f"lot/{name}/Q"]
    if precision == "fp64":
        assert res.sweeps == int(UNIT[f"lot/{name}/sweeps"])
        assert res.converged == bool(UNIT[f"lot/{name}/converged"])
        assert res.deviation == pytest.approx(float(UNIT[f"lot/{name}/dev"]), rel=1e-3, abs=1e-12)
    np.testing.assert_allclose(res.matrix, Qref, atol=TOL_Q[precision])


@pytest.mark.parametrize("name", list(UNIT["sk/names"]))
def test_sinkhorn_knopp_matches_reference(name):
    res = gb.sinkhorn_knopp(UNIT[f"sk/{name}/K"])
    assert res.sweeps == int(UNIT[f"sk/{name}/sweeps"])
    np.testing.assert_allclose(res.matrix, UNIT[f"sk/{name}/Q"], atol=1e-12)
    if res.sweeps == 0:
        np.testing.assert_array_equal(res.matrix, UNIT[f"sk/{name}/K"])


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", list(UNIT["lap/names"]))
def test_lap_matches_scipy(name, precision):
    M = UNIT[f"lap/{name}/M"]
    if precision == "fp32" and not np.array_equal(M.astype(np.float32), M):
        M32 = M.astype(np.float32).astype(np.float64)
        for sense in ("minimize", "maximize"):
            sol = gb.solve_lap(M32, sense, precision="fp32")
            p, _ = O.lap(M32, sense)
            np.testing.assert_array_equal(sol.assignment, p)
        return
    for sense in ("minimize", "maximize"):
        sol = gb.solve_lap(M, sense, precision=precision)
        np.testing.assert_array_equal(sol.assignment, UNIT[f"lap/{name}/{sense}/assignment"])
        assert sol.objective == float(UNIT[f"lap/{name}/{sense}/objective"])


def test_lap_random_and_tie_heavy_vs_scipy():
    rng = np.random.default_rng(11)
    for t in range(60):
        n = int(rng.integers(1, 90))
        kind = t % 3
        M = rng.random((n, n)) if kind == 0 else rng.integers(0, 3 if kind == 1 else 2, size=(n, n)).astype(float)
        for sense in ("minimize", "maximize"):
            p, v = O.lap(M, sense)
            sol = gb.solve_lap(M, sense)
            np.testing.assert_array_equal(sol.assignment, p)
            assert sol.objective == v


def test_lap_known_answers():
    T = O.TIE_MATRIX
    sol = gb.solve_lap(T, "minimize")
    assert sol.objective == 172.0 and sol.assignment.tolist() in ([0, 1, 3, 2], [0, 3, 1, 2])
    assert gb.solve_lap(T, "maximize").objective == 183.0
    assert gb.solve_lap(np.diag([10.0, 10.0]), "maximize").assignment.tolist() == [0, 1]
    with pytest.raises(ValueError, match="finite"):
        gb.solve_lap(np.array([[1.0, np.inf], [0.0, 1.0]]))
    with pytest.raises(ValueError, match="sense"):
        gb.solve_lap(np.eye(2), "best")


def test_lap_large_instance_fast():
    import time
    rng = np.random.default_rng(4)
    M = rng.random((2000, 2000))
    t0 = time.perf_counter()
    sol = gb.solve_lap(M, "minimize")
    assert time.perf_counter() - t0 < 30.0
    p, v = O.lap(M, "minimize")
    np.testing.assert_array_equal(sol.assignment, p)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_gradient_linesearch_objective(precision):
    # fp32 mode runs the products on tcgen05 with bf16-split operands: error is
    # relative to the gradient's scale (max|G|), ~1e-6 measured.
    tol = 1e-12 if precision == "fp64" else 2e-6
    for k in range(3):
        A, B, P, Q = (UNIT[f"grad/{k}/{x}"] for x in "ABPQ")
        G = UNIT[f"grad/{k}/G"]
        err = np.abs(gb.gradient(A, B, P, precision=precision) - G).max() / np.abs(G).max()
        assert err < tol, err
        a_max = gb.exact_line_search(A, B, P, Q, "maximize", precision=precision)
        a_min = gb.exact_line_search(A, B, P, Q, "minimize", precision=precision)
        atol = 1e-4 if precision == "fp32" else 1e-10  # interior alpha = -c1/(2 c2) from fp32 G
        assert a_max == pytest.approx(float(UNIT[f"grad/{k}/alpha_max"]), abs=atol)
        assert a_min == pytest.approx(float(UNIT[f"grad/{k}/alpha_min"]), abs=atol)
    A, B, p = UNIT["grad/2/A"], UNIT["grad/2/B"], UNIT["grad/2/perm"]
    assert gb.qap_objective(A, B, p) == pytest.approx(float(UNIT["grad/2/qap_perm"]), rel=1e-13)


def test_gradient_finite_differences():
    rng = np.random.default_rng(1)
    A, B, P = rng.random((5, 5)), rng.random((5, 5)), rng.random((5, 5))
    G = gb.gradient(A, B, P)
    h = 1e-5
    for i in range(5):
        for j in range(5):
            Pp = P.copy(); Pp[i, j] += h
            Pm = P.copy(); Pm[i, j] -= h
            fd = (gb.qap_objective(A, B, Pp) - gb.qap_objective(A, B, Pm)) / (2 * h)
            assert G[i, j] == pytest.approx(fd, abs=1e-4)


def test_engine_known_answers_and_determinism():
    res = gb.frank_wolfe_match(np.array([[3.0]]), np.array([[2.0]]))
    assert res.alignment.tolist() == [0] and res.objective == pytest.approx(6.0)
    assert gb.frank_wolfe_match(np.zeros((4, 4)), np.zeros((4, 4)),
                                gb.MatchOptions(step_solver="lot")).objective == 0.0
    rng = np.random.default_rng(8)
    A = (rng.random((15, 15)) < 0.3).astype(float)
    B = (rng.random((15, 15)) < 0.3).astype(float)
    for precision in ("fp64", "fp32"):
        opts = gb.MatchOptions(step_solver="lot", init="randomized_blend", n_restarts=3,
                               shuffle_input=True, rng_seed=99, precision=precision)
        r1 = gb.frank_wolfe_match(A, B, opts)
        r2 = gb.frank_wolfe_match(A, B, opts)
        np.testing.assert_array_equal(r1.alignment, r2.alignment)
        assert r1.objective == r2.objective
        assert r1.iterate_history == r2.iterate_history  # bit-identical reruns


def test_monotone_objective_and_sandwich():
    import itertools
    rng = np.random.default_rng(6)
    for _ in range(5):
        A = (rng.random((12, 12)) < 0.4).astype(float)
        B = (rng.random((12, 12)) < 0.4).astype(float)
        res = gb.frank_wolfe_match(A, B, gb.MatchOptions(step_solver="lot"))
        objs = [o for _, o, _ in res.iterate_history]
        assert all(b >= a - 1e-9 for a, b in zip(objs, objs[1:]))
    for _ in range(3):
        A, B = rng.random((5, 5)), rng.random((5, 5))
        vals = [gb.qap_objective(A, B, np.array(p)) for p in itertools.permutations(range(5))]
        res = gb.frank_wolfe_match(A, B, gb.MatchOptions(step_solver="lot"))
        assert min(vals) - 1e-9 <= res.objective <= max(vals) + 1e-9


@pytest.mark.parametrize("m", [1, 7, 39])
def test_seeded_device_L_matches_oracle(m):
    """The seed term L = A21 B21^T + A12^T B12 (matcher.py:267) formed on the device
    (goat_fw_core_seeded) on weighted directed graphs: the oracle's seeded run,
    including the m = n - 1 case (a 1 x 1 free block)."""
    n = 40
    rng = np.random.default_rng(100 + m)
    A = (rng.random((n, n)) < 0.3) * rng.lognormal(0, 1, (n, n))
    B = (rng.random((n, n)) < 0.3) * rng.lognormal(0, 1, (n, n))
    np.fill_diagonal(A, 0)
    np.fill_diagonal(B, 0)
    perm = rng.permutation(n)
    seeds = np.stack([np.arange(m), perm[:m]], axis=1)
    opts = gb.MatchOptions(step_solver="lot", precision="fp64", shuffle_input=True, max_iters=12)
    res = gb.seeded_match(A, B, gb.SeedSet(seeds), opts)
    align, obj, iters, hist, conv = O.run_seeded(A, B, seeds, shuffle_input=True, max_iters=12)
    np.testing.assert_array_equal(res.alignment, align)
    assert res.objective == pytest.approx(obj, rel=1e-12)
    assert res.iterations == iters and res.converged == conv
    np.testing.assert_allclose([h[1] for h in res.iterate_history], [h[1] for h in hist], rtol=1e-9)


@pytest.mark.parametrize("which", ["A", "B"])
@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan])
def test_nonfinite_inputs_raise_valueerror(which, bad):
    """core.py:23-26: non-finite entries are a ValueError (checked on the device
    during the upload for unseeded dense runs)."""
    rng = np.random.default_rng(0)
    A = (rng.random((30, 30)) < 0.3).astype(float)
    B = A.copy()
    (A if which == "A" else B)[3, 7] = bad
    with pytest.raises(ValueError, match=f"{which} contains non-finite entries"):
        gb.frank_wolfe_match(A, B, gb.MatchOptions(step_solver="lot"))


def test_bit_identical_reruns_at_c2():
    """Identical inputs and options give a bit-identical MatchResult including the
    iterate history (test_matcher.py:160-170), at config 2's size and in both
    precisions (fixed reduction trees, no order-varying atomics on the value path)."""
    case = "c2_r0"
    for precision in ("fp64", "fp32"):
        a, b = _run(case, precision), _run(case, precision)
        np.testing.assert_array_equal(a.alignment, b.alignment)
        assert a.objective == b.objective and a.iterations == b.iterations
        assert a.iterate_history == b.iterate_history
        assert a.diagnostics["lot_sweeps"] == b.diagnostics["lot_sweeps"]
        assert a.diagnostics["lot_deviation"] == b.diagnostics["lot_deviation"]
