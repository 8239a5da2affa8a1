"""Host-side pieces of the experiment CLI and the text formats (no GPU): parser
defaults mirror the reference harness (cli.py:450-521), `shuffle` round-trips, and
pass_to_ranks / text formats keep the reference's contract (core.py:166-229)."""
import numpy as np
import pytest

import paper_2111_05366_b200 as gb
from paper_2111_05366_b200 import cli


def test_parser_defaults_follow_reference():
    a = cli.build_parser().parse_args(["rho-sbm"])
    assert (a.n, a.replicates, a.solvers, a.max_iters, a.fw_tol, a.lam, a.seed, a.out) == \
        (150, 25, ["faq", "goat"], 30, 1e-2, 100.0, 0, "rho_sbm.csv")
    assert a.rho_grid == [0.5, 0.6, 0.7, 0.8, 0.9, 1.0]
    a = cli.build_parser().parse_args(["seeded"])
    assert (a.n, a.seed_grid, a.rho_grid, a.replicates) == (90, [0, 5, 10, 20], [0.9], 20)
    a = cli.build_parser().parse_args(["er-scaling", "--n-grid", "30,40"])
    assert a.n_grid == [30, 40] and a.rho == 1.0
    a = cli.build_parser().parse_args(["lap-vs-lot"])
    assert (a.n_grid, a.cost_low, a.cost_high) == ([250, 500, 1000], 100.0, 150.0)


def test_child_seed_is_stable_63_bit():
    s = cli.child_seed(7, 900, 3)
    assert s == cli.child_seed(7, 900, 3) and 0 <= s < 2 ** 63
    assert s != cli.child_seed(7, 900, 4)


def test_shuffle_command_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    A = (rng.random((9, 9)) < 0.4).astype(float)
    src = tmp_path / "a.txt"
    src.write_text(gb.format_matrix_text(A))
    out = tmp_path / "s.txt"
    assert cli.main(["shuffle", str(src), "--seed", "9", "--out", str(out)]) == 0
    Bs = gb.parse_matrix_text(out.read_text())
    truth = gb.parse_permutation_text((tmp_path / "s.txt.truth.txt").read_text())
    np.testing.assert_array_equal(Bs[np.ix_(truth, truth)], A)


def test_seeded_rejects_seed_count_at_n(tmp_path):
    with pytest.raises(SystemExit):
        cli.main(["seeded", "--n", "10", "--seed-grid", "10", "--out", str(tmp_path / "x.csv")])


def test_grouped_mean():
    header = ["k", "v"]
    rows = [["a", 1.0], ["b", 4.0], ["a", 3.0]]
    out = cli.grouped_mean(rows, header, ["k"], "v")
    assert out[0][:3] == ["a", 2, 2.0] and out[0][3] == pytest.approx(1.0)
    assert out[1] == ["b", 1, 4.0, 0.0]


def test_pass_to_ranks_contract():
    W = np.array([[0.0, 5.0, 2.0], [5.0, 0.0, 0.0], [2.0, 0.0, 9.0]])
    R = gb.pass_to_ranks(W)
    # 5 nonzeros: ranks 2:1.5,1.5  5:3.5,3.5  9:5 -> / 6
    np.testing.assert_allclose(R, np.array([[0, 3.5, 1.5], [3.5, 0, 0], [1.5, 0, 5]]) / 6)
    np.testing.assert_array_equal(R, R.T)
    np.testing.assert_array_equal(gb.pass_to_ranks(W ** 3), R)  # monotone reweighting
    with pytest.raises(ValueError):
        gb.pass_to_ranks(-W)
    assert not gb.pass_to_ranks(np.zeros((3, 3))).any()


def test_text_formats():
    M = np.array([[0.1, 2.0], [3.5, 1e-9]])
    assert np.array_equal(gb.parse_matrix_text(gb.format_matrix_text(M)), M)
    for bad in ("", "x 1", "0", "2 1 2 3", "1 z"):
        with pytest.raises(ValueError):
            gb.parse_matrix_text(bad)
    assert gb.format_permutation_text([2, 0, 1]) == "2 0 1\n"
    np.testing.assert_array_equal(gb.parse_permutation_text("2 0 1\n"), [2, 0, 1])
    with pytest.raises(ValueError):
        gb.parse_permutation_text("0 0 1")
    with pytest.raises(ValueError):
        gb.parse_permutation_text("0 a")


def test_sbm_spec_validation():
    with pytest.raises(ValueError):
        gb.SbmSpec((2, 0), np.eye(2) * 0.5, 0.5)
    with pytest.raises(ValueError):
        gb.SbmSpec((2, 2), np.array([[0.1, 0.2], [0.3, 0.1]]), 0.5)
    with pytest.raises(ValueError):
        gb.SbmSpec((2, 2), np.eye(2) * 0.5, 1.5)
    spec = gb.SbmSpec((3, 4), [[0.5, 0.1], [0.1, 0.5]], 1.0)
    A, B = gb.sample_sbm_pair(spec, np.random.default_rng(0))
    assert spec.n == 7 and np.array_equal(A, B) and np.array_equal(A, A.T) and not A.diagonal().any()
