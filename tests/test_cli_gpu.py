"""The experiment CLI over the GPU backend (reference harness: cli.py:143-421): CSV
schema, sidecars, determinism of the non-timing columns, and `shuffle` + `match`
recovering a planted permutation."""
import csv
import json

import numpy as np
import pytest

import paper_2111_05366_b200 as gb
from paper_2111_05366_b200 import cli

pytestmark = pytest.mark.gpu


def _rows(path):
    with open(path, newline="") as fh:
        r = list(csv.reader(fh))
    return r[0], r[1:]


def test_er_scaling_schema_and_determinism(tmp_path):
    outs = []
    for k in range(2):
        out = tmp_path / f"er{k}.csv"
        assert cli.main(["er-scaling", "--n-grid", "30,40", "--replicates", "2", "--seed", "3", "--out", str(out)]) == 0
        outs.append(_rows(out))
    header, rows = outs[0]
    assert header == ["n", "replicate", "solver", "t_solve", "match_ratio", "objective", "iterations"]
    assert len(rows) == 2 * 2 * 2  # n-grid x replicates x {faq, goat}
    t = header.index("t_solve")
    strip = lambda rs: [[c for i, c in enumerate(r) if i != t] for r in rs]
    assert strip(rows) == strip(outs[1][1])  # every non-timing column reproduces
    sh, srows = _rows(tmp_path / "er0.summary.csv")
    assert sh == ["n", "solver", "replicates", "mean_match_ratio", "se_match_ratio"] and len(srows) == 4
    meta = json.loads((tmp_path / "er0.csv.meta.json").read_text())
    assert meta["command"] == "er-scaling" and meta["config"]["seed"] == 3 and meta["schema_version"] == 1


def test_seeded_with_zero_seeds_equals_rho_sbm(tmp_path):
    common = ["--n", "30", "--rho-grid", "0.9", "--replicates", "2", "--seed", "5", "--solvers", "goat",
              "--block-probs", "[[0.7, 0.3], [0.3, 0.7]]"]  # the two subcommands default to different blocks
    assert cli.main(["rho-sbm", *common, "--out", str(tmp_path / "r.csv")]) == 0
    assert cli.main(["seeded", *common, "--seed-grid", "0", "--out", str(tmp_path / "s.csv")]) == 0
    hr, rr = _rows(tmp_path / "r.csv")
    hs, rs = _rows(tmp_path / "s.csv")
    for a, b in zip(rr, rs):
        assert a[hr.index("match_ratio")] == b[hs.index("match_ratio_all")]
        assert a[hr.index("objective")] == b[hs.index("objective")]


def test_shuffle_then_match_recovers(tmp_path, capsys):
    rng = np.random.default_rng(11)
    A, _ = gb.sample_er_pair(40, 0.3, 1.0, rng)
    a_path, s_path, out = tmp_path / "a.txt", tmp_path / "s.txt", tmp_path / "p.txt"
    a_path.write_text(gb.format_matrix_text(A))
    assert cli.main(["shuffle", str(a_path), "--seed", "9", "--out", str(s_path)]) == 0
    truth = gb.parse_permutation_text((tmp_path / "s.txt.truth.txt").read_text())
    assert cli.main(["match", str(a_path), str(s_path), "--solver", "goat", "--out", str(out)]) == 0
    p = gb.parse_permutation_text(out.read_text())
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert gb.match_ratio(p, truth) == 1.0 and summary["edge_disagreements"] == 0
    assert summary["objective"] == gb.qap_objective(A, gb.parse_matrix_text(s_path.read_text()), p)


def test_lap_vs_lot_rows(tmp_path):
    out = tmp_path / "l.csv"
    assert cli.main(["lap-vs-lot", "--n-grid", "60", "--replicates", "2", "--out", str(out)]) == 0
    header, rows = _rows(out)
    assert header == ["n", "replicate", "t_lap", "t_lot", "ofv_lap", "ofv_lot", "rel_gap", "lot_sweeps", "lot_converged"]
    assert len(rows) == 2 and all(abs(float(r[header.index("rel_gap")])) < 0.01 for r in rows)
