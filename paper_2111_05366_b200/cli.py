"""Experiment CLI over the B200 backend.

Same subcommands, flags, CSV columns, sidecar files and seeding rules as the
reference harness (cli.py:143-421), so a row produced here is comparable, column
for column, with a row the reference writes for the same ``--seed``:

  lap-vs-lot   exact LAP vs LOT on uniform cost matrices        (cli.py:143-171)
  rho-sbm      match ratio vs edge correlation on SBM pairs      (cli.py:174-218)
  seeded       match ratio vs number of seeds                    (cli.py:221-270)
  er-scaling   run time and accuracy vs n on ER pairs            (cli.py:273-310)
  match        align two matrix text files                       (cli.py:370-410)
  shuffle      write a relabelled copy of a matrix text file     (cli.py:413-421)

Every solve runs in libgoat.so on one GPU (``--device``, ``--precision``); the
replicates of an experiment are independent, so ``--workers`` is accepted for
compatibility but the grid runs serially on the device -- one process per GPU is
the parallel unit here (run disjoint ``--rho-grid`` / ``--n-grid`` slices per GPU).
The QAPLIB subcommand is not provided: QAPLIB ingestion is outside the GOAT path
(DESIGN.md §7).

    python -m paper_2111_05366_b200.cli er-scaling --n-grid 100,200 --replicates 2
"""

from __future__ import annotations

import argparse
import csv
import json
import math
import sys
import time
from dataclasses import dataclass
from pathlib import Path
from typing import Callable

import numpy as np

from . import __version__
from .engine import frank_wolfe_match, seeded_match
from .formats import (format_matrix_text, format_permutation_text, parse_matrix_text,
                      pass_to_ranks)
from .graphs import SbmSpec, sample_sbm_pair
from .graphs import shuffle as _relabel
from .matrices import as_square_matrix, edge_disagreements, match_ratio
from .ops import lot, solve_lap
from .records import MatchOptions, SeedSet, SinkhornParams

SCHEMA_VERSION = 1
STEP_OF = {"faq": "exact_lap", "goat": "lot"}
DEFAULT_ACCURACY_BLOCKS = [[0.2, 0.01, 0.01], [0.01, 0.1, 0.01], [0.01, 0.01, 0.2]]
DEFAULT_SEEDED_BLOCKS = [[0.7, 0.3, 0.4], [0.3, 0.7, 0.3], [0.4, 0.3, 0.7]]


# ----------------------------------------------------------------- plumbing
def child_seed(master: int, *tags: int) -> int:
    """63-bit per-task seed from SeedSequence([master, *tags]) (cli.py:58-61)."""
    state = np.random.SeedSequence([int(master)] + [int(t) for t in tags]).generate_state(1, dtype=np.uint64)
    return int(state[0] >> 1)


def cell(x) -> str:
    return repr(x) if isinstance(x, float) else str(x)


def write_table(path: Path, header, rows) -> None:
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows([[cell(v) for v in r] for r in rows])


def write_sidecar(out: Path, command: str, args) -> None:
    cfg = {k: v for k, v in vars(args).items() if k != "run"}
    cfg["out"] = str(out)
    doc = {"schema_version": SCHEMA_VERSION, "otmatch_version": __version__, "command": command, "config": cfg}
    Path(str(out) + ".meta.json").write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def grouped_mean(rows, header, keys, value):
    """[(key..., count, mean, standard error)] in first-seen key order (cli.py:104-119)."""
    ki = [header.index(k) for k in keys]
    vi = header.index(value)
    seen: dict = {}
    for r in rows:
        seen.setdefault(tuple(r[i] for i in ki), []).append(float(r[vi]))
    out = []
    for key, vals in seen.items():
        v = np.asarray(vals)
        se = float(v.std(ddof=1) / math.sqrt(v.size)) if v.size > 1 else 0.0
        out.append([*key, v.size, float(v.mean()), se])
    return out


def solver_options(solver: str, args, seed: int = 0) -> MatchOptions:
    return MatchOptions(step_solver=STEP_OF[solver], sinkhorn=SinkhornParams(lam=args.lam), init="barycenter",
                        max_iters=args.max_iters, fw_tol=args.fw_tol, n_restarts=1, shuffle_input=False,
                        rng_seed=seed, objective_sense="maximize", precision=args.precision, device=args.device)


def balanced_blocks(n: int, block_probs, rho: float) -> SbmSpec:
    k = len(block_probs)
    sizes = tuple(n // k + (1 if b < n % k else 0) for b in range(k))
    return SbmSpec(sizes, np.asarray(block_probs, dtype=float), rho)


def timed(fn: Callable, *a):
    t0 = time.perf_counter()
    r = fn(*a)
    return r, time.perf_counter() - t0


# ----------------------------------------------------------------- experiments
@dataclass
class Experiment:
    """One aggregate subcommand: a grid of tasks, each yielding CSV rows."""

    name: str
    header: list
    grid: Callable      # args -> iterable of task tuples
    task: Callable      # (args, *task) -> list of rows
    summary: tuple | None = None  # (key columns, value column, summary header)

    def run(self, args) -> int:
        rows = []
        for t in self.grid(args):
            rows.extend(self.task(args, *t))
        out = Path(args.out)
        write_table(out, self.header, rows)
        if self.summary:
            keys, value, shead = self.summary
            write_table(out.with_name(out.stem + ".summary.csv"), shead, grouped_mean(rows, self.header, keys, value))
        write_sidecar(out, self.name, args)
        return 0


def lap_vs_lot_task(args, n, rep):
    rng = np.random.default_rng([args.seed, n, rep])
    M = rng.uniform(args.cost_low, args.cost_high, size=(n, n))
    sol, t_lap = timed(lambda: solve_lap(M, "minimize", device=args.device, precision=args.precision))
    res, t_lot = timed(lambda: lot(M, "minimize", SinkhornParams(lam=args.lam), device=args.device,
                                   precision=args.precision))
    ofv = float((res.matrix * M).sum())
    return [[n, rep, t_lap, t_lot, sol.objective, ofv, (sol.objective - ofv) / sol.objective, res.sweeps,
             res.converged]]


def sbm_pair(args, rho, rep, n, block_probs):
    rng = np.random.default_rng([args.seed, round(rho * 1000), rep])
    A, B = sample_sbm_pair(balanced_blocks(n, block_probs, rho), rng)
    Bs, truth = _relabel(as_square_matrix(B, "B"), rng)
    return A, Bs, truth


def rho_sbm_task(args, rho, rep):
    A, Bs, truth = sbm_pair(args, rho, rep, args.n, json.loads(args.block_probs))
    seed = child_seed(args.seed, round(rho * 1000), rep)
    rows = []
    for s in args.solvers:
        res, dt = timed(frank_wolfe_match, A, Bs, solver_options(s, args, seed))
        rows.append([rho, rep, s, match_ratio(res.alignment, truth), res.objective, res.iterations, res.converged, dt])
    return rows


def seeded_task(args, rho, m, rep):
    n = args.n
    A, Bs, truth = sbm_pair(args, rho, rep, n, json.loads(args.block_probs))  # shared across m
    pick = np.random.default_rng([args.seed, round(rho * 1000), rep, m])
    g1 = np.sort(pick.choice(n, size=m, replace=False)) if m else np.empty(0, dtype=int)
    pairs = np.stack([g1, truth[g1]], axis=1) if m else np.empty((0, 2), dtype=int)
    free = np.setdiff1d(np.arange(n), g1)
    seed = child_seed(args.seed, round(rho * 1000), rep)  # no m: the m = 0 rows equal rho-sbm's
    rows = []
    for s in args.solvers:
        res, dt = timed(seeded_match, A, Bs, SeedSet(pairs), solver_options(s, args, seed))
        free_ratio = float(np.mean(res.alignment[free] == truth[free])) if free.size else 1.0
        rows.append([rho, m, rep, s, free_ratio, match_ratio(res.alignment, truth), res.objective, res.iterations, dt])
    return rows


def er_scaling_task(args, n, rep):
    rng = np.random.default_rng([args.seed, n, rep])
    A, B = sample_sbm_pair(SbmSpec((n,), np.array([[math.log(n) / n]]), args.rho), rng)
    Bs, truth = _relabel(as_square_matrix(B, "B"), rng)
    seed = child_seed(args.seed, n, rep)
    rows = []
    for s in args.solvers:
        res, dt = timed(frank_wolfe_match, A, Bs, solver_options(s, args, seed))
        rows.append([n, rep, s, dt, match_ratio(res.alignment, truth), res.objective, res.iterations])
    return rows


def seeded_grid(args):
    for m in args.seed_grid:
        if m >= args.n:
            raise SystemExit(f"seed count {m} must be less than n = {args.n}")
    return [(rho, m, rep) for rho in args.rho_grid for m in args.seed_grid for rep in range(args.replicates)]


EXPERIMENTS = {
    "lap-vs-lot": Experiment(
        "lap-vs-lot",
        ["n", "replicate", "t_lap", "t_lot", "ofv_lap", "ofv_lot", "rel_gap", "lot_sweeps", "lot_converged"],
        lambda a: [(n, rep) for n in a.n_grid for rep in range(a.replicates)], lap_vs_lot_task),
    "rho-sbm": Experiment(
        "rho-sbm", ["rho", "replicate", "solver", "match_ratio", "objective", "iterations", "converged", "t_solve"],
        lambda a: [(rho, rep) for rho in a.rho_grid for rep in range(a.replicates)], rho_sbm_task,
        (["rho", "solver"], "match_ratio", ["rho", "solver", "replicates", "mean_match_ratio", "se_match_ratio"])),
    "seeded": Experiment(
        "seeded", ["rho", "m", "replicate", "solver", "match_ratio_nonseed", "match_ratio_all", "objective",
                   "iterations", "t_solve"],
        seeded_grid, seeded_task,
        (["rho", "m", "solver"], "match_ratio_nonseed",
         ["rho", "m", "solver", "replicates", "mean_match_ratio_nonseed", "se_match_ratio_nonseed"])),
    "er-scaling": Experiment(
        "er-scaling", ["n", "replicate", "solver", "t_solve", "match_ratio", "objective", "iterations"],
        lambda a: [(n, rep) for n in a.n_grid for rep in range(a.replicates)], er_scaling_task,
        (["n", "solver"], "match_ratio", ["n", "solver", "replicates", "mean_match_ratio", "se_match_ratio"])),
}


# ----------------------------------------------------------------- match / shuffle
def run_match(args) -> int:
    A = parse_matrix_text(Path(args.file_a).read_text())
    B = parse_matrix_text(Path(args.file_b).read_text())
    if A.shape != B.shape:
        raise SystemExit(f"order mismatch: {A.shape[0]} vs {B.shape[0]}")
    if args.ptr:
        A, B = pass_to_ranks(A), pass_to_ranks(B)
    opts = MatchOptions(step_solver=STEP_OF[args.solver], sinkhorn=SinkhornParams(lam=args.lam),
                        init="randomized_blend" if args.n_restarts > 1 else args.init, max_iters=args.max_iters,
                        fw_tol=args.fw_tol, n_restarts=args.n_restarts, shuffle_input=args.shuffle,
                        rng_seed=args.seed, objective_sense="maximize", precision=args.precision,
                        device=args.device)
    res = frank_wolfe_match(A, B, opts)
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(format_permutation_text(res.alignment))
    line = json.dumps({
        "objective": res.objective, "edge_disagreements": edge_disagreements(A, B, res.alignment),
        "iterations": res.iterations, "converged": res.converged, "wall_time": res.wall_time,
        "config": {"solver": args.solver, "lam": args.lam, "max_iters": args.max_iters, "fw_tol": args.fw_tol,
                   "n_restarts": args.n_restarts, "shuffle": args.shuffle, "ptr": args.ptr, "seed": args.seed,
                   "init": args.init}}, sort_keys=True)
    with open(str(out) + ".summary.jsonl", "a") as fh:
        fh.write(line + "\n")
    print(line)
    return 0


def run_shuffle(args) -> int:
    B = parse_matrix_text(Path(args.file).read_text())
    Bs, truth = _relabel(B, np.random.default_rng(args.seed))
    out = Path(args.out)
    out.parent.mkdir(parents=True, exist_ok=True)
    out.write_text(format_matrix_text(Bs))
    Path(str(out) + ".truth.txt").write_text(format_permutation_text(truth))
    return 0


# ----------------------------------------------------------------- parser
def ints(text):
    return [int(t) for t in text.split(",") if t]


def floats(text):
    return [float(t) for t in text.split(",") if t]


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="otmatch", description=__doc__,
                                 formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p, out, solvers=True):
        if solvers:
            p.add_argument("--solvers", type=lambda s: s.split(","), default=["faq", "goat"])
            p.add_argument("--max-iters", type=int, default=30)
            p.add_argument("--fw-tol", type=float, default=1e-2)
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--out", default=out)
        p.add_argument("--workers", type=int, default=1, help="accepted for compatibility; the grid runs on one GPU")
        p.add_argument("--lam", type=float, default=100.0)
        p.add_argument("--device", type=int, default=0, help="CUDA ordinal")
        p.add_argument("--precision", choices=["fp64", "fp32"], default="fp64")

    p = sub.add_parser("lap-vs-lot")
    p.add_argument("--n-grid", type=ints, default=[250, 500, 1000])
    p.add_argument("--replicates", type=int, default=20)
    p.add_argument("--cost-low", type=float, default=100.0)
    p.add_argument("--cost-high", type=float, default=150.0)
    common(p, "lap_vs_lot.csv", solvers=False)
    p.set_defaults(run=EXPERIMENTS["lap-vs-lot"].run)

    p = sub.add_parser("rho-sbm")
    p.add_argument("--n", type=int, default=150)
    p.add_argument("--block-probs", default=json.dumps(DEFAULT_ACCURACY_BLOCKS))
    p.add_argument("--rho-grid", type=floats, default=[0.5, 0.6, 0.7, 0.8, 0.9, 1.0])
    p.add_argument("--replicates", type=int, default=25)
    common(p, "rho_sbm.csv")
    p.set_defaults(run=EXPERIMENTS["rho-sbm"].run)

    p = sub.add_parser("seeded")
    p.add_argument("--n", type=int, default=90)
    p.add_argument("--block-probs", default=json.dumps(DEFAULT_SEEDED_BLOCKS))
    p.add_argument("--rho-grid", type=floats, default=[0.9])
    p.add_argument("--seed-grid", type=ints, default=[0, 5, 10, 20])
    p.add_argument("--replicates", type=int, default=20)
    common(p, "seeded.csv")
    p.set_defaults(run=EXPERIMENTS["seeded"].run)

    p = sub.add_parser("er-scaling")
    p.add_argument("--n-grid", type=ints, default=[100, 200, 400])
    p.add_argument("--replicates", type=int, default=10)
    p.add_argument("--rho", type=float, default=1.0)
    common(p, "er_scaling.csv")
    p.set_defaults(run=EXPERIMENTS["er-scaling"].run)

    p = sub.add_parser("match")
    p.add_argument("file_a")
    p.add_argument("file_b")
    p.add_argument("--solver", choices=["faq", "goat"], default="goat")
    p.add_argument("--init", choices=["barycenter", "randomized_blend"], default="barycenter")
    p.add_argument("--ptr", action="store_true")
    p.add_argument("--shuffle", action="store_true")
    p.add_argument("--n-restarts", type=int, default=1)
    p.add_argument("--max-iters", type=int, default=30)
    p.add_argument("--fw-tol", type=float, default=1e-2)
    common(p, "alignment.txt", solvers=False)
    p.set_defaults(run=run_match)

    p = sub.add_parser("shuffle")
    p.add_argument("file")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default="shuffled.txt")
    p.set_defaults(run=run_shuffle)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.run(args)
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
