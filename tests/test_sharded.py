"""Row-sharded driver (paper_2111_05366_b200/sharded.py) across world_size 1-3 on CPU.

Each rank is a gloo process running the real driver -- row blocks, all-gathers,
rank-order merges of the Sinkhorn column sums, the shared stopping decision, the
scalar allreduces and the rank-0 LAP + broadcast -- with the numpy stand-in of
the goat_shard_* kernels (tests/shard_np.py).  The sharded run must reproduce the
oracle's GOAT run (oracle/goat_oracle.py fw_core, matcher.py:177-212): the same
permutation, the same per-iteration Sinkhorn sweep counts and step sizes.
"""
import multiprocessing as mp
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist

from oracle import goat_oracle as O
from paper_2111_05366_b200.sharded import Comm, ShardLayout, sharded_fw_core


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, A, B, kw, q, bkw):
    try:
        from shard_np import NumpyShardBackend
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        comm = Comm()
        lay = ShardLayout(A.shape[0], world, rank)
        be = NumpyShardBackend(lay, **bkw)
        sym = np.array_equal(A, A.T) and np.array_equal(B, B.T)
        r0, m = lay.r0, lay.m
        A_rows = be.upload(A[r0:r0 + m], lay.m_pad)
        AT_rows = None if sym else be.upload(A.T[r0:r0 + m], lay.m_pad)
        res = sharded_fw_core(be, comm, A_rows, AT_rows, be.upload(B), **kw)
        if rank == 0:
            q.put(("ok", res.assignment.tolist(), res.hist_obj, res.hist_alpha, res.lot_sweeps,
                   res.iterations, res.converged, res.collectives))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put(("err", rank, repr(e)))


def run_sharded(A, B, world, backend_kw=None, **kw):
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, A, B, kw, q, backend_kw or {})) for r in range(world)]
    for p in procs:
        p.start()
    try:
        out = q.get(timeout=240)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    assert out[0] == "ok", out
    keys = ("assignment", "hist_obj", "hist_alpha", "lot_sweeps", "iterations", "converged", "collectives")
    return dict(zip(keys, out[1:]))


def _er_pair(n, p, rho, directed, seed):
    rng = np.random.default_rng(seed)
    A = (rng.random((n, n)) < p).astype(float)
    np.fill_diagonal(A, 0)
    if not directed:
        A = np.triu(A, 1)
        A = A + A.T
    keep = rng.random((n, n)) < rho + (1 - rho) * p
    flip = rng.random((n, n)) < p * (1 - rho)
    B = np.where(A > 0, keep, flip).astype(float)
    np.fill_diagonal(B, 0)
    if not directed:
        B = np.triu(B, 1)
        B = B + B.T
    perm = rng.permutation(n)
    return A, B[np.ix_(perm, perm)]


def _oracle(A, B, **kw):
    n = A.shape[0]
    tr = {}
    a, hist, iters, conv = O.fw_core(A, B, None, np.full((n, n), 1.0 / n), trace=tr, **kw)
    return a, hist, iters, conv, tr


@pytest.mark.parametrize("world,n,directed,seed", [(2, 40, False, 1), (3, 37, True, 2), (2, 33, True, 3)])
def test_sharded_matches_oracle(world, n, directed, seed):
    A, B = _er_pair(n, 0.3, 0.8, directed, seed)
    kw = dict(max_iters=30, max_sweeps=1000, sense="maximize", lam=100.0, sk_tol=1e-8, fw_tol=1e-2)
    r = run_sharded(A, B, world, **kw)
    a, hist, iters, conv, tr = _oracle(A, B, **kw)
    assert r["iterations"] == iters and r["converged"] == conv
    assert r["lot_sweeps"] == tr["sweeps"]
    np.testing.assert_allclose(r["hist_alpha"][1:], [h[2] for h in hist[1:]], rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(r["hist_obj"], [h[1] for h in hist], rtol=1e-9)
    assert r["assignment"] == list(a)


def test_world_sizes_agree():
    A, B = _er_pair(30, 0.3, 0.9, True, 7)
    kw = dict(max_iters=10, max_sweeps=1000)
    r1 = run_sharded(A, B, 1, **kw)
    r2 = run_sharded(A, B, 2, **kw)
    assert r1["assignment"] == r2["assignment"]
    assert r1["lot_sweeps"] == r2["lot_sweeps"]
    np.testing.assert_allclose(r1["hist_alpha"][1:], r2["hist_alpha"][1:], rtol=1e-9)
    # per iteration: 1 all-gather (Q) + 1 dot allreduce + 1 min/max + one all-gather per pass
    assert r2["collectives"] > 3 * r2["iterations"]


def test_column_repair_round_is_exact():
    # A column-sum floor far above the fp64 range flags many columns every sweep;
    # the repair round (exact (max, sumexp) pairs over each rank's rows, gathered
    # and combined in rank order) must reproduce the unrepaired run.
    A, B = _er_pair(32, 0.3, 0.8, True, 11)
    kw = dict(max_iters=6, max_sweeps=1000)
    plain = run_sharded(A, B, 2, **kw)
    rep = run_sharded(A, B, 2, backend_kw=dict(tiny=0.5), **kw)
    assert rep["assignment"] == plain["assignment"]
    assert rep["lot_sweeps"] == plain["lot_sweeps"]
    np.testing.assert_allclose(rep["hist_alpha"][1:], plain["hist_alpha"][1:], rtol=1e-9)
    assert rep["collectives"] > plain["collectives"]  # the repair all-gathers ran


def test_layout_blocks_cover_rows():
    for n, w in [(10, 3), (40000, 8), (7, 7), (10, 4)]:
        rows = [ShardLayout(n, w, r).rows() for r in range(w)]
        assert rows[0][0] == 0 and sum(m for _, m in rows) == n
        assert all(rows[i][0] + rows[i][1] == rows[i + 1][0] for i in range(w - 1))
    with pytest.raises(ValueError):
        ShardLayout(9, 4, 0)  # ceil blocks of 3 leave the 4th rank empty
