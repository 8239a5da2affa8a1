"""Restarts spread over ranks (frank_wolfe_match / seeded_match with a process
group, matcher.py:254-285): each gloo rank runs its share of the independent
restarts, the results are gathered and the best is chosen in restart order --
the same result as the sequential loop.  The Frank-Wolfe core is the CPU
oracle here (no GPU in this container); the host bookkeeping under test is
the real engine's."""
import multiprocessing as mp
import socket

import numpy as np
import pytest
import torch.distributed as dist

from oracle import goat_oracle as O


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _patch_engine(setattr_=setattr):
    """Oracle stand-ins for the device calls the engine makes."""
    from paper_2111_05366_b200 import engine

    def core(A22, B22, L, P0, opts):
        n = A22.shape[0]
        P0 = np.full((n, n), 1.0 / n) if P0 is None else P0
        a, hist, it, conv = O.fw_core(A22, B22, L, P0, fw_tol=opts.fw_tol, max_iters=opts.max_iters,
                                      sense=opts.objective_sense)
        return np.asarray(a), hist, it, conv, None

    setattr_(engine, "fw_core", core)
    setattr_(engine, "fw_core_seeded", lambda A22, B22, A21, A12, B21, B12, P0, opts: core(
        A22, B22, A21 @ B21.T + A12.T @ B12, P0, opts))
    setattr_(engine, "qap_objective", lambda A, B, p, device=0: O.qap_objective_perm(A, B, p))
    return engine


def _run(A, B, seeds, opts_kw, group=None, setattr_=setattr):
    from paper_2111_05366_b200.records import MatchOptions, SeedSet
    engine = _patch_engine(setattr_)
    opts = MatchOptions(**opts_kw)
    if seeds is None:
        return engine.frank_wolfe_match(A, B, opts, group=group)
    return engine.seeded_match(A, B, SeedSet(seeds), opts, group=group)


def _worker(rank, world, port, A, B, seeds, opts_kw, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        r = _run(A, B, seeds, opts_kw, group=dist.group.WORLD)
        q.put((rank, r.alignment.tolist(), r.objective, r.iterations, [h[1] for h in r.iterate_history]))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, "err", repr(e), None, None))


@pytest.mark.parametrize("world,n_restarts,seeded", [(2, 4, False), (3, 5, True), (2, 1, False)])
def test_distributed_restarts_equal_sequential(world, n_restarts, seeded, monkeypatch):
    rng = np.random.default_rng(7 + world + n_restarts)
    n = 24
    A = (rng.random((n, n)) < 0.3).astype(float)
    np.fill_diagonal(A, 0)
    B = A[np.ix_(rng.permutation(n), rng.permutation(n))]
    seeds = np.array([[0, 3], [5, 1]]) if seeded else None
    opts_kw = dict(step_solver="lot", n_restarts=n_restarts, shuffle_input=True, rng_seed=3, max_iters=6)
    ref = _run(A, B, seeds, opts_kw, setattr_=monkeypatch.setattr)  # sequential loop, this process
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, A, B, seeds, opts_kw, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
    for rank, align, obj, iters, hist in outs:
        assert align != "err", (rank, obj)
        assert align == ref.alignment.tolist()
        assert obj == ref.objective and iters == ref.iterations
        np.testing.assert_array_equal(hist, [h[1] for h in ref.iterate_history])
