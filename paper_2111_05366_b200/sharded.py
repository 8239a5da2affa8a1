"""Row-sharded GOAT iteration: one process per GPU, NCCL between them.

The reference has no distributed path; this splits the Frank-Wolfe core
(matcher.py:177-212) by row blocks as SURVEY.md 8(e) lays out.  Rank r owns
rows [r*m, r*m + m) of the n x n iterates P, Q, G (m = ceil(n / world), the last
block may be short) plus the same rows of A and A^T; B is replicated.  Per outer
iteration:

  LOT (sinkhorn.py:103-130)   global min/max of G (2 allreduces), then per sweep
                              one local pass over the block, an all-gather of the
                              (n+1)-vector [column sums | row deviation] and a
                              merge in rank order -- identical on every rank, so
                              every rank takes the same stopping decision
  gradient (matcher.py:107)   all-gather Q, then G_r = (A_r Q) B^T + (A^T_r Q) B
                              on the rank's own rows
  line search (:110-135)      6 local dot products, one sum-allreduce
  update (:197)               local axpby on P and G (the recurrence G(P') =
                              a G(P) + (1-a) G(Q) needs no communication)
  final LAP (:205-211)        all-gather G, rank 0 solves, broadcast.

The compute runs behind a backend (GpuShardBackend: the goat_shard_* C ABI on
this rank's GPU); the collectives go through torch.distributed (NCCL on GPUs,
gloo in the CPU tests, which substitute a numpy backend for the kernels).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .ops import optimal_alpha


def ld_for(n: int) -> int:
    return (max(n, 1) + 7) // 8 * 8


@dataclass
class ShardLayout:
    """Row-block partition of n rows over `world` ranks."""

    n: int
    world: int
    rank: int

    def __post_init__(self):
        if self.world < 1 or not (0 <= self.rank < self.world):
            raise ValueError("bad rank / world size")
        self.m_pad = -(-self.n // self.world)
        if self.m_pad * (self.world - 1) >= self.n:
            raise ValueError(f"n={self.n} is too small to give each of {self.world} ranks a row block")
        self.r0 = self.rank * self.m_pad
        self.m = min(self.m_pad, self.n - self.r0)
        self.ld = ld_for(self.n)

    def rows(self, rank=None):
        r = self.rank if rank is None else rank
        r0 = r * self.m_pad
        return r0, min(self.m_pad, self.n - r0)


class Comm:
    """The collectives the driver needs, over a torch.distributed process group."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_gather_rows(self, out_full: torch.Tensor, block: torch.Tensor):
        dist.all_gather_into_tensor(out_full, block, group=self.group)

    def sum(self, values) -> np.ndarray:
        t = torch.tensor(np.asarray(values, dtype=np.float64), device=self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def min_max(self, lo: float, hi: float):
        t = torch.tensor([-lo, hi], dtype=torch.float64, device=self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return -float(t[0]), float(t[1])

    def broadcast_perm(self, perm: np.ndarray | None, n: int) -> np.ndarray:
        t = torch.zeros(n, dtype=torch.int64, device=self._dev())
        if self.rank == 0:
            t.copy_(torch.from_numpy(np.asarray(perm, dtype=np.int64)))
        dist.broadcast(t, src=0, group=self.group)
        return t.cpu().numpy()

    def _dev(self):
        return torch.device("cuda", torch.cuda.current_device()) \
            if dist.get_backend(self.group) == "nccl" else torch.device("cpu")


class GpuShardBackend:
    """This rank's compute: the goat_shard_* entry points of libgoat.so."""

    def __init__(self, layout: ShardLayout, precision: str = "fp32", device: int | None = None,
                 gemm: str = "auto"):
        if not torch.cuda.is_available():
            raise RuntimeError("GpuShardBackend needs a CUDA device (no CPU fallback)")
        self.layout = layout
        self.device = torch.cuda.current_device() if device is None else device
        self.dtype = torch.float32 if precision == "fp32" else torch.float64
        self.h = _lib.Handle(self.device, precision, gemm)
        self.lib = _lib.load()
        self.dev = torch.device("cuda", self.device)
        # the library and torch (all-gathers, uploads) share this rank's current stream
        _lib.check(self.lib.goat_set_stream(self.h.ptr, _lib.stream_handle(torch.cuda.current_stream(self.dev))))

    # buffers ------------------------------------------------------------
    def block(self):
        return torch.zeros((self.layout.m_pad, self.layout.ld), dtype=self.dtype, device=self.dev)

    def full(self):
        return torch.zeros((self.layout.m_pad * self.layout.world, self.layout.ld), dtype=self.dtype,
                           device=self.dev)

    def vec(self, *shape):
        return torch.zeros(shape, dtype=torch.float64, device=self.dev)

    def upload(self, x: np.ndarray, rows: int | None = None) -> torch.Tensor:
        L = self.layout
        out = torch.zeros((rows or x.shape[0], L.ld), dtype=self.dtype, device=self.dev)
        out[: x.shape[0], : L.n] = torch.from_numpy(np.ascontiguousarray(x)).to(self.dev, self.dtype)
        return out

    # kernels ------------------------------------------------------------
    def setup(self, A_rows: torch.Tensor, AT_rows: torch.Tensor | None, B: torch.Tensor):
        L = self.layout
        _lib.check(self.lib.goat_shard_setup(self.h.ptr, L.n, L.m, A_rows.data_ptr(),
                                             AT_rows.data_ptr() if AT_rows is not None else None,
                                             B.data_ptr(), L.ld))

    def setup_csr(self, A_rows, AT_rows, B, BT):
        """CSR variant of ``setup``: each argument is (rowptr, colidx[, values]) of
        CUDA tensors (AT_rows and BT None together for symmetric inputs)."""
        L = self.layout
        self._csr_keep = (A_rows, AT_rows, B, BT)  # the library copies; keep until the call returns
        st = [None if x is None else _lib.csr_struct_device(*x) for x in (A_rows, AT_rows, B, BT)]
        ref = [None if c is None else ctypes.byref(c) for c in st]
        _lib.check(self.lib.goat_shard_setup_csr(self.h.ptr, L.n, L.m, *ref))

    def gradient(self, Q_full, out):
        _lib.check(self.lib.goat_shard_gradient(self.h.ptr, Q_full.data_ptr(), out.data_ptr()))

    def minmax(self, X):
        o = (ctypes.c_double * 2)()
        _lib.check(self.lib.goat_shard_minmax(self.h.ptr, X.data_ptr(), o))
        return o[0], o[1]

    def lot_begin(self, sense, lam, lo, hi, max_sweeps, tol):
        _lib.check(self.lib.goat_shard_lot_begin(self.h.ptr, sense, lam, lo, hi, max_sweeps, tol))

    def lot_pass(self, G, send):
        _lib.check(self.lib.goat_shard_lot_pass(self.h.ptr, G.data_ptr(), send.data_ptr()))

    def lot_merge(self, recv, world):
        _lib.check(self.lib.goat_shard_lot_merge(self.h.ptr, recv.data_ptr(), world))

    def lot_status(self):
        """(done, sweeps, converged, deviation, columns repaired, repair pending)"""
        d, s, c, r, p = (ctypes.c_int32() for _ in range(5))
        dev = ctypes.c_double()
        _lib.check(self.lib.goat_shard_lot_status(self.h.ptr, ctypes.byref(d), ctypes.byref(s), ctypes.byref(c),
                                                  ctypes.byref(dev), ctypes.byref(r), ctypes.byref(p)))
        return d.value, s.value, c.value, dev.value, r.value, p.value

    def lot_refine(self, G) -> bool:
        """fp32: re-open a LOT that stopped at the fp32 deviation floor, in fp64 arithmetic."""
        started = ctypes.c_int32()
        _lib.check(self.lib.goat_shard_lot_refine(self.h.ptr, G.data_ptr(), ctypes.byref(started)))
        return bool(started.value)

    def lot_repair_pass(self, G, pairs):
        _lib.check(self.lib.goat_shard_lot_repair_pass(self.h.ptr, G.data_ptr(), pairs.data_ptr()))

    def lot_repair_merge(self, recv_pairs, world):
        _lib.check(self.lib.goat_shard_lot_repair_merge(self.h.ptr, recv_pairs.data_ptr(), world))

    def lot_emit(self, G, Q):
        _lib.check(self.lib.goat_shard_lot_emit(self.h.ptr, G.data_ptr(), Q.data_ptr()))

    def dots(self, GP, GQ, P, Q):
        o = (ctypes.c_double * 6)()
        _lib.check(self.lib.goat_shard_dots(self.h.ptr, GP.data_ptr(), GQ.data_ptr(), P.data_ptr(), Q.data_ptr(), o))
        return np.array(o[:])

    def axpby(self, a, X, b, Y):
        _lib.check(self.lib.goat_shard_axpby(self.h.ptr, a, X.data_ptr(), b, Y.data_ptr()))

    def fill(self, value, X):
        _lib.check(self.lib.goat_shard_fill(self.h.ptr, value, X.data_ptr()))

    def lap(self, G_full, sense):
        n = self.layout.n
        perm = np.zeros(n, dtype=np.int64)
        _lib.check(self.lib.goat_lap_device(self.h.ptr, n, G_full.data_ptr(), self.layout.ld, sense,
                                            perm.ctypes.data_as(_lib._c_i64_p), None, None))
        return perm


@dataclass
class ShardedResult:
    assignment: np.ndarray
    hist_obj: list = field(default_factory=list)
    hist_alpha: list = field(default_factory=list)
    lot_sweeps: list = field(default_factory=list)
    lot_converged: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    collectives: int = 0


def sharded_fw_core(backend, comm: Comm, A_rows, AT_rows, B, *, max_iters=30, max_sweeps=1000,
                    sense="maximize", lam=100.0, sk_tol=1e-8, fw_tol=1e-2, poll=8,
                    trace: dict | None = None) -> ShardedResult:
    """GOAT's _fw_core (matcher.py:177-212) from the barycenter, row-sharded.

    A_rows / AT_rows: this rank's rows of A and A^T (AT_rows None: A, B symmetric);
    B: the full B.  All are backend buffers.  Returns the same history as goat_fw_core.
    ``trace`` (small n, diagnostics): receives this rank's G and Q blocks per iteration.
    """
    L = backend.layout
    world = comm.world
    sense_code = _lib.GOAT_MAXIMIZE if sense == "maximize" else _lib.GOAT_MINIMIZE
    if A_rows is not None:  # None: the caller already ran backend.setup_csr
        backend.setup(A_rows, AT_rows, B)
    P, Q, G, GQ = backend.block(), backend.block(), backend.block(), backend.block()
    full = backend.full()
    send = backend.vec(L.n + 1)
    recv = backend.vec(world, L.n + 1)
    pairs = backend.vec(2 * L.n)
    recv_pairs = backend.vec(world, 2 * L.n)
    res = ShardedResult(assignment=np.zeros(L.n, dtype=np.int64))
    ncoll = 0

    # P0 = J / n (core.py:89-93) and G(P0)
    backend.fill(1.0 / L.n, P)
    comm.all_gather_rows(full, P); ncoll += 1
    backend.gradient(full, G)
    d = comm.sum(backend.dots(G, G, P, P)); ncoll += 1
    res.hist_obj.append(0.5 * d[2])
    res.hist_alpha.append(float("nan"))

    for it in range(1, max_iters + 1):
        # ---- LOT step (matcher.py:193-194)
        lo, hi = comm.min_max(*backend.minmax(G)); ncoll += 1
        backend.lot_begin(sense_code, lam, lo, hi, max_sweeps, sk_tol)
        done, sweeps, conv, _, _, pending = backend.lot_status()
        rounds = 0
        refined = False
        while True:
            if done:
                # fp32 sweeps that stopped at the fp32 deviation floor go on in fp64
                # (every rank holds the same loop state, so all take the same branch)
                if refined or not backend.lot_refine(G):
                    break
                refined = True
                done, sweeps, conv, _, _, pending = backend.lot_status()
                continue
            # `poll` sweeps per host check; once a sweep is left pending for a column
            # repair the rest of the chunk is no-ops on every rank
            for _ in range(poll):
                backend.lot_pass(G, send)
                comm.all_gather_rows(recv.view(-1), send); ncoll += 1
                backend.lot_merge(recv, world)
            done, sweeps, conv, _, _, pending = backend.lot_status()
            if pending:
                backend.lot_repair_pass(G, pairs)
                comm.all_gather_rows(recv_pairs.view(-1), pairs); ncoll += 1
                backend.lot_repair_merge(recv_pairs, world)
                done, sweeps, conv, _, _, pending = backend.lot_status()
            rounds += 1
            if not done and rounds * poll > 4 * (max_sweeps + 2):
                raise RuntimeError("sharded Sinkhorn loop did not terminate")
        backend.lot_emit(G, Q)
        if trace is not None:
            trace.setdefault("G", []).append(G[: L.m, : L.n].cpu().numpy().copy())
            trace.setdefault("Q", []).append(Q[: L.m, : L.n].cpu().numpy().copy())
        res.lot_sweeps.append(sweeps)
        res.lot_converged.append(bool(conv))
        # ---- gradient at Q
        comm.all_gather_rows(full, Q); ncoll += 1
        backend.gradient(full, GQ)
        # ---- exact line search (matcher.py:110-135) in difference form
        d = comm.sum(backend.dots(G, GQ, P, Q)); ncoll += 1
        c1, c2, fQ, nrm = d[0], 0.5 * d[1], 0.5 * d[2], d[3]
        al = optimal_alpha(c2, c1, sense)
        bl = 1.0 - al
        res.hist_obj.append(fQ + al * c1 + al * al * c2)
        res.hist_alpha.append(al)
        step = abs(bl) * math.sqrt(max(nrm, 0.0))
        if al == 0.0:
            P, Q = Q, P
            G, GQ = GQ, G
        elif al != 1.0:
            backend.axpby(bl, Q, al, P)
            backend.axpby(bl, GQ, al, G)
        res.iterations = it
        if step < fw_tol:
            res.converged = True
            break

    # ---- final projection (matcher.py:205-211)
    comm.all_gather_rows(full, G); ncoll += 1
    perm = backend.lap(full, sense_code) if comm.rank == 0 else None
    res.assignment = comm.broadcast_perm(perm, L.n); ncoll += 1
    res.collectives = ncoll
    return res


def _csr_rows_to_device(M, dev, dtype):
    rowptr = torch.from_numpy(np.ascontiguousarray(M.indptr, dtype=np.int64)).to(dev)
    col = torch.from_numpy(np.ascontiguousarray(M.indices, dtype=np.int32)).to(dev)
    if np.all(M.data == 1.0):
        return (rowptr, col)
    return (rowptr, col, torch.from_numpy(np.ascontiguousarray(M.data)).to(dev, dtype))


def prepare_csr(A, B, *, precision="fp32", group=None, gemm="auto"):
    """Upload this rank's CSR rows of A and A^T and the whole CSR of B (and B^T)
    and set up the shard handle; returns (backend, comm) for ``sharded_fw_core``
    with ``A_rows=None`` (inputs resident on the device)."""
    from . import engine
    comm = Comm(group)
    A = engine.as_csr(A, "A")
    B = engine.as_csr(B, "B")
    layout = ShardLayout(A.shape[0], comm.world, comm.rank)
    be = GpuShardBackend(layout, precision, gemm=gemm)
    r0, m = layout.r0, layout.m
    sym = (A != A.T).nnz == 0 and (B != B.T).nnz == 0
    dev, dt = be.dev, be.dtype
    a_rows = _csr_rows_to_device(A[r0:r0 + m], dev, dt)
    At = A.T.tocsr(); At.sort_indices()
    at_rows = None if sym else _csr_rows_to_device(At[r0:r0 + m], dev, dt)
    b_full = _csr_rows_to_device(B, dev, dt)
    Bt = B.T.tocsr(); Bt.sort_indices()
    bt_full = None if sym else _csr_rows_to_device(Bt, dev, dt)
    be.setup_csr(a_rows, at_rows, b_full, bt_full)
    return be, comm


def sharded_match(A, B, *, precision="fp32", group=None, gemm="auto", **kw) -> ShardedResult:
    """Row-sharded GOAT on this rank's GPU (every rank passes the full matrices;
    each uploads only its own rows of A and A^T, and B).  Dense host arrays run the
    GEMM gradient; scipy.sparse / CSR graphs run the SpMM gradient on CSR rows."""
    from . import engine
    if engine.is_sparse(A) or engine.is_sparse(B):
        be, comm = prepare_csr(A, B, precision=precision, group=group, gemm=gemm)
        return sharded_fw_core(be, comm, None, None, None, **kw)
    comm = Comm(group)
    n = A.shape[0]
    layout = ShardLayout(n, comm.world, comm.rank)
    be = GpuShardBackend(layout, precision, gemm=gemm)
    r0, m = layout.r0, layout.m
    sym = bool(np.array_equal(A, A.T) and np.array_equal(B, B.T))
    A_rows = be.upload(A[r0:r0 + m], layout.m_pad)
    AT_rows = None if sym else be.upload(np.ascontiguousarray(A.T[r0:r0 + m]), layout.m_pad)
    Bd = be.upload(B)
    return sharded_fw_core(be, comm, A_rows, AT_rows, Bd, **kw)
