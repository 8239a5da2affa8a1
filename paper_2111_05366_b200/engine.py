"""Frank-Wolfe graph matching entry points (drop-in for otmatch's engine).

``frank_wolfe_match`` / ``seeded_match`` keep the reference's signatures,
options and results (matcher.py:298-310).  The host keeps exactly the
bookkeeping the reference does around its Frank-Wolfe core -- input
validation, seed reordering, per-restart numpy RNG streams
``default_rng([rng_seed, r])``, input shuffling, the seeded linear term and
the best-of-restarts choice (matcher.py:230-295) -- so the random streams and
relabelings are identical; the core itself (matcher.py:177-212: gradient,
LOT, exact line search, update, final LAP) runs on the device in one
``goat_fw_core`` call.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .matrices import as_square_matrix, invert_permutation, permute_matrix, qap_objective
from .ops import randomized_blend_init
from .records import MatchOptions, MatchResult, SeedSet

__all__ = ["frank_wolfe_match", "seeded_match", "fw_core", "fw_core_csr", "as_csr", "is_sparse"]


def fw_core(A, B, L, P0, opts: MatchOptions):
    """Device Frank-Wolfe core: the replacement for ``_fw_core`` (matcher.py:177-212).

    ``P0=None`` means the barycenter.  Returns (assignment, history, iterations,
    converged, diagnostics).
    """
    n = A.shape[0]
    h = _lib.handle(opts.device, opts.precision)
    A_ = _lib.f64(A)
    B_ = _lib.f64(B)
    L_ = _lib.f64(L) if L is not None else None
    P_ = _lib.f64(P0) if P0 is not None else None
    return _call_core(n, opts, h, lambda lib, o, res: lib.goat_fw_core(
        h.ptr, n, _lib.dptr(A_), _lib.ld_of(A_), _lib.dptr(B_), _lib.ld_of(B_),
        _lib.dptr(L_) if L_ is not None else None, _lib.ld_of(L_) if L_ is not None else n,
        _lib.dptr(P_) if P_ is not None else None, _lib.ld_of(P_) if P_ is not None else n, o, res))


def fw_core_seeded(A22, B22, A21, A12, B21, B12, P0, opts: MatchOptions):
    """``fw_core`` with the seed term formed on the device (goat_fw_core_seeded):
    L = A21 B21^T + A12^T B12 (matcher.py:267) from the seed blocks."""
    nf, m = A21.shape
    h = _lib.handle(opts.device, opts.precision)
    blocks = [_lib.f64(x) for x in (A22, B22, A21, A12, B21, B12)]
    P_ = _lib.f64(P0) if P0 is not None else None
    args = []
    for b in blocks:
        args += [_lib.dptr(b), _lib.ld_of(b) if b.shape[0] > 1 else b.shape[1]]
    return _call_core(nf, opts, h, lambda lib, o, res: lib.goat_fw_core_seeded(
        h.ptr, nf, m, *args, _lib.dptr(P_) if P_ is not None else None, _lib.ld_of(P_) if P_ is not None else nf,
        o, res))


def _call_core(n, opts: MatchOptions, h, call):
    mi = opts.max_iters
    assign = np.empty(n, dtype=np.int64)
    hobj = np.empty(mi + 1)
    halpha = np.empty(mi + 1)
    sweeps = np.zeros(mi, dtype=np.int32)
    lconv = np.zeros(mi, dtype=np.int32)
    ldev = np.zeros(mi)
    f64from = np.full(mi, -1, dtype=np.int32)
    lot_ms = np.zeros(mi)
    res = _lib.GoatFwResult()
    res.assignment = assign.ctypes.data_as(_lib._c_i64_p)
    res.hist_obj = _lib.dptr(hobj)
    res.hist_alpha = _lib.dptr(halpha)
    res.lot_sweeps = sweeps.ctypes.data_as(_lib._c_i32_p)
    res.lot_converged = lconv.ctypes.data_as(_lib._c_i32_p)
    res.lot_dev = _lib.dptr(ldev)
    res.lot_fp64_from = f64from.ctypes.data_as(_lib._c_i32_p)
    res.lot_ms = _lib.dptr(lot_ms)
    o = _lib.GoatOptions(
        max_iters=mi, max_sweeps=opts.sinkhorn.max_sweeps,
        sense=_lib.GOAT_MAXIMIZE if opts.objective_sense == "maximize" else _lib.GOAT_MINIMIZE,
        step_solver=_lib.GOAT_STEP_LOT if opts.step_solver == "lot" else _lib.GOAT_STEP_EXACT_LAP,
        fw_tol=opts.fw_tol, lam=opts.sinkhorn.lam, sk_tol=opts.sinkhorn.tol)
    lib = _lib.load()
    with h.lock:
        _lib.check(call(lib, ctypes.byref(o), ctypes.byref(res)))
    it = int(res.iterations)
    history = [(0, float(hobj[0]), None)]
    history += [(i, float(hobj[i]), float(halpha[i])) for i in range(1, it + 1)]
    diag = dict(lot_sweeps=sweeps[:it].tolist(), lot_converged=lconv[:it].astype(bool).tolist(),
                lot_deviation=ldev[:it].tolist(), lot_fp64_from=f64from[:it].tolist(), lot_ms=lot_ms[:it].tolist(),
                lap_certified=bool(res.lap_certified),
                gpu_launches=int(res.gpu_launches), objective=float(res.objective),
                time_ms=dict(zip(("gradient", "lot", "line_search", "lap", "setup", "total"),
                                 list(res.time_ms))))
    return assign.astype(np.intp), history, it, bool(res.converged), diag


def is_sparse(M) -> bool:
    """scipy.sparse matrices and CSR graphs (graphs.CsrGraph) take the CSR path."""
    from .graphs import CsrGraph
    try:
        import scipy.sparse as sp
        if sp.issparse(M):
            return True
    except ImportError:  # pragma: no cover
        pass
    return isinstance(M, CsrGraph)


def CsrGraphType():
    from .graphs import CsrGraph
    return CsrGraph


def as_csr(M, name: str = "matrix"):
    """Canonical float64 scipy CSR (sorted rows, duplicates summed) with the
    reference's validation (core.py:17-27): square, finite."""
    import scipy.sparse as sp

    from .graphs import CsrGraph
    if isinstance(M, CsrGraph):
        M = sp.csr_matrix((np.ones(M.indices.size), M.indices, M.indptr), shape=(M.n, M.n))
    M = sp.csr_matrix(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError(f"{name} must be square, got shape {M.shape}")
    M.sum_duplicates()
    M.sort_indices()
    if not np.all(np.isfinite(M.data)):
        raise ValueError(f"{name} contains non-finite entries")
    return M


def _csr_arrays(M):
    indptr = np.ascontiguousarray(M.indptr, dtype=np.int64)
    indices = np.ascontiguousarray(M.indices, dtype=np.int32)
    vals = None if np.all(M.data == 1.0) else np.ascontiguousarray(M.data, dtype=np.float64)
    return indptr, indices, vals


def fw_core_csr(A, B, L, P0, opts: MatchOptions):
    """``fw_core`` for CSR adjacency (gradient by SpMM; goat_fw_core_csr)."""
    A = as_csr(A, "A")
    B = as_csr(B, "B")
    n = A.shape[0]
    h = _lib.handle(opts.device, opts.precision)
    aa, ba = _csr_arrays(A), _csr_arrays(B)
    ca, cb = _lib.csr_struct(*aa), _lib.csr_struct(*ba)
    L_ = _lib.f64(L) if L is not None else None
    P_ = _lib.f64(P0) if P0 is not None else None
    return _call_core(n, opts, h, lambda lib, o, res: lib.goat_fw_core_csr(
        h.ptr, n, ctypes.byref(ca), ctypes.byref(cb),
        _lib.dptr(L_) if L_ is not None else None, _lib.ld_of(L_) if L_ is not None else n,
        _lib.dptr(P_) if P_ is not None else None, _lib.ld_of(P_) if P_ is not None else n, o, res))


def _initial(n, opts: MatchOptions, rng):
    # matcher.py:215-223; None = barycenter (the device forms it on the fly)
    if isinstance(opts.init, str):
        if opts.init == "barycenter":
            return None
        return randomized_blend_init(n, rng, device=opts.device)
    P0 = as_square_matrix(opts.init, "init")
    if P0.shape[0] != n:
        raise ValueError(f"supplied init has order {P0.shape[0]}, expected {n}")
    return P0


def _quadratic_1x1(A22, B22, L):
    val = float(A22[0, 0] * B22[0, 0])
    return val + (float(L[0, 0]) if L is not None else 0.0)


def _match(A, B, pairs: np.ndarray, opts: MatchOptions, group=None) -> MatchResult:
    t0 = time.perf_counter()
    sparse = is_sparse(A) or is_sparse(B)
    if sparse:
        # CSR path: the same host bookkeeping on scipy CSR matrices; the core
        # runs goat_fw_core_csr (SpMM gradient, no dense A or B on the device)
        A = as_csr(A, "A")
        B = as_csr(B, "B")
    else:
        # unseeded dense runs of order > 1 go straight to goat_fw_core, which checks
        # finiteness during the upload (same ValueError); everything else checks here
        dev_check = pairs.shape[0] == 0 and np.ndim(A) == 2 and np.shape(A)[0] > 1
        A = as_square_matrix(A, "A", check_finite=not dev_check)
        B = as_square_matrix(B, "B", check_finite=not dev_check)
    if A.shape != B.shape:
        raise ValueError(f"order mismatch: {A.shape[0]} vs {B.shape[0]}")
    n = A.shape[0]
    m = pairs.shape[0]
    if m >= n:
        raise ValueError(f"seed count {m} must be less than order {n}")
    if m and (pairs.min() < 0 or pairs.max() >= n):
        raise ValueError("seed vertex out of range")
    # seeds first, identity-aligned at [0, m) (matcher.py:244-250)
    rest1 = np.setdiff1d(np.arange(n), pairs[:, 0]) if m else np.arange(n)
    rest2 = np.setdiff1d(np.arange(n), pairs[:, 1]) if m else np.arange(n)
    ord1 = np.concatenate([pairs[:, 0], rest1]).astype(np.intp)
    ord2 = np.concatenate([pairs[:, 1], rest2]).astype(np.intp)
    if sparse:
        Ar = A[ord1][:, ord1] if m else A
        Br = B[ord2][:, ord2] if m else B
    else:
        Ar = A[np.ix_(ord1, ord1)] if m else A
        Br = B[np.ix_(ord2, ord2)] if m else B
    nf = n - m

    def restart(r):
        rng = np.random.default_rng([opts.rng_seed, r])
        if opts.shuffle_input and nf > 1:
            shuf = rng.permutation(nf).astype(np.intp)
        else:
            shuf = np.arange(nf, dtype=np.intp)
        inv = invert_permutation(shuf)
        if sparse:
            B22 = Br[m:, m:][inv][:, inv] if opts.shuffle_input else Br[m:, m:]
        else:
            B22 = permute_matrix(Br[m:, m:], shuf) if opts.shuffle_input else Br[m:, m:]
        A22 = Ar[m:, m:]
        L = None
        seed_blocks = None
        if m:
            B12 = Br[:m, m:][:, inv]
            B21 = Br[m:, :m][inv, :]
            if sparse:
                L = Ar[m:, :m] @ B21.T + Ar[:m, m:].T @ B12  # constant seed term (matcher.py:267)
                L = np.asarray(L.toarray(), dtype=np.float64)
            else:
                # formed on the device from the seed blocks (goat_fw_core_seeded)
                seed_blocks = (Ar[m:, :m], Ar[:m, m:], B21, B12)
        diag = None
        if nf == 1:
            p22 = np.zeros(1, dtype=np.intp)
            if seed_blocks is not None:  # 1 x 1 seed term on the host (matcher.py:267)
                L = seed_blocks[0] @ seed_blocks[2].T + seed_blocks[1].T @ seed_blocks[3]
            history, iters, conv = [(0, _quadratic_1x1(A22, B22, L), None)], 0, True
        else:
            P0 = _initial(nf, opts, rng)
            if seed_blocks is not None:
                A21, A12, B21_, B12_ = seed_blocks
                p22, history, iters, conv, diag = fw_core_seeded(A22, B22, A21, A12, B21_, B12_, P0, opts)
            else:
                core = fw_core_csr if sparse else fw_core
                p22, history, iters, conv, diag = core(A22, B22, L, P0, opts)
        p22 = inv[p22]
        align = np.empty(n, dtype=np.intp)
        align[ord1[:m]] = ord2[:m]
        align[ord1[m:]] = ord2[m + p22]
        if m == 0 and diag is not None:
            # same terms A_ij B_{align(i) align(j)}, already reduced on the device
            obj = diag["objective"]
        elif sparse:
            obj = float(A.multiply(B[align][:, align]).sum())  # core.py:120-124 on the CSR inputs
        else:
            obj = qap_objective(A, B, align, device=opts.device)
        return align, obj, iters, history, conv, diag

    # restarts are independent (matcher.py:254-285): with a process group each
    # rank runs restarts r = rank, rank + world, ... on its own GPU and the
    # results are gathered; the choice below is the reference's, in restart order
    if group is not None and _dist_world(group) > 1:
        results = _gather_restarts(restart, opts.n_restarts, group)
    else:
        results = [restart(r) for r in range(opts.n_restarts)]
    best = None
    for res_r in results:
        obj = res_r[1]
        if best is None or (obj > best[1] if opts.objective_sense == "maximize" else obj < best[1]):
            best = res_r
    align, obj, iters, history, conv, diag = best
    return MatchResult(alignment=align, objective=obj, iterations=iters, iterate_history=history,
                       converged=conv, wall_time=time.perf_counter() - t0, diagnostics=diag)


def _dist_world(group):
    import torch.distributed as dist
    return dist.get_world_size(group)


def _gather_restarts(restart, n_restarts, group):
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = {r: restart(r) for r in range(rank, n_restarts, world)}
    allres = [None] * world
    dist.all_gather_object(allres, mine, group=group)
    merged = {}
    for d in allres:
        merged.update(d)
    return [merged[r] for r in range(n_restarts)]


def frank_wolfe_match(A, B, opts: MatchOptions = MatchOptions(), *, group=None) -> MatchResult:
    """Match two equal-order graphs; FAQ or GOAT depending on ``opts.step_solver``.
    ``group`` (a torch.distributed process group, one rank per GPU) spreads the
    ``n_restarts`` independent restarts over the ranks; every rank returns the
    same result as the sequential loop."""
    return _match(A, B, np.empty((0, 2), dtype=np.intp), opts, group)


def seeded_match(A, B, seeds: SeedSet, opts: MatchOptions = MatchOptions(), *, group=None) -> MatchResult:
    """Match with seed pairs pinned; Frank-Wolfe over the free block only."""
    return _match(A, B, seeds.pairs, opts, group)
