"""Seeded synthetic graph pairs for the five BASELINE configurations.

These produce the *inputs* of the GOAT path (they are not part of the hot
path).  c1/c3 follow the reference sampler's law and RNG draw order exactly
(``samplers.py:48-72`` and ``:75-78``), so they reproduce the reference's
matrices bit-for-bit from the same ``numpy.random.Generator``; c2 (directed)
and c4 (weighted) need laws the reference does not have, defined here and in
DESIGN.md; c5 is generated block-wise straight into CSR because a dense
40000^2 float64 draw does not fit host memory.

Seeding convention: ``rng = default_rng([config, replicate])``,
sample (A, B), then ``Bs, truth = shuffle(B, rng)`` with the same rng.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "SbmSpec", "sample_sbm_pair", "replicate_rng",
    "correlated_sbm_pair", "correlated_er_pair", "directed_er_pair",
    "weighted_directed_pair", "shuffle", "relabel", "CsrGraph",
    "sparse_er_pair_csr", "config_pair", "CONFIGS",
]


def _correlated_bernoulli(Pm, rho, rng):
    # samplers.py:60-65: A ~ Bern(p); B | A=1 ~ Bern(p + rho(1-p)); B | A=0 ~ Bern(p(1-rho)).
    n = Pm.shape[0]
    U = rng.uniform(size=(n, n))
    A = (U < Pm).astype(np.float64)
    V = rng.uniform(size=(n, n))
    B = np.where(A == 1.0, V < Pm + rho * (1.0 - Pm), V < Pm * (1.0 - rho)).astype(np.float64)
    return A, B


def correlated_sbm_pair(block_sizes, block_probs, rho, rng):
    """Undirected rho-correlated SBM pair, identity-aligned (law of samplers.py:48-72)."""
    sizes = [int(s) for s in block_sizes]
    probs = np.asarray(block_probs, dtype=np.float64)
    labels = np.repeat(np.arange(len(sizes)), sizes)
    Pm = probs[np.ix_(labels, labels)]
    A, B = _correlated_bernoulli(Pm, float(rho), rng)
    n = Pm.shape[0]
    lo = np.tril_indices(n)
    iu = np.triu_indices(n, 1)
    for M in (A, B):  # upper triangle mirrored, hollow (samplers.py:68-71)
        M[lo] = 0.0
        M[(iu[1], iu[0])] = M[iu]
    return A, B


@dataclass(frozen=True)
class SbmSpec:
    """Block sizes, symmetric block edge probabilities and edge correlation of a
    correlated SBM (samplers.py:17-46; same validation and ValueErrors)."""

    block_sizes: tuple
    block_probs: np.ndarray
    rho: float

    def __post_init__(self):
        sizes = tuple(int(b) for b in self.block_sizes)
        if len(sizes) == 0 or min(sizes) < 1:
            raise ValueError("block_sizes must be positive integers")
        probs = np.asarray(self.block_probs, dtype=float)
        if probs.shape != (len(sizes), len(sizes)):
            raise ValueError(f"block_probs must be {len(sizes)}x{len(sizes)}, got {probs.shape}")
        if not np.allclose(probs, probs.T):
            raise ValueError("block_probs must be symmetric")
        if probs.min() < 0 or probs.max() > 1:
            raise ValueError("block_probs entries must lie in [0, 1]")
        if not 0.0 <= self.rho <= 1.0:
            raise ValueError("rho must lie in [0, 1]")
        object.__setattr__(self, "block_sizes", sizes)
        object.__setattr__(self, "block_probs", probs)

    @property
    def n(self) -> int:
        return sum(self.block_sizes)


def sample_sbm_pair(spec: SbmSpec, rng):
    """rho-correlated SBM pair with identity correspondence (samplers.py:48-72)."""
    return correlated_sbm_pair(spec.block_sizes, spec.block_probs, spec.rho, rng)


def replicate_rng(master_seed: int, replicate: int):
    """Independent deterministic stream of one replicate (samplers.py:92-94)."""
    return np.random.default_rng([master_seed, replicate])


def correlated_er_pair(n, p, rho, rng):
    """Undirected correlated ER pair = single-block SBM (samplers.py:75-78)."""
    return correlated_sbm_pair((n,), [[p]], rho, rng)


def directed_er_pair(n, p, rho, rng):
    """Directed correlated ER (config 2): the same per-entry conditional law over
    every off-diagonal (i, j) independently, no symmetrisation, zero diagonal."""
    A, B = _correlated_bernoulli(np.full((n, n), float(p)), float(rho), rng)
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(B, 0.0)
    return A, B


def weighted_directed_pair(n, p, rng, sigma=1.0, noise_sigma=0.2, resample=0.1):
    """Config 4: directed ER(p) support with lognormal(0, sigma) weights.

    B = A * lognormal(0, noise_sigma) on A's support, then a uniformly chosen
    ``resample`` fraction of B's edges is deleted and the same number of edges
    is inserted at uniformly chosen off-diagonal non-edges with fresh
    lognormal(0, sigma) weights (the definition SURVEY.md §8d suggests).
    """
    S = rng.uniform(size=(n, n)) < p
    np.fill_diagonal(S, False)
    W = rng.lognormal(0.0, sigma, size=(n, n))
    A = np.where(S, W, 0.0)
    noise = rng.lognormal(0.0, noise_sigma, size=(n, n))
    B = np.where(S, A * noise, 0.0)
    edges = np.flatnonzero(S.ravel())
    k = int(round(resample * edges.size))
    if k:
        drop = rng.choice(edges, size=k, replace=False)
        offdiag_gap = ~S
        np.fill_diagonal(offdiag_gap, False)
        gaps = np.flatnonzero(offdiag_gap.ravel())
        add = rng.choice(gaps, size=k, replace=False)
        flat = B.ravel()
        flat[drop] = 0.0
        flat[add] = rng.lognormal(0.0, sigma, size=k)
    return A, B


def relabel(B, p):
    """Vertex v of B becomes vertex p[v] (core.py:152-163): out[p[i], p[j]] = B[i, j]."""
    inv = np.empty_like(p)
    inv[p] = np.arange(p.size)
    return B[np.ix_(inv, inv)]


def shuffle(B, rng):
    """samplers.py:81-89: random relabelling; returns (shuffled, truth)."""
    p = rng.permutation(B.shape[0]).astype(np.intp)
    return relabel(np.asarray(B, dtype=np.float64), p), p


@dataclass(frozen=True)
class CsrGraph:
    """0/1 adjacency in CSR form (int32 indices; values implicit 1)."""

    n: int
    indptr: np.ndarray  # int64 [n+1]
    indices: np.ndarray  # int32 [nnz], sorted within each row

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    def to_dense(self, dtype=np.float64):
        M = np.zeros((self.n, self.n), dtype=dtype)
        rows = np.repeat(np.arange(self.n), np.diff(self.indptr))
        M[rows, self.indices] = 1
        return M

    def relabel(self, p):
        """Relabel vertices: v -> p[v] (same convention as ``relabel``)."""
        n = self.n
        rows = np.repeat(np.arange(n), np.diff(self.indptr))
        r2 = p[rows]
        c2 = p[self.indices]
        return _csr_from_coo(n, r2, c2)


def _csr_from_coo(n, rows, cols):
    order = np.lexsort((cols, rows))
    rows = rows[order]
    cols = cols[order].astype(np.int32)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    np.cumsum(indptr, out=indptr)
    return CsrGraph(n, indptr, cols)


def sparse_er_pair_csr(n, p, rho, config=5, replicate=0, block_rows=2000):
    """Config 5: undirected correlated sparse ER straight into CSR.

    Row block b (rows [b*block_rows, ...)) draws its upper-triangle slots from
    ``default_rng([config, replicate, b])`` with the samplers.py:60-65 law; the
    pair is mirrored to be symmetric and hollow.  The hidden permutation is
    drawn from ``default_rng([config, replicate])``.
    """
    ra, ca, rb, cb = [], [], [], []
    for b, r0 in enumerate(range(0, n, block_rows)):
        r1 = min(n, r0 + block_rows)
        rng = np.random.default_rng([config, replicate, b])
        U = rng.uniform(size=(r1 - r0, n))
        V = rng.uniform(size=(r1 - r0, n))
        a = U < p
        bb = np.where(a, V < p + rho * (1.0 - p), V < p * (1.0 - rho))
        cols = np.arange(n)[None, :]
        upper = cols > np.arange(r0, r1)[:, None]
        a &= upper
        bb &= upper
        i, j = np.nonzero(a)
        ra.append(i + r0); ca.append(j)
        i, j = np.nonzero(bb)
        rb.append(i + r0); cb.append(j)
    ra = np.concatenate(ra); ca = np.concatenate(ca)
    rb = np.concatenate(rb); cb = np.concatenate(cb)
    A = _csr_from_coo(n, np.concatenate([ra, ca]), np.concatenate([ca, ra]))
    B = _csr_from_coo(n, np.concatenate([rb, cb]), np.concatenate([cb, rb]))
    perm = np.random.default_rng([config, replicate]).permutation(n).astype(np.int64)
    return A, B.relabel(perm), perm


#: The five BASELINE.json configurations.
CONFIGS = {
    1: dict(n=100, kind="er", p=0.5, rho=0.9, precision="fp64", fw_tol=0.03),
    2: dict(n=1000, kind="directed_er", p=0.1, rho=0.8, precision="fp32", fw_tol=1e-2),
    3: dict(n=5000, kind="sbm", sizes=(2000, 2000, 1000), p_in=0.3, p_out=0.05,
            rho=0.7, precision="fp32", fw_tol=1e-2),
    4: dict(n=2000, kind="weighted", p=0.3, precision="fp32", fw_tol=1e-2),
    5: dict(n=40000, kind="sparse_er", p=0.01, rho=0.9, precision="fp32", fw_tol=1e-2),
}


def config_pair(config, replicate=0, n=None):
    """(A, Bs, truth) for a BASELINE config; ``n`` scales it down (tests)."""
    c = CONFIGS[config]
    n = int(n or c["n"])
    if c["kind"] == "sparse_er":
        A, Bs, truth = sparse_er_pair_csr(n, c["p"], c["rho"], config, replicate)
        return A, Bs, truth
    rng = np.random.default_rng([config, replicate])
    if c["kind"] == "er":
        A, B = correlated_er_pair(n, c["p"], c["rho"], rng)
    elif c["kind"] == "directed_er":
        A, B = directed_er_pair(n, c["p"], c["rho"], rng)
    elif c["kind"] == "sbm":
        sizes = np.asarray(c["sizes"], dtype=np.float64)
        sizes = np.maximum(1, np.round(sizes * n / sizes.sum())).astype(int)
        sizes[-1] = n - sizes[:-1].sum()
        k = len(sizes)
        probs = np.full((k, k), c["p_out"])
        np.fill_diagonal(probs, c["p_in"])
        A, B = correlated_sbm_pair(sizes, probs, c["rho"], rng)
    elif c["kind"] == "weighted":
        A, B = weighted_directed_pair(n, c["p"], rng)
    else:  # pragma: no cover
        raise ValueError(c["kind"])
    Bs, truth = shuffle(B, rng)
    return A, Bs, truth


def sparse_er_pair_csr_device(n, p, rho, seed=0, device="cuda", block_rows=2048):
    """Config-5 law (undirected correlated sparse ER, samplers.py:60-65 conditional
    law, hollow, mirrored) drawn on the GPU with torch's generator -- the bench's
    fast stand-in for ``sparse_er_pair_csr`` (same law, different random stream).

    Returns ((rowptr_A, col_A), (rowptr_B, col_B), truth) as CUDA tensors (int64
    rowptr, int32 columns, rows sorted) with B relabelled by the hidden permutation.
    """
    import torch

    g = torch.Generator(device=device).manual_seed(int(seed))
    ra, ca, rb, cb = [], [], [], []
    cols = torch.arange(n, device=device)
    for r0 in range(0, n, block_rows):
        r1 = min(n, r0 + block_rows)
        U = torch.rand((r1 - r0, n), generator=g, device=device)
        V = torch.rand((r1 - r0, n), generator=g, device=device)
        upper = cols[None, :] > torch.arange(r0, r1, device=device)[:, None]
        a = (U < p) & upper
        b = torch.where(U < p, V < p + rho * (1.0 - p), V < p * (1.0 - rho)) & upper
        i, j = torch.nonzero(a, as_tuple=True)
        ra.append(i + r0); ca.append(j)
        i, j = torch.nonzero(b, as_tuple=True)
        rb.append(i + r0); cb.append(j)
        del U, V, a, b, upper
    perm = torch.randperm(n, generator=g, device=device)

    def csr(r, c, relabel=None):
        r = torch.cat(r); c = torch.cat(c)
        r, c = torch.cat([r, c]), torch.cat([c, r])
        if relabel is not None:
            r, c = relabel[r], relabel[c]
        key, _ = torch.sort(r * n + c)
        r, c = key // n, (key % n).to(torch.int32)
        rowptr = torch.zeros(n + 1, dtype=torch.int64, device=device)
        rowptr[1:] = torch.cumsum(torch.bincount(r, minlength=n), 0)
        return rowptr, c.contiguous()

    return csr(ra, ca), csr(rb, cb, perm), perm
