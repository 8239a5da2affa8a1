"""Input conditioning and the text formats either side of the GOAT path
(SURVEY.md §8f rank 4): ``pass_to_ranks`` (core.py:166-184) and the matrix /
permutation text formats of the reference CLI (core.py:189-229).  Host-only
O(n^2) glue; the same error contract (ValueError with the same conditions)."""

from __future__ import annotations

import numpy as np

from .matrices import as_permutation, as_square_matrix

__all__ = ["pass_to_ranks", "parse_matrix_text", "format_matrix_text", "parse_permutation_text",
           "format_permutation_text"]


def _average_ranks(values: np.ndarray) -> np.ndarray:
    """1-based ranks with ties sharing their mean rank (scipy rankdata 'average')."""
    order = np.argsort(values, kind="mergesort")
    sorted_v = values[order]
    # boundaries of runs of equal values
    start = np.flatnonzero(np.concatenate(([True], sorted_v[1:] != sorted_v[:-1])))
    end = np.concatenate((start[1:], [values.size]))
    mean_rank = (start + 1 + end) / 2.0  # mean of start+1 .. end
    ranks = np.empty(values.size, dtype=np.float64)
    ranks[order] = np.repeat(mean_rank, end - start)
    return ranks


def pass_to_ranks(W) -> np.ndarray:
    """Nonzero weights -> average rank / (nnz + 1) in (0, 1); zeros stay zero
    (core.py:166-184).  Invariant under strictly monotone reweighting."""
    W = as_square_matrix(W, "W")
    if W.size and W.min() < 0:
        raise ValueError("pass_to_ranks requires nonnegative weights")
    out = np.zeros_like(W)
    nz = W != 0
    count = int(nz.sum())
    if count:
        out[nz] = _average_ranks(W[nz]) / (count + 1)
    return out


def parse_matrix_text(text: str) -> np.ndarray:
    """``n`` then n*n row-major entries, whitespace separated (core.py:189-208)."""
    tok = text.split()
    if not tok:
        raise ValueError("empty matrix text")
    try:
        n = int(tok[0])
    except ValueError:
        raise ValueError(f"expected integer order, got {tok[0]!r}") from None
    if n < 1:
        raise ValueError(f"order must be positive, got {n}")
    if len(tok) - 1 != n * n:
        raise ValueError(f"expected {n * n} entries, found {len(tok) - 1}")
    try:
        vals = np.array([float(t) for t in tok[1:]], dtype=np.float64)
    except ValueError as e:
        raise ValueError(f"non-numeric matrix entry: {e}") from None
    return as_square_matrix(vals.reshape(n, n))


def format_matrix_text(M) -> str:
    """Inverse of ``parse_matrix_text``; entries printed with repr (round-trips float64)."""
    M = as_square_matrix(M)
    rows = [" ".join(repr(v) for v in r) for r in M.tolist()]
    return "\n".join([str(M.shape[0]), *rows]) + "\n"


def parse_permutation_text(text: str) -> np.ndarray:
    """n whitespace-separated 0-based indices (core.py:217-224)."""
    try:
        p = np.array([int(t) for t in text.split()], dtype=np.intp)
    except ValueError as e:
        raise ValueError(f"non-integer permutation entry: {e}") from None
    return as_permutation(p)


def format_permutation_text(p) -> str:
    return " ".join(str(int(i)) for i in as_permutation(p)) + "\n"
