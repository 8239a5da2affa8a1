"""B200-native GOAT iteration (arXiv 2111.05366) behind the ``otmatch`` API.

Drop-in names for the accelerated path (reference ``otmatch/__init__.py``):
``frank_wolfe_match``, ``seeded_match``, ``MatchOptions``, ``MatchResult``,
``SeedSet``, ``SinkhornParams``, ``SinkhornResult``, ``LapSolution``, ``lot``,
``sinkhorn_knopp``, ``gradient``, ``exact_line_search``, ``solve_lap``,
``qap_objective`` and the permutation helpers.  The compute runs in
``libgoat.so`` (hand-written sm_100a CUDA, C ABI in include/goat.h); there is
no CPU fallback.
"""

from .engine import fw_core, frank_wolfe_match, seeded_match
from .formats import (format_matrix_text, format_permutation_text, parse_matrix_text,
                      parse_permutation_text, pass_to_ranks)
from .graphs import (SbmSpec, correlated_er_pair, correlated_sbm_pair, replicate_rng, sample_sbm_pair,
                     shuffle as _shuffle)
from .matrices import (DS_TOL, as_doubly_stochastic, as_permutation, as_square_matrix,
                       barycenter, compose_permutations, edge_disagreements,
                       invert_permutation, match_ratio, permutation_matrix, permute_matrix,
                       qap_objective)
from .ops import (exact_line_search, gradient, lap_tie_set, lot, random_doubly_stochastic,
                  randomized_blend_init, sinkhorn_knopp, solve_lap)
from .records import (LapSolution, MatchOptions, MatchResult, SeedSet, SinkhornParams,
                      SinkhornResult)

__version__ = "0.1.0"


def sample_er_pair(n, p, rho, rng):
    """Correlated undirected ER pair (same law and RNG draws as samplers.py:75-78)."""
    return correlated_er_pair(n, p, rho, rng)


def shuffle_pair(B, rng):
    """Random relabelling (samplers.py:81-89): returns (shuffled, truth)."""
    return _shuffle(as_square_matrix(B, "B"), rng)


__all__ = [
    "DS_TOL", "LapSolution", "MatchOptions", "MatchResult", "SeedSet", "SinkhornParams",
    "SinkhornResult", "as_doubly_stochastic", "as_permutation", "as_square_matrix",
    "barycenter", "compose_permutations", "correlated_sbm_pair", "edge_disagreements",
    "exact_line_search", "frank_wolfe_match", "fw_core", "gradient", "invert_permutation",
    "lot", "match_ratio", "permutation_matrix", "permute_matrix", "qap_objective",
    "random_doubly_stochastic", "randomized_blend_init", "sample_er_pair", "seeded_match",
    "shuffle_pair", "sinkhorn_knopp", "solve_lap", "SbmSpec", "sample_sbm_pair", "replicate_rng",
    "lap_tie_set", "pass_to_ranks", "parse_matrix_text", "format_matrix_text", "parse_permutation_text",
    "format_permutation_text",
]
