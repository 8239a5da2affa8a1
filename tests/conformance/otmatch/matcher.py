from paper_2111_05366_b200.engine import frank_wolfe_match, seeded_match  # noqa: F401
from paper_2111_05366_b200.ops import (exact_line_search, gradient, random_doubly_stochastic,  # noqa: F401
                                       randomized_blend_init)
from paper_2111_05366_b200.records import MatchOptions, MatchResult, SeedSet  # noqa: F401
from paper_2111_05366_b200.ops import relaxed_objective as _objective  # noqa: F401,E402
