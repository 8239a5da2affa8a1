from paper_2111_05366_b200.ops import TIE_SET_MAX_N, lap_tie_set, solve_lap  # noqa: F401
from paper_2111_05366_b200.records import LapSolution  # noqa: F401
