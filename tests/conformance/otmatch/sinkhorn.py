from paper_2111_05366_b200.ops import lot, sinkhorn_knopp  # noqa: F401
from paper_2111_05366_b200.records import SinkhornParams, SinkhornResult  # noqa: F401
