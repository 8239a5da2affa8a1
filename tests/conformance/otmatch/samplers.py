from paper_2111_05366_b200 import sample_er_pair, shuffle_pair  # noqa: F401
from paper_2111_05366_b200.graphs import SbmSpec, replicate_rng, sample_sbm_pair  # noqa: F401
