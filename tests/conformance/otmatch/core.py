from paper_2111_05366_b200.formats import *  # noqa: F401,F403
from paper_2111_05366_b200.matrices import *  # noqa: F401,F403
from paper_2111_05366_b200.matrices import DS_TOL  # noqa: F401
