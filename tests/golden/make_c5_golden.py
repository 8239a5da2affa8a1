"""Oracle run of config 5 scaled to n = 4000 (graphs.config_pair(5, 0, n=4000)):
the oracle restatement (oracle/goat_oracle.py, pinned against the reference's
own outputs by tests/test_oracle.py) at full float64, GOAT defaults, 4 outer
iterations.  Writes c5_n4000.npz; ~1 minute on CPU."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import numpy as np

from oracle import goat_oracle as O
from paper_2111_05366_b200 import graphs

n = 4000
A, Bs, truth = graphs.config_pair(5, 0, n=n)
Ad, Bd = A.to_dense(), Bs.to_dense()
tr = {}
a, hist, iters, conv = O.fw_core(Ad, Bd, None, np.full((n, n), 1.0 / n), trace=tr, max_iters=4)
np.savez_compressed(os.path.join(HERE, "c5_n4000.npz"), assignment=np.asarray(a, dtype=np.int32),
                    alpha=np.array([h[2] for h in hist[1:]]), obj=np.array([h[1] for h in hist]),
                    sweeps=np.array(tr["sweeps"]), iterations=iters, converged=conv,
                    objective=O.qap_objective_perm(Ad, Bd, a))
print("iterations", iters, "sweeps", tr["sweeps"], "objective", O.qap_objective_perm(Ad, Bd, a))
