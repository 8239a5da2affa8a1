import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2111_05366_b200 as gb
from oracle import goat_oracle as O
sys.path.insert(0, "tests")
from test_lap_auction_gpu import _hub
for n, sense in [(2500, "maximize"), (2500, "minimize")]:
    rng = np.random.default_rng(n + 1)
    M = _hub(n, rng)
    for precision in ("fp64", "fp32"):
        Mp = M if precision == "fp64" else M.astype(np.float32).astype(np.float64)
        p, v = O.lap(Mp, sense)
        sol = gb.solve_lap(Mp, sense, precision=precision)
        ours = Mp[np.arange(n), sol.assignment].sum()
        print(n, sense, precision, "mismatch", int((sol.assignment != p).sum()), "scipy", repr(v), "ours", repr(ours),
              "diff", ours - v, flush=True)
