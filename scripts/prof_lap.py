"""One device LAP (auction + price tightening + repair) on a hub-dominated n x n cost: the ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2111_05366_b200 as gb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
rng = np.random.default_rng(n)
d1, d2 = rng.gamma(2.0, 1.0, n), rng.gamma(2.0, 1.0, n)
M = np.outer(d1, d2) + 1e-3 * rng.random((n, n))
sol = gb.solve_lap(M, "maximize", precision="fp32")
print("n", n, "objective", sol.objective)
