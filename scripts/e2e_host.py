"""Host-side cost of the public entry point at c2 (where e2e loses vs device time)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_05366_b200 as gb
from paper_2111_05366_b200 import graphs
from paper_2111_05366_b200.matrices import as_square_matrix
A, B, _ = graphs.config_pair(2, 0)
pA = torch.empty(A.shape, dtype=torch.float64, pin_memory=True).numpy(); pA[:] = A
pB = torch.empty(B.shape, dtype=torch.float64, pin_memory=True).numpy(); pB[:] = B
opts = gb.MatchOptions(step_solver="lot", precision="fp32")
gb.frank_wolfe_match(pA, pB, opts)
t = time.perf_counter(); [as_square_matrix(pA) for _ in range(20)]; print("as_square_matrix ms", (time.perf_counter() - t) / 20 * 1e3)
t = time.perf_counter()
for _ in range(5): r = gb.frank_wolfe_match(pA, pB, opts)
dt = (time.perf_counter() - t) / 5 * 1e3
print("frank_wolfe_match ms", dt, "device total ms", r.diagnostics["time_ms"]["total"], "setup", r.diagnostics["time_ms"]["setup"])
