"""Compare each sharded LOT (world 1) with the oracle's lot on the same G."""
import os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from oracle import goat_oracle as O
from paper_2111_05366_b200.sharded import sharded_match
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_sharded_gpu import _er_pair
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
n = 100
A, B = _er_pair(n, 0.3, 0.8, False, 1)
tr = {}
r = sharded_match(A, B, precision="fp64", max_iters=8, trace=tr)
print("sharded sweeps", r.lot_sweeps, "alpha", r.hist_alpha)
otr = {}
a, hist, iters, conv = O.fw_core(A, B, None, np.full((n, n), 1.0 / n), trace=otr, max_iters=8)
print("oracle  sweeps", otr["sweeps"], "alpha", [h[2] for h in hist])
for i, (G, Q) in enumerate(zip(tr["G"], tr["Q"])):
    Qo, cv, sw, dv = O.lot(G, "maximize", 100.0, 1000, 1e-8)
    print(i, "sweeps oracle-on-sharded-G", sw, "maxdiff Q", np.abs(Q - Qo).max(), "rowsum", np.abs(Q.sum(1) - 1).max(), "colsum", np.abs(Q.sum(0) - 1).max())
dist.destroy_process_group()
