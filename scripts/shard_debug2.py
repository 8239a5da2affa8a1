"""Run sharded LOT primitives by hand on a given G; print per-pass state."""
import os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from oracle import goat_oracle as O
from paper_2111_05366_b200.sharded import sharded_match, ShardLayout, GpuShardBackend, Comm
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_sharded_gpu import _er_pair
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
n = 100
A, B = _er_pair(n, 0.3, 0.8, False, 1)
tr = {}
r = sharded_match(A, B, precision="fp64", max_iters=6, trace=tr)
lay = ShardLayout(n, 1, 0)
be = GpuShardBackend(lay, "fp64")
comm = Comm()
be.setup(be.upload(A, lay.m_pad), None, be.upload(B))
send = be.vec(n + 1); recv = be.vec(1, n + 1)
def run(Gnp, label, maxp=1003, verbose=10):
    G = be.upload(Gnp, lay.m_pad)
    lo, hi = be.minmax(G)
    be.lot_begin(1, 100.0, lo, hi, 1000, 1e-8)
    for p in range(maxp):
        st = be.lot_status()
        if st[0]: break
        be.lot_pass(G, send)
        comm.all_gather_rows(recv.view(-1), send)
        s0 = send.cpu().numpy().copy()
        be.lot_merge(recv, 1)
        if p < verbose: print(label, "pass", p, "send dev", s0[n], "colsum[:3]", s0[:3], "status", be.lot_status())
    print(label, "final", be.lot_status())
    Q = be.block(); be.lot_emit(G, Q)
    Qo, cv, sw, dv = O.lot(Gnp, "maximize", 100.0, 1000, 1e-8)
    print(label, "oracle sweeps", sw, "maxdiff", np.abs(Q.cpu().numpy()[:n, :n] - Qo).max())
run(tr["G"][4], "fresh-G4")
run(tr["G"][3], "G3", verbose=3)
run(tr["G"][4], "after-G3-G4")
dist.destroy_process_group()
