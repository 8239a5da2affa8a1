"""Which sweeps of an fp32 LOT produce under/overflowing column sums (single GPU, sharded primitives)."""
import os, socket, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_2111_05366_b200.sharded import ShardLayout, GpuShardBackend, Comm
from paper_2111_05366_b200 import engine
from paper_2111_05366_b200.records import MatchOptions
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_sharded_gpu import _er_pair
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
for n, directed in [(1000, True), (2000, False)]:
    A, B = _er_pair(n, 0.1, 0.8, directed, n)
    lay = ShardLayout(n, 1, 0)
    be = GpuShardBackend(lay, "fp32")
    comm = Comm()
    AT = None if not directed else be.upload(A.T.copy(), lay.m_pad)
    be.setup(be.upload(A, lay.m_pad), AT, be.upload(B))
    P = be.block(); be.fill(1.0 / n, P)
    full = be.full(); comm.all_gather_rows(full, P)
    G = be.block(); be.gradient(full, G)
    send = be.vec(n + 1); recv = be.vec(1, n + 1)
    lo, hi = be.minmax(G)
    be.lot_begin(1, 100.0, lo, hi, 1000, 1e-8)
    last = 0
    for p in range(1003):
        st = be.lot_status()
        if st[4] != last:
            print(n, "pass", p - 1, "bad columns so far", st[4]); last = st[4]
        if st[0]: break
        be.lot_pass(G, send); comm.all_gather_rows(recv.view(-1), send); be.lot_merge(recv, 1)
    print(n, "final", be.lot_status())
dist.destroy_process_group()
