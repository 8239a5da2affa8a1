"""Row-sharded LOT sweep at NCCL world 1: device time of each step of one sweep
(pass kernel + column-sum reduction, all-gather, merge) over `reps` sweeps, against the
unsharded persistent kernel on the same cost matrix.

usage: python scripts/prof_shard_sweep.py [n] [reps] [fp32|fp64]
"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
import numpy as np
import torch
import torch.distributed as dist
from paper_2111_05366_b200 import _lib, sharded

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="env://", device_id=torch.device("cuda", 0))
comm = sharded.Comm()
layout = sharded.ShardLayout(n, 1, 0)
be = sharded.GpuShardBackend(layout, prec)
# a setup is needed for the shard plan: tiny CSR (identity) is enough for the LOT primitives
import scipy.sparse as sp
I = sp.identity(n, format="csr")
rows = sharded._csr_rows_to_device(I, be.dev, be.dtype)
be.setup_csr(rows, None, rows, None)
G = torch.rand((layout.m_pad, layout.ld), dtype=be.dtype, device=be.dev) * 100
send = be.vec(n + 1); recv = be.vec(1, n + 1)
stream = torch.cuda.current_stream()


def timed(fn, k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(k):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / k


def begin():
    be.lot_begin(_lib.GOAT_MAXIMIZE, 100.0, 0.0, 100.0, 10 ** 6, 1e-300)


def sweep():
    be.lot_pass(G, send)
    comm.all_gather_rows(recv.view(-1), send)
    be.lot_merge(recv, 1)


begin(); sweep(); sweep()  # pre-check + first sweep (max-shift passes)
t_all = timed(sweep, reps)
begin(); sweep(); sweep()
t_pass = timed(lambda: be.lot_pass(G, send), reps)       # state does not advance without the merge: same pass repeated
t_gather = timed(lambda: comm.all_gather_rows(recv.view(-1), send), reps)
begin(); sweep(); sweep()
t_merge_seq = timed(lambda: (be.lot_pass(G, send), be.lot_merge(recv, 1)), reps) - t_pass
print(f"n={n} {prec} world=1: sweep {t_all*1e3:.1f} us = pass+colsum {t_pass*1e3:.1f} + all-gather {t_gather*1e3:.1f} "
      f"+ merge ~{t_merge_seq*1e3:.1f} us", flush=True)
dist.destroy_process_group()
