"""CSR gradient (SpMM) vs the dense tcgen05 gradient on BASELINE config 5.

usage: python scripts/prof_spmm.py [n] [reps]   (default n = 40000)
Prints ms per gradient for the CSR path (goat_bench_gradient_csr) and, when
memory allows, the dense tcgen05 path (goat_bench_gradient) on the same graphs.
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2111_05366_b200 import _lib, graphs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dense_too = n <= 20000 or os.environ.get("DENSE", "0") == "1"
t0 = time.perf_counter()
A, Bs, truth = graphs.config_pair(5, 0, n=n)
t_gen = time.perf_counter() - t0
dev = torch.device("cuda", 0)
lib = _lib.load()
h = _lib.handle(0, "fp32")
rA, cA = torch.from_numpy(A.indptr).to(dev), torch.from_numpy(A.indices).to(dev)
rB, cB = torch.from_numpy(Bs.indptr).to(dev), torch.from_numpy(Bs.indices).to(dev)
sA, sB = _lib.csr_struct_device(rA, cA), _lib.csr_struct_device(rB, cB)
g = torch.Generator(device=dev).manual_seed(0)
X = torch.rand((n, n), device=dev, generator=g)
X /= X.sum(1, keepdim=True)
ms = ctypes.c_double()
_lib.check(lib.goat_bench_gradient_csr(h.ptr, n, ctypes.byref(sA), ctypes.byref(sB), X.data_ptr(), reps,
                                       ctypes.byref(ms)))
nnz = int(A.indices.size) + int(Bs.indices.size)
# algorithmic traffic of the two gathers: every nonzero reads one row of the dense operand
gather_bytes = (A.indices.size + Bs.indices.size) * n * 4
out = dict(n=n, nnz_A=int(A.indices.size), nnz_B=int(Bs.indices.size), gen_s=round(t_gen, 1),
           csr_ms=ms.value, csr_gather_TBps=gather_bytes / (ms.value * 1e-3) / 1e12,
           csr_useful_TFLOPs=2 * 2.0 * (nnz / 2) * n / (ms.value * 1e-3) / 1e12)
if dense_too:
    dA = torch.zeros((n, n), device=dev)
    dB = torch.zeros((n, n), device=dev)
    rows = torch.from_numpy(np.repeat(np.arange(n), np.diff(A.indptr))).to(dev)
    dA[rows, cA.long()] = 1.0
    rows = torch.from_numpy(np.repeat(np.arange(n), np.diff(Bs.indptr))).to(dev)
    dB[rows, cB.long()] = 1.0
    msd = ctypes.c_double(); prods = ctypes.c_int32(); terms = ctypes.c_int32()
    hd = _lib.handle(0, "fp32", "tcgen05")
    _lib.check(lib.goat_bench_gradient(hd.ptr, n, dA.data_ptr(), dB.data_ptr(), X.data_ptr(), reps,
                                       ctypes.byref(msd), ctypes.byref(prods), ctypes.byref(terms)))
    out.update(dense_tc_ms=msd.value, speedup=msd.value / ms.value)
print(json.dumps(out), flush=True)
