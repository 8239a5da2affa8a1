"""Config 5 (n = 40000 sparse correlated ER, fp32) on one B200: the unsharded
device path (goat_fw_core_device) for a few outer iterations, phase split,
per-iteration LOT sweeps, and the match ratio against the hidden permutation.

usage: python scripts/run_c5.py [max_iters] [n] [fp32|fp64] [csr|auto|simt]
(csr = goat_fw_core_csr_device, the SpMM gradient on the CSR graphs; the other
modes densify A and B and run goat_fw_core_device)
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

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n_arg = int(sys.argv[2]) if len(sys.argv) > 2 else None
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
tdt = torch.float32 if prec == "fp32" else torch.float64
gemm = sys.argv[4] if len(sys.argv) > 4 else "csr"
t0 = time.perf_counter()
A, Bs, truth = graphs.config_pair(5, 0, n=n_arg)
n = A.n
t_gen = time.perf_counter() - t0
dev = torch.device("cuda", 0)


def dense(g):
    rows = np.repeat(np.arange(g.n), np.diff(g.indptr))
    d = torch.zeros((g.n, g.n), dtype=tdt, device=dev)
    d[torch.from_numpy(rows).to(dev), torch.from_numpy(g.indices.astype(np.int64)).to(dev)] = 1.0
    return d


if gemm != "csr":
    dA, dB = dense(A), dense(Bs)
else:
    csr_t = [torch.from_numpy(x).to(dev) for x in (A.indptr, A.indices, Bs.indptr, Bs.indices)]
    sA, sB = _lib.csr_struct_device(csr_t[0], csr_t[1]), _lib.csr_struct_device(csr_t[2], csr_t[3])
torch.cuda.synchronize()
h = _lib.handle(0, prec, "auto" if gemm == "csr" else gemm)
lib = _lib.load()
_lib.check(lib.goat_set_stream(h.ptr, _lib.stream_handle(torch.cuda.current_stream(dev))))
assign = np.empty(n, dtype=np.int64)
hobj, halpha = np.empty(iters + 1), np.empty(iters + 1)
sweeps, lconv = np.zeros(iters, dtype=np.int32), np.zeros(iters, dtype=np.int32)
res = _lib.GoatFwResult()
res.assignment = assign.ctypes.data_as(_lib._c_i64_p)
res.hist_obj, res.hist_alpha = _lib.dptr(hobj), _lib.dptr(halpha)
res.lot_sweeps = sweeps.ctypes.data_as(_lib._c_i32_p)
res.lot_converged = lconv.ctypes.data_as(_lib._c_i32_p)
o = _lib.GoatOptions(max_iters=iters, max_sweeps=1000, sense=_lib.GOAT_MAXIMIZE, step_solver=_lib.GOAT_STEP_LOT,
                     fw_tol=1e-2, lam=100.0, sk_tol=1e-8)
t1 = time.perf_counter()
if gemm == "csr":
    _lib.check(lib.goat_fw_core_csr_device(h.ptr, n, ctypes.byref(sA), ctypes.byref(sB), None, n, None, n,
                                           ctypes.byref(o), ctypes.byref(res)))
else:
    _lib.check(lib.goat_fw_core_device(h.ptr, n, ctypes.c_void_p(dA.data_ptr()), n, ctypes.c_void_p(dB.data_ptr()),
                                       n, None, n, None, n, o, res))
wall = time.perf_counter() - t1
it = res.iterations
inv = np.empty(n, dtype=np.int64)
inv[assign] = np.arange(n)
print(json.dumps({
    "config": 5, "n": n, "precision": prec, "gemm": gemm, "max_iters": iters, "iterations": it, "converged": bool(res.converged),
    "wall_s": round(wall, 2), "gen_s": round(t_gen, 1),
    "phase_ms": dict(zip(("gradient", "lot", "line_search", "lap", "setup", "total"),
                         [round(x, 1) for x in res.time_ms])),
    "lot_sweeps": sweeps[:it].tolist(), "alpha": [round(float(a), 6) for a in halpha[1:it + 1]],
    "objective": res.objective, "lap_certified": bool(res.lap_certified),
    "match_ratio": max(float(np.mean(assign == truth)), float(np.mean(inv == truth))),
    "gpu_launches": res.gpu_launches}), flush=True)
