"""Weighted (non-bf16-exact) directed gradient at n: all operands split into planes."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_05366_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
h = _lib.handle(0, "fp32")
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand((n, n), device="cuda", generator=g) * (torch.rand((n, n), device="cuda", generator=g) < 0.3)
B = torch.rand((n, n), device="cuda", generator=g) * (torch.rand((n, n), device="cuda", generator=g) < 0.3)
X = torch.rand((n, n), device="cuda", generator=g); X = X / X.sum(1, keepdim=True)
ms = ctypes.c_double(); p = ctypes.c_int32(); t = ctypes.c_int32()
for _ in range(2):
    _lib.check(_lib.load().goat_bench_gradient(h.ptr, n, A.data_ptr(), B.data_ptr(), X.data_ptr(), 3,
                                               ctypes.byref(ms), ctypes.byref(p), ctypes.byref(t)))
    print(f"n={n} weighted directed ms/gradient={ms.value:.3f} products={p.value}", flush=True)
