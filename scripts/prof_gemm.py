"""One tcgen05 gradient at order n (symmetric 0/1 inputs): the ncu target."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_05366_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
sym = (sys.argv[2] == "sym") if len(sys.argv) > 2 else True
h = _lib.handle(0, "fp32")
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.rand((n, n), device="cuda", generator=g) < 0.3).float()
B = (torch.rand((n, n), device="cuda", generator=g) < 0.3).float()
if sym:
    A = torch.triu(A, 1); A = A + A.T; B = torch.triu(B, 1); B = B + B.T
X = torch.rand((n, n), device="cuda", generator=g); X = X / X.sum(1, keepdim=True)
ms = ctypes.c_double(); p = ctypes.c_int32(); t = ctypes.c_int32()
_lib.check(_lib.load().goat_bench_gradient(h.ptr, n, A.data_ptr(), B.data_ptr(), X.data_ptr(), 2,
                                           ctypes.byref(ms), ctypes.byref(p), ctypes.byref(t)))
print(f"n={n} sym={sym} ms/gradient={ms.value:.3f} products={p.value} terms={t.value} "
      f"useful TFLOP/s={p.value*2*n**3/ms.value/1e9:.1f}")
