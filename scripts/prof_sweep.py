"""One persistent LOT launch (reps sweeps) over a random G: the ncu target."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_05366_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
h = _lib.handle(0, prec)
dt = torch.float32 if prec == "fp32" else torch.float64
G = torch.rand((n, n), dtype=dt, device="cuda") * 100
out = ctypes.c_double()
_lib.check(_lib.load().goat_bench_sweep(h.ptr, n, G.data_ptr(), n, reps, ctypes.byref(out)))
print(f"n={n} {prec} ms/sweep={out.value:.5f} GB/s={n*n*G.element_size()/out.value/1e6:.1f}")
