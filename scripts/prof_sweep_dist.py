"""Per-sweep time of the persistent LOT kernel at order n for several value distributions of G
(goat_bench_sweep: E = G - 100 in [-100, 0]): is the sweep time data dependent?"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_05366_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
h = _lib.handle(0, "fp32")
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(0)


def run(name, G):
    out = ctypes.c_double()
    torch.cuda.synchronize()
    _lib.check(lib.goat_bench_sweep(h.ptr, n, G.data_ptr(), n, reps, ctypes.byref(out)))
    print(f"{name:28s} ms/sweep={out.value:.4f} GB/s={n*n*4/out.value/1e6:.0f}", flush=True)


G = torch.rand((n, n), device="cuda", generator=g) * 100
run("uniform [0,100)", G)
G.zero_()
run("all zero", G)
G = torch.rand((n, n), device="cuda", generator=g)
G = (G < 0.001).float() * 100
run("0.1% entries at 100, rest 0", G)
G = torch.rand((n, n), device="cuda", generator=g)
G.pow_(16).mul_(100)
run("100 * u^16 (skewed)", G)
d1 = torch.rand(n, device="cuda", generator=g); d2 = torch.rand(n, device="cuda", generator=g)
G = torch.outer(d1, d2) * 100
run("rank-1 outer product", G)
G = torch.rand((n, n), device="cuda", generator=g) * 1e-3 + 99.0
run("near-tied: 99 + 1e-3 u", G)
