"""One CSR gradient at order n (config-5 law, device-drawn): the ncu target for spmm_t_kernel."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_05366_b200 import _lib, graphs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
dev = torch.device("cuda", 0)
(rA, cA), (rB, cB), perm = graphs.sparse_er_pair_csr_device(n, 0.01, 0.9, seed=5, device=dev)
sA, sB = _lib.csr_struct_device(rA, cA), _lib.csr_struct_device(rB, cB)
X = torch.rand((n, n), device=dev)
ms = ctypes.c_double()
h = _lib.handle(0, "fp32")
_lib.check(_lib.load().goat_bench_gradient_csr(h.ptr, n, ctypes.byref(sA), ctypes.byref(sB), X.data_ptr(), 1,
                                               ctypes.byref(ms)))
print(f"n={n} csr gradient ms={ms.value:.3f}")
