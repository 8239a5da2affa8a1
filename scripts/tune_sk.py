"""Per-sweep time of the LOT loop vs CTA count (GOAT_SK_BLOCKS), fp32/fp64."""
import ctypes, os, subprocess, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

def one(n, prec, blocks):
    env = dict(os.environ, GOAT_SK_BLOCKS=str(blocks))
    code = f"""
import ctypes, torch, sys
sys.path.insert(0, '.')
from paper_2111_05366_b200 import _lib
h = _lib.handle(0, '{prec}')
dt = torch.float32 if '{prec}' == 'fp32' else torch.float64
G = torch.rand(({n}, {n}), dtype=dt, device='cuda') * 100
out = ctypes.c_double()
_lib.check(_lib.load().goat_bench_sweep(h.ptr, {n}, G.data_ptr(), {n}, 300, ctypes.byref(out)))
print(out.value)
"""
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    try:
        return float(r.stdout.strip().splitlines()[-1])
    except Exception:
        return r.stderr[-300:]

res = {}
for n, prec in [(1000, "fp32"), (2000, "fp32"), (5000, "fp32"), (1000, "fp64")]:
    for b in [8, 16, 32, 64, 96, 148, 296]:
        ms = one(n, prec, b)
        es = 4 if prec == "fp32" else 8
        gbs = n * n * es / (ms * 1e-3) / 1e9 if isinstance(ms, float) else None
        res[f"{n}-{prec}-{b}"] = (ms, gbs)
        print(n, prec, b, ms, gbs, flush=True)
json.dump(res, open("gpurun_out/tune_sk.json", "w"), indent=1)
