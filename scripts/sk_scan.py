"""Per-sweep LOT time (goat_bench_sweep) over orders and planner knobs.

usage: python scripts/sk_scan.py OUT.json "n,prec,ENV=V;ENV2=V2" ...
Each case runs in its own process (env knobs are read at plan time).
"""
import json
import os
import subprocess
import sys

CODE = """
import ctypes, torch, sys
sys.path.insert(0, '.')
from paper_2111_05366_b200 import _lib
h = _lib.handle(0, '{prec}')
dt = torch.float32 if '{prec}' == 'fp32' else torch.float64
g = torch.Generator(device='cuda').manual_seed(0)
G = torch.rand(({n}, {n}), dtype=dt, device='cuda', generator=g) * 100
out = ctypes.c_double()
best = 1e30
for _ in range(3):
    _lib.check(_lib.load().goat_bench_sweep(h.ptr, {n}, G.data_ptr(), {n}, {sweeps}, ctypes.byref(out)))
    best = min(best, out.value)
print(best)
"""


def run(n, prec, env, sweeps):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", CODE.format(n=n, prec=prec, sweeps=sweeps)], env=e,
                       capture_output=True, text=True, timeout=600)
    try:
        return float(r.stdout.strip().splitlines()[-1]), (r.stderr.strip().splitlines() or [None])[-1]
    except Exception:
        return None, r.stderr[-400:]


def main():
    out = sys.argv[1]
    res = []
    for spec in sys.argv[2:]:
        parts = spec.split(",")
        n, prec = int(parts[0]), parts[1]
        env = dict(kv.split("=") for kv in parts[2].split(";")) if len(parts) > 2 and parts[2] else {}
        sweeps = 300 if n <= 5000 else 60
        ms, err = run(n, prec, env, sweeps)
        es = 4 if prec == "fp32" else 8
        gbs = n * n * es / (ms * 1e-3) / 1e9 if ms else None
        rec = dict(n=n, prec=prec, env=env, ms_per_sweep=ms, gbs=gbs, err=err)
        res.append(rec)
        print(json.dumps(rec), flush=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
