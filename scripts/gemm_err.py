"""fp32 tcgen05 gradient error vs split-K slice count (GOAT_TC_KSLICES)."""
import os, subprocess, sys
code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
import paper_2111_05366_b200 as gb
for n in (300, 1000, 3000):
    rng = np.random.default_rng(n)
    A = (rng.random((n, n)) < 0.3).astype(float)
    B = (rng.random((n, n)) < 0.3).astype(float)
    P = rng.random((n, n)); P /= P.sum(1, keepdims=True)
    G = A @ P @ B.T + A.T @ P @ B
    G32 = gb.gradient(A, B, P, precision="fp32")
    print(n, np.abs(G32 - G).max() / np.abs(G).max(), flush=True)
'''
for s in ("1", "2", "4", "8", "16"):
    env = dict(os.environ, GOAT_TC_KSLICES=s)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    print("slices", s, out.stdout.replace("\n", " | "), out.stderr[-300:], flush=True)
