"""fp32 tcgen05 gradient: error vs promotion chunk (GOAT_TC_CHUNK) and time at n=5000."""
import os, subprocess, sys
code = r'''
import numpy as np, sys, ctypes, time
sys.path.insert(0, ".")
import paper_2111_05366_b200 as gb
for n in (300, 1000, 3000):
    rng = np.random.default_rng(n)
    A = (rng.random((n, n)) < 0.3).astype(float)
    B = (rng.random((n, n)) < 0.3).astype(float)
    P = rng.random((n, n)); P /= P.sum(1, keepdims=True)
    G = A @ P @ B.T + A.T @ P @ B
    G32 = gb.gradient(A, B, P, precision="fp32")
    print(n, "%.2e" % (np.abs(G32 - G).max() / np.abs(G).max()), flush=True)
'''
for c in ("1", "2", "4", "8", "32"):
    env = dict(os.environ, GOAT_TC_CHUNK=c)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    t = subprocess.run([sys.executable, "scripts/prof_gemm.py", "5000", "sym"], env=env, capture_output=True, text=True, timeout=600)
    t2 = subprocess.run([sys.executable, "scripts/prof_gemm.py", "2000", "dir"], env=env, capture_output=True, text=True, timeout=600)
    print("chunk", c, out.stdout.replace("\n", " | "), out.stderr[-300:], "||", t.stdout.strip(), t.stderr[-300:], "||", t2.stdout.strip(), flush=True)
