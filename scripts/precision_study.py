"""Precision study for fp32 mode at full-size config 3 (CPU, build container only).

Runs the reference algorithm (the oracle's restatement, float64) with fp32
rounding injected at chosen places, to find which roundings change the GOAT
trajectory (per-LOT sweeps, alpha) and the final permutation vs the unmodified
reference's golden (tests/golden/full_cases.npz):

  --round-g    round every gradient to fp32 before LOT and before the final LAP
  --round-q    round every LOT output Q (and hence P) to fp32
  --lot32      LOT potentials evaluated with fp32 exponent arguments (the fp32
               GPU kernel's element arithmetic) instead of float64

Not a test: a one-off measurement whose output is quoted in DESIGN.md §4.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import goat_oracle as O  # noqa: E402
from paper_2111_05366_b200 import graphs  # noqa: E402

torch.set_num_threads(os.cpu_count())


def lot64(G, lam=100.0, max_sweeps=1000, tol=1e-8, lot32=False):
    """sinkhorn.py:103-130 (maximize), standard domain in float64 via torch."""
    G = torch.from_numpy(G)
    shifted = G.max() - G
    scale = float(shifted.max())
    E = (-lam / scale) * shifted
    if lot32:
        return lot_log32(E.numpy(), max_sweeps, tol)
    K = torch.exp(E)
    rs, cs = K.sum(1), K.sum(0)
    dev = max(float((rs - 1).abs().max()), float((cs - 1).abs().max()))
    if dev < tol:
        return K.numpy(), 0, dev
    v = torch.ones(K.shape[0], dtype=torch.float64)
    Kv = K @ v
    KT = K.t().contiguous()
    for s in range(1, max_sweeps + 1):
        u = 1.0 / Kv
        v = 1.0 / (KT @ u)
        Kv = K @ v
        dev = float((u * Kv - 1.0).abs().max())
        if dev < tol:
            break
    return (u[:, None] * K * v[None, :]).numpy(), s, dev


def lot_log32(E, max_sweeps, tol):
    """Log-domain sweeps with the GPU fp32 kernel's element arithmetic: the
    exponent argument E_ij + g_j - shift is formed in fp32, exp in fp32, sums fp64."""
    E32 = torch.from_numpy(E.astype(np.float32))
    n = E.shape[0]
    f = torch.zeros(n, dtype=torch.float64)
    g = torch.zeros(n, dtype=torch.float64)
    fprev = None
    dev = np.inf
    for s in range(1, max_sweeps + 2):
        X = E32 + g.float()[None, :]
        m = X.max(1).values
        fnew = -(m.double() + torch.log(torch.exp(X - m[:, None]).double().sum(1)))
        if fprev is not None:
            dev = float(torch.expm1(fprev - fnew).abs().max())
            if dev < tol or s == max_sweeps + 1:
                sw = s - 1
                break
        Y = E32 + fnew.float()[:, None]
        mc = Y.max(0).values
        g = -(mc.double() + torch.log(torch.exp(Y - mc[None, :]).double().sum(0)))
        fprev, gprev = fnew, g
    Q = torch.exp(torch.from_numpy(E) + fprev[:, None] + gprev[None, :])
    return Q.numpy(), sw, dev


def run(A, B, round_g, round_q, lot32, max_iters=30, fw_tol=1e-2, g_noise=0.0, g_trunc=0, final_exact=False):
    n = A.shape[0]
    At, Bt = torch.from_numpy(A), torch.from_numpy(B)
    rng = np.random.default_rng(1)

    def grad(P, final=False):
        Pt = torch.from_numpy(P)
        G = (At @ Pt @ Bt.t() + At.t() @ Pt @ Bt).numpy()
        if final and final_exact:  # the LAP input formed in float64 from the (rounded) iterate
            return G
        if g_noise:  # a gradient accurate to g_noise * max|G| (e.g. a split-bf16 tensor-core product)
            G = G + g_noise * np.abs(G).max() * rng.standard_normal(G.shape)
        if g_trunc:  # the iterate cut to g_trunc mantissa bits before the product (bf16 planes)
            m, e = np.frexp(P)
            Pc = np.ldexp(np.trunc(m * 2.0 ** g_trunc) / 2.0 ** g_trunc, e)
            Pc = torch.from_numpy(Pc)
            G = (At @ Pc @ Bt.t() + At.t() @ Pc @ Bt).numpy()
        return G.astype(np.float32).astype(np.float64) if round_g else G

    def rel(P):
        Pt = torch.from_numpy(P)
        return float((At.t() @ Pt @ Bt * Pt).sum())

    P = np.full((n, n), 1.0 / n)
    sweeps, alphas = [], []
    for i in range(1, max_iters + 1):
        G = grad(P)
        Q, sw, dev = lot64(G, lot32=lot32)
        if round_q:
            Q = Q.astype(np.float32).astype(np.float64)
        sweeps.append(sw)
        D = torch.from_numpy(P - Q)
        Qt = torch.from_numpy(Q)
        ADB = At.t() @ D @ Bt
        c2 = float((ADB * D).sum())
        c1 = float((ADB * Qt).sum() + (At.t() @ Qt @ Bt * D).sum())
        a = O.best_alpha(c2, c1, "maximize")
        alphas.append(a)
        Pn = a * P + (1 - a) * Q
        step = float(np.linalg.norm(Pn - P))
        P = Pn
        print(f"  it {i}: sweeps {sw} dev {dev:.3e} alpha {a} step {step:.4f}", flush=True)
        if step < fw_tol:
            break
    G = grad(P, final=True)
    p, _ = O.lap(G, "maximize")
    return p, sweeps, alphas, O.qap_objective_perm(A, B, p)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--round-g", action="store_true")
    ap.add_argument("--round-q", action="store_true")
    ap.add_argument("--lot32", action="store_true")
    ap.add_argument("--g-noise", type=float, default=0.0)
    ap.add_argument("--g-trunc", type=int, default=0)
    ap.add_argument("--final-exact", action="store_true")
    args = ap.parse_args()
    A, B, _ = graphs.config_pair(args.config, 0)
    z = np.load(os.path.join(ROOT, "tests/golden/full_cases.npz"))
    key = f"c{args.config}_full"
    t0 = time.time()
    p, sw, al, obj = run(A, B, args.round_g, args.round_q, args.lot32, g_noise=args.g_noise, g_trunc=args.g_trunc, final_exact=args.final_exact)
    same = np.array_equal(p, z[f"{key}/alignment"])
    print(f"config {args.config} round_g={args.round_g} round_q={args.round_q} lot32={args.lot32} "
          f"g_noise={args.g_noise} g_trunc={args.g_trunc} final_exact={args.final_exact}: "
          f"sweeps {sw} (ref {z[f'{key}/lot_sweeps'].tolist()}) alpha {al} obj {obj} "
          f"(ref {float(z[f'{key}/objective'])}) same_perm={same} "
          f"perm_agree={np.mean(p == z[f'{key}/alignment']):.4f} {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
