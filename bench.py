"""GOAT iteration benchmark (BASELINE.json metric: outer iterations/s and
time-to-converge; Sinkhorn HBM GB/s).

One *step* = one complete GOAT solve (``_fw_core``: every outer iteration plus
the final exact LAP) of the BASELINE config-2 workload -- n=1000 directed
correlated ER pair, p=0.1, rho=0.8, fp32, barycenter init, maxiter=30 --
on a seeded synthetic input.  ``value`` = outer iterations per second over the
timed steps with inputs already resident in HBM (goat_fw_core_device);
``e2e`` = the same metric through the public API (frank_wolfe_match on pinned
host float64 arrays, host<->device copies inside the timed region).

Multi-GPU: config 2 does not shard (n=1000 fits L2); N ranks run N independent
replicas (replicate r = rank), weak scaling, max-over-ranks device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = 2
WORKLOAD = "c2: n=1000 directed correlated ER p=0.1 rho=0.8, fp32, barycenter init, maxiter=30"
METRIC = "goat_outer_iters_per_sec"


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _sample(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                  "--format=csv,noheader,nounits"], capture_output=True,
                                 text=True, timeout=5).stdout.strip()
            if out:
                self.rows.append([x.strip() for x in out.split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        self._sample()  # the state right at the end of the timed region

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for name, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def _inputs(replicate):
    from paper_2111_05366_b200 import graphs
    A, Bs, truth = graphs.config_pair(CONFIG, replicate)
    return A, Bs, truth


def _opts():
    import paper_2111_05366_b200 as gb
    return gb.MatchOptions(step_solver="lot", precision="fp32", max_iters=30)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def cpu_baseline(A, B, budget_s=12.0):
    """The CPU oracle (numpy port of the reference path) on the same input."""
    from oracle import goat_oracle as O
    cores = len(os.sched_getaffinity(0))
    iters = 0
    t0 = time.perf_counter()
    solves = 0
    while True:
        _, _, it, _, _ = O.run_seeded(A, B, np.empty((0, 2)), step_solver="lot")
        iters += it
        solves += 1
        if time.perf_counter() - t0 > budget_s or solves >= 8:
            break
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "iter/s", "cores": cores, "kind": "port",
            "sample": f"{solves} full c2 solves (n=1000, float64 numpy/OpenBLAS + scipy LSAP), "
                      f"{iters} outer iterations in {dt:.1f}s",
            "time_to_converge_ms": 1000.0 * dt / solves}


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return
    A, B, _ = _inputs(0)
    from oracle import goat_oracle as O
    for _ in range(max(0, min(args.warmup, 1))):
        O.run_seeded(A, B, np.empty((0, 2)), step_solver="lot")
    iters = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _, _, it, _, _ = O.run_seeded(A, B, np.empty((0, 2)), step_solver="lot")
        iters += it
    dt = time.perf_counter() - t0
    cores = len(os.sched_getaffinity(0))
    v = iters / dt
    line = {"metric": METRIC, "value": v, "unit": "iter/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * dt / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": WORKLOAD, "replicates": 1},
            "cpu_baseline": {"value": v, "unit": "iter/s", "cores": cores, "kind": "port",
                             "sample": f"{args.steps} full c2 solves of the oracle port "
                                       f"(oracle/goat_oracle.py, float64, all host threads)"},
            "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = _dist()
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    import paper_2111_05366_b200 as gb
    from paper_2111_05366_b200 import _lib

    A, B, truth = _inputs(rank)
    n = A.shape[0]
    opts = gb.MatchOptions(step_solver="lot", precision="fp32", max_iters=30, device=local)
    h = _lib.handle(local, "fp32")
    lib = _lib.load()
    stream = torch.cuda.current_stream(dev)
    _lib.check(lib.goat_set_stream(h.ptr, _lib.stream_handle(stream)))

    dA = torch.from_numpy(A.astype(np.float32)).to(dev)
    dB = torch.from_numpy(B.astype(np.float32)).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > L2

    phases = {}

    def device_step():
        mi = opts.max_iters
        assign = np.empty(n, dtype=np.int64)
        hobj = np.empty(mi + 1)
        halpha = np.empty(mi + 1)
        sweeps = np.zeros(mi, dtype=np.int32)
        res = _lib.GoatFwResult()
        res.assignment = assign.ctypes.data_as(_lib._c_i64_p)
        res.hist_obj = _lib.dptr(hobj)
        res.hist_alpha = _lib.dptr(halpha)
        res.lot_sweeps = sweeps.ctypes.data_as(_lib._c_i32_p)
        o = _lib.GoatOptions(max_iters=mi, max_sweeps=1000, sense=_lib.GOAT_MAXIMIZE,
                             step_solver=_lib.GOAT_STEP_LOT, fw_tol=opts.fw_tol, lam=100.0,
                             sk_tol=1e-8)
        _lib.check(lib.goat_fw_core_device(h.ptr, n, dA.data_ptr(), n, dB.data_ptr(), n, None, n,
                                           None, n, o, res))
        phases.clear()
        phases.update(zip(("gradient", "lot", "line_search", "lap", "setup", "total"),
                          [round(x, 3) for x in res.time_ms]))
        phases["lot_sweeps"] = sweeps[: int(res.iterations)].tolist()
        return int(res.iterations), int(res.gpu_launches), assign, float(res.objective)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(3, args.warmup)):
        device_step()
    # ---- timed: device-resident inputs
    iters = 0
    launches = 0
    ms_steps = []
    with ClockSampler(local) as clocks:
        barrier()
        for _ in range(args.steps):
            flush.zero_()  # evict L2 between steps (inputs are L2-sized)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            it, nl, assign, obj = device_step()
            e1.record(stream)
            e1.synchronize()
            ms_steps.append(e0.elapsed_time(e1))
            iters += it
            launches += nl
        barrier()
    total_ms = sum(ms_steps)
    match = float(np.mean(assign == truth))

    # ---- e2e through the public API, pinned host float64 inputs
    pA = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
    pB = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
    pA[:] = A
    pB[:] = B
    gb.frank_wolfe_match(pA, pB, opts)  # warm the host path
    e2e_ms = []
    e2e_iters = 0
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = gb.frank_wolfe_match(pA, pB, opts)
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
        e2e_iters += r.iterations
    barrier()

    # ---- roofline: the fused Sinkhorn sweep kernel (dominant), live CUDA events
    G = torch.rand((n, n), dtype=torch.float32, device=dev) * 100.0
    msw = _ms_per_sweep(lib, h, n, G)
    bytes_per_sweep = n * n * 4
    achieved = bytes_per_sweep / (msw * 1e-3) / 1e9
    peak, peak_kind = _peaks()
    kernels = _kernel_scan(lib, h, dev, peak)
    traffic = None
    try:  # measured DRAM bytes per sweep of this kernel (one ncu --set full capture)
        with open(os.path.join(ROOT, "profiles", "round1_ncu_traffic.json")) as f:
            traffic = json.load(f)["sk_tile_kernel_n1000_fp32"]["bytes_per_sweep"]
    except Exception:
        traffic = None

    if world > 1:
        t = torch.tensor([total_ms, float(iters), sum(e2e_ms), float(e2e_iters)], dtype=torch.float64, device=dev)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        total_max = max(float(x[0]) for x in allt)
        iters_all = sum(float(x[1]) for x in allt)
        e2e_max = max(float(x[2]) for x in allt)
        e2e_iters_all = sum(float(x[3]) for x in allt)
    else:
        total_max, iters_all = total_ms, float(iters)
        e2e_max, e2e_iters_all = sum(e2e_ms), float(e2e_iters)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    c5 = _c5_solve(lib, dev) if os.environ.get("GOAT_BENCH_C5", "1") != "0" else None
    cpu = cpu_baseline(A, B)
    line = {
        "metric": METRIC, "value": iters_all / (total_max / 1000.0), "unit": "iter/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": total_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n": n, "replicates_per_gpu": 1,
                   "l2": "flushed between steps (256 MiB write); inputs 4 MB are L2-sized",
                   "iterations_per_step": iters / args.steps, "match_ratio": match,
                   "time_to_converge_ms": total_max / args.steps,
                   "phase_ms_last_step": phases,
                   "parallelism": f"replicas x{world}"},
        "e2e": {"value": e2e_iters_all / (e2e_max / 1000.0), "unit": "iter/s",
                "h2d_bytes_per_step": 2 * n * n * 8, "d2h_bytes_per_step": n * 8 + 8 * 2 * 31,
                "time_to_converge_ms": e2e_max / args.steps},
        "roofline": {"kernel": "sk_tile_kernel (persistent log-domain Sinkhorn LOT, one read of G per sweep)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_kind": peak_kind, "traffic": traffic,
                     "note": f"{bytes_per_sweep} algorithmic bytes per sweep (n^2 fp32, one read of G), "
                             f"{msw * 1000:.2f} us per sweep; at n=1000 the G tiles stay in shared memory "
                             f"for the whole LOT, so the sweep is latency-bound (one grid barrier, one "
                             f"DSMEM row exchange, one L2 column merge), not HBM-bound"},
        "cpu_baseline": {k: v for k, v in cpu.items()},
        "kernels": kernels,
        "c5": c5,
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _c5_solve(lib, dev):
    """BASELINE config 5 (n = 40000 sparse correlated ER, p = 0.01, rho = 0.9, fp32,
    maxiter = 30) on this GPU through the CSR path: one full solve, inputs drawn on
    the device (graphs.sparse_er_pair_csr_device).  The north star's target is the
    outer-iteration time at this size; reported beside the c2 headline."""
    import ctypes
    import torch
    from paper_2111_05366_b200 import _lib, graphs
    n = 40000
    (rA, cA), (rB, cB), perm = graphs.sparse_er_pair_csr_device(n, 0.01, 0.9, seed=5, device=dev)
    sA, sB = _lib.csr_struct_device(rA, cA), _lib.csr_struct_device(rB, cB)
    h = _lib.handle(dev.index, "fp32")
    _lib.check(lib.goat_set_stream(h.ptr, _lib.stream_handle(torch.cuda.current_stream(dev))))
    mi = 30
    assign = np.empty(n, dtype=np.int64)
    hobj, halpha = np.empty(mi + 1), np.empty(mi + 1)
    sweeps = np.zeros(mi, dtype=np.int32)
    res = _lib.GoatFwResult()
    res.assignment = assign.ctypes.data_as(_lib._c_i64_p)
    res.hist_obj, res.hist_alpha = _lib.dptr(hobj), _lib.dptr(halpha)
    res.lot_sweeps = sweeps.ctypes.data_as(_lib._c_i32_p)
    o = _lib.GoatOptions(max_iters=mi, max_sweeps=1000, sense=_lib.GOAT_MAXIMIZE,
                         step_solver=_lib.GOAT_STEP_LOT, fw_tol=1e-2, lam=100.0, sk_tol=1e-8)
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.goat_fw_core_csr_device(h.ptr, n, ctypes.byref(sA), ctypes.byref(sB), None, n, None, n,
                                           ctypes.byref(o), ctypes.byref(res)))
    e1.record()
    e1.synchronize()
    it = int(res.iterations)
    ph = dict(zip(("gradient", "lot", "line_search", "lap", "setup", "total"), [round(x, 1) for x in res.time_ms]))
    truth = perm.cpu().numpy()
    out = {"workload": "c5: n=40000 sparse correlated ER p=0.01 rho=0.9, CSR adjacency (nnz %d + %d), fp32, "
                       "barycenter init, maxiter=30, one GPU" % (cA.numel(), cB.numel()),
           "time_to_converge_ms": e0.elapsed_time(e1), "iterations": it, "converged": bool(res.converged),
           "outer_iteration_ms": (ph["gradient"] + ph["lot"] + ph["line_search"]) / max(1, it),
           "phase_ms": ph, "lot_sweeps": sweeps[:it].tolist(), "objective": float(res.objective),
           "match_ratio": max(float(np.mean(assign == truth)), float(np.mean(truth[assign] == np.arange(n)))),
           "gpu_launches": int(res.gpu_launches)}
    del rA, cA, rB, cB
    torch.cuda.empty_cache()
    return out


def _ms_per_sweep(lib, h, n, G, reps=200):
    import ctypes
    from paper_2111_05366_b200 import _lib
    out = ctypes.c_double()
    _lib.check(lib.goat_bench_sweep(h.ptr, n, G.data_ptr(), n, reps, ctypes.byref(out)))
    return out.value


def _bf16_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), "measured"
    except Exception:
        return 1590.0, "fallback"


def _kernel_scan(lib, h, dev, hbm_peak):
    """Per-kernel rates at the other BASELINE sizes (context for the metric's
    'Sinkhorn HBM GB/s; GEMM TFLOP/s' parts; not the headline)."""
    import ctypes
    import torch
    from paper_2111_05366_b200 import _lib
    out = {}
    tf_peak, tf_kind = _bf16_peak()
    for n in (2000, 5000, 12288, 40000):
        G = torch.rand((n, n), dtype=torch.float32, device=dev) * 100.0
        ms = _ms_per_sweep(lib, h, n, G, reps=200 if n < 10000 else 20)
        gbs = n * n * 4 / (ms * 1e-3) / 1e9
        out[f"sinkhorn_sweep_n{n}"] = {"us": ms * 1e3, "GB_s": gbs, "frac_hbm": gbs / hbm_peak,
                                       "bytes": n * n * 4}
        del G
    for n, sym in ((2000, False), (5000, True), (8192, True)):
        g = torch.Generator(device=dev).manual_seed(n)
        A = (torch.rand((n, n), device=dev, generator=g) < 0.3).float()
        B = (torch.rand((n, n), device=dev, generator=g) < 0.3).float()
        if sym:
            A = torch.triu(A, 1); A = A + A.T
            B = torch.triu(B, 1); B = B + B.T
        X = torch.rand((n, n), device=dev, generator=g)
        X = X / X.sum(1, keepdim=True)
        ms = ctypes.c_double(); prods = ctypes.c_int32(); terms = ctypes.c_int32()
        _lib.check(lib.goat_bench_gradient(h.ptr, n, A.data_ptr(), B.data_ptr(), X.data_ptr(), 5,
                                           ctypes.byref(ms), ctypes.byref(prods), ctypes.byref(terms)))
        useful = prods.value * 2.0 * n ** 3 / (ms.value * 1e-3) / 1e12
        issued = useful * max(1, terms.value)
        out[f"gradient_n{n}_{'sym' if sym else 'directed'}"] = {
            "ms": ms.value, "useful_TFLOP_s": useful, "issued_bf16_TFLOP_s": issued,
            "frac_bf16_issued": issued / tf_peak, "bf16_terms_per_product": terms.value,
            "peak": tf_peak, "peak_kind": tf_kind}
        del A, B, X
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
