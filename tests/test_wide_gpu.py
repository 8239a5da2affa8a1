"""The 2-CTA wide-row Sinkhorn kernel (sk_wide_kernel: planned for 22000 < n <= 40960
fp32, config 5's n = 40000; forced here down to n = 12289) against the previous cluster kernel on the same device
G, through goat_lot_device: same sweep count and stopping flag, iterates within
fp32 accumulation-order noise, bit-identical reruns; and its fixed-shift redo
path (every sweep redone with the max shift == the max-shift run, bit for bit).
The previous kernels are checked against the CPU oracle in test_lot_large_gpu.py."""
import ctypes

import numpy as np
import pytest

from paper_2111_05366_b200 import _lib

pytestmark = pytest.mark.gpu


def _lot_device(G, n, sweeps):
    import torch
    h = _lib.handle(0, "fp32")
    Q = torch.empty_like(G)
    conv, sw, dev = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_double()
    ld = G.shape[1]
    _lib.check(_lib.load().goat_lot_device(h.ptr, n, G.data_ptr(), ld, _lib.GOAT_MAXIMIZE, 100.0, sweeps, 1e-8,
                                           Q.data_ptr(), ld, ctypes.byref(conv), ctypes.byref(sw), ctypes.byref(dev)))
    torch.cuda.synchronize()
    return Q, sw.value, conv.value, dev.value


def _cost(n):
    import torch
    g = torch.Generator(device="cuda").manual_seed(n)
    ld = (n + 7) // 8 * 8
    d1 = torch.randint(50, 150, (n,), device="cuda", generator=g).float()
    d2 = torch.randint(50, 150, (n,), device="cuda", generator=g).float()
    G = torch.zeros((n, ld), device="cuda")
    G[:, :n] = torch.outer(d1, d2) / n + torch.rand((n, n), device="cuda", generator=g)
    torch.cuda.synchronize()  # the library runs on the handle's own stream, not torch's
    return G


@pytest.mark.parametrize("n", [12289, 16384, 25003, 40000])
def test_wide_kernel_matches_cluster_kernel(n, monkeypatch):
    G = _cost(n)
    monkeypatch.setenv("GOAT_SK_WIDE", "2")  # the wide kernel at every tested order
    Q1, s1, c1, d1 = _lot_device(G, n, 25)
    Q1b, s1b, _, d1b = _lot_device(G, n, 25)
    assert s1 == s1b and d1 == d1b
    assert bool((Q1[:, :n] == Q1b[:, :n]).all()), "rerun not bit-identical"
    monkeypatch.setenv("GOAT_SK_WIDE", "0")
    Q0, s0, c0, d0 = _lot_device(G, n, 25)
    assert (s1, c1) == (s0, c0)
    assert d1 == pytest.approx(d0, rel=1e-2)
    err = float((Q1[:, :n] - Q0[:, :n]).abs().max())
    assert err < 1e-5, err
    rs = Q1[:, :n].double().sum(1)
    cs = Q1[:, :n].double().sum(0)
    assert float((cs - 1).abs().max()) < 1e-4  # the returned iterate's columns are balanced
    assert float((rs - 1).abs().max()) == pytest.approx(d1, rel=0.05, abs=1e-5)


@pytest.mark.parametrize("n", [16384, 40000])
def test_wide_kernel_redo_path(n, monkeypatch):
    """Sweeps >= 2 shift each row by its previous LSE; a row whose sum leaves the
    window redoes the sweep with the max shift.  Forcing every sweep through the
    redo (GOAT_SK_RES=3) must reproduce the max-shift-only run (GOAT_SK_RES=2)
    exactly, and the default must agree with both to fp32 accuracy."""
    G = _cost(n)
    monkeypatch.setenv("GOAT_SK_WIDE", "2")
    out = {}
    for mode in ("2", "3", "1"):
        monkeypatch.setenv("GOAT_SK_RES", mode)
        out[mode] = _lot_device(G, n, 12)
    assert bool((out["3"][0][:, :n] == out["2"][0][:, :n]).all())
    assert out["3"][1:] == out["2"][1:]
    assert float((out["1"][0][:, :n] - out["2"][0][:, :n]).abs().max()) < 1e-5
    assert out["1"][1] == out["2"][1]
