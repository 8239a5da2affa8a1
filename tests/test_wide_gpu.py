"""The 2-CTA wide-row Sinkhorn kernel (sk_wide_kernel, 12288 < n <= 40960 fp32,
config 5's n = 40000) against the previous cluster kernel on the same device
G, through goat_lot_device: same sweep count and stopping flag, iterates within
fp32 accumulation-order noise, bit-identical reruns.  Smaller orders of the
same kernel are checked against the CPU oracle in test_lot_large_gpu.py
(n = 17000, 20000)."""
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
    return G


@pytest.mark.parametrize("n", [12289, 16384, 25003, 40000])
def test_wide_kernel_matches_cluster_kernel(n, monkeypatch):
    G = _cost(n)
    monkeypatch.setenv("GOAT_SK_WIDE", "1")
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
