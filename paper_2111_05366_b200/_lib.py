"""ctypes binding of libgoat.so (include/goat.h).

The library is built in-tree (``python -m paper_2111_05366_b200.build``).
There is no CPU fallback: if the shared library or a CUDA device is missing,
every entry point raises ``RuntimeError`` instead of computing anything.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgoat.so")

GOAT_OK, GOAT_EINVAL, GOAT_ECUDA, GOAT_EOOM, GOAT_ENOTSUP = 0, 1, 2, 3, 4
GOAT_FP32, GOAT_FP64 = 0, 1
GOAT_MINIMIZE, GOAT_MAXIMIZE = 0, 1
GOAT_STEP_EXACT_LAP, GOAT_STEP_LOT = 0, 1
GOAT_GEMM_AUTO, GOAT_GEMM_SIMT, GOAT_GEMM_TCGEN05 = 0, 1, 2

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)
_c_i32_p = ctypes.POINTER(ctypes.c_int32)


class GoatConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("gemm", ctypes.c_int32), ("split_terms", ctypes.c_int32)]


class GoatOptions(ctypes.Structure):
    _fields_ = [("max_iters", ctypes.c_int32), ("max_sweeps", ctypes.c_int32),
                ("sense", ctypes.c_int32), ("step_solver", ctypes.c_int32),
                ("fw_tol", ctypes.c_double), ("lam", ctypes.c_double),
                ("sk_tol", ctypes.c_double)]


class GoatFwResult(ctypes.Structure):
    _fields_ = [("assignment", _c_i64_p), ("hist_obj", _c_double_p),
                ("hist_alpha", _c_double_p), ("lot_sweeps", _c_i32_p),
                ("lot_converged", _c_i32_p), ("lot_dev", _c_double_p),
                ("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("lap_certified", ctypes.c_int32), ("gpu_launches", ctypes.c_int32),
                ("objective", ctypes.c_double), ("time_ms", ctypes.c_double * 6),
                ("lot_fp64_from", _c_i32_p), ("lot_ms", _c_double_p)]


class GoatCsr(ctypes.Structure):
    _fields_ = [("rowptr", _c_i64_p), ("colidx", _c_i32_p), ("values", ctypes.c_void_p),
                ("nnz", ctypes.c_int64)]


_lib = None
_lib_lock = threading.Lock()


def _bind(lib):
    H = ctypes.c_void_p
    sig = {
        "goat_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(GoatConfig)]),
        "goat_destroy": (ctypes.c_int, [H]),
        "goat_last_error": (ctypes.c_char_p, []),
        "goat_version": (ctypes.c_char_p, []),
        "goat_reserve": (ctypes.c_int, [H, ctypes.c_int64]),
        "goat_fw_core": (ctypes.c_int, [H, ctypes.c_int64, _c_double_p, ctypes.c_int64, _c_double_p,
                                        ctypes.c_int64, _c_double_p, ctypes.c_int64, _c_double_p,
                                        ctypes.c_int64, ctypes.POINTER(GoatOptions),
                                        ctypes.POINTER(GoatFwResult)]),
        "goat_fw_core_device": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                               ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                               ctypes.POINTER(GoatOptions),
                                               ctypes.POINTER(GoatFwResult)]),
        "goat_fw_core_csr": (ctypes.c_int, [H, ctypes.c_int64, ctypes.POINTER(GoatCsr), ctypes.POINTER(GoatCsr),
                                            _c_double_p, ctypes.c_int64, _c_double_p, ctypes.c_int64,
                                            ctypes.POINTER(GoatOptions), ctypes.POINTER(GoatFwResult)]),
        "goat_fw_core_csr_device": (ctypes.c_int, [H, ctypes.c_int64, ctypes.POINTER(GoatCsr),
                                                   ctypes.POINTER(GoatCsr), ctypes.c_void_p, ctypes.c_int64,
                                                   ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(GoatOptions),
                                                   ctypes.POINTER(GoatFwResult)]),
        "goat_fw_core_seeded": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_int64] + [_c_double_p, ctypes.c_int64] * 7
                                + [ctypes.POINTER(GoatOptions), ctypes.POINTER(GoatFwResult)]),
        "goat_gradient_csr": (ctypes.c_int, [H, ctypes.c_int64, ctypes.POINTER(GoatCsr), ctypes.POINTER(GoatCsr),
                                             _c_double_p, ctypes.c_int64, _c_double_p, ctypes.c_int64]),
        "goat_bench_gradient_csr": (ctypes.c_int, [H, ctypes.c_int64, ctypes.POINTER(GoatCsr),
                                                   ctypes.POINTER(GoatCsr), ctypes.c_void_p, ctypes.c_int32,
                                                   _c_double_p]),
        "goat_gradient": (ctypes.c_int, [H, ctypes.c_int64, _c_double_p, ctypes.c_int64, _c_double_p,
                                         ctypes.c_int64, _c_double_p, ctypes.c_int64, _c_double_p,
                                         ctypes.c_int64]),
        "goat_lot": (ctypes.c_int, [H, ctypes.c_int64, _c_double_p, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.c_double, ctypes.c_int32, ctypes.c_double, _c_double_p,
                                    ctypes.c_int64, _c_i32_p, _c_i32_p, _c_double_p]),
        "goat_lot_device": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                           ctypes.c_double, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p,
                                           ctypes.c_int64, _c_i32_p, _c_i32_p, _c_double_p]),
        "goat_sinkhorn_knopp": (ctypes.c_int, [H, ctypes.c_int64, _c_double_p, ctypes.c_int64,
                                               ctypes.c_int32, ctypes.c_double, _c_double_p,
                                               ctypes.c_int64, _c_i32_p, _c_i32_p, _c_double_p]),
        "goat_line_search_coeffs": (ctypes.c_int, [H, ctypes.c_int64, _c_double_p, ctypes.c_int64,
                                                   _c_double_p, ctypes.c_int64, _c_double_p,
                                                   ctypes.c_int64, _c_double_p, ctypes.c_int64,
                                                   _c_double_p, ctypes.c_int64, _c_double_p,
                                                   _c_double_p]),
        "goat_lap": (ctypes.c_int, [H, ctypes.c_int64, _c_double_p, ctypes.c_int64, ctypes.c_int32,
                                    _c_i64_p, _c_double_p, _c_i32_p]),
        "goat_qap_objective_perm": (ctypes.c_int, [H, ctypes.c_int64, _c_double_p, ctypes.c_int64,
                                                   _c_double_p, ctypes.c_int64, _c_i64_p,
                                                   _c_double_p]),
        "goat_set_stream": (ctypes.c_int, [H, ctypes.c_void_p]),
        "goat_bench_sweep": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_int32, _c_double_p]),
        "goat_bench_gradient": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_int32, _c_double_p, _c_i32_p,
                                               _c_i32_p]),
        "goat_lap_device": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                           _c_i64_p, _c_double_p, _c_i32_p]),
        "goat_shard_setup": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_int64]),
        "goat_shard_gradient": (ctypes.c_int, [H, ctypes.c_void_p, ctypes.c_void_p]),
        "goat_shard_setup_csr": (ctypes.c_int, [H, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(GoatCsr),
                                                ctypes.POINTER(GoatCsr), ctypes.POINTER(GoatCsr),
                                                ctypes.POINTER(GoatCsr)]),
        "goat_shard_minmax": (ctypes.c_int, [H, ctypes.c_void_p, _c_double_p]),
        "goat_shard_lot_begin": (ctypes.c_int, [H, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                                ctypes.c_double, ctypes.c_int32, ctypes.c_double]),
        "goat_shard_lot_pass": (ctypes.c_int, [H, ctypes.c_void_p, ctypes.c_void_p]),
        "goat_shard_lot_merge": (ctypes.c_int, [H, ctypes.c_void_p, ctypes.c_int32]),
        "goat_shard_lot_status": (ctypes.c_int, [H, _c_i32_p, _c_i32_p, _c_i32_p, _c_double_p, _c_i32_p,
                                                 _c_i32_p]),
        "goat_shard_lot_refine": (ctypes.c_int, [H, ctypes.c_void_p, _c_i32_p]),
        "goat_shard_lot_repair_pass": (ctypes.c_int, [H, ctypes.c_void_p, ctypes.c_void_p]),
        "goat_shard_lot_repair_merge": (ctypes.c_int, [H, ctypes.c_void_p, ctypes.c_int32]),
        "goat_shard_lot_emit": (ctypes.c_int, [H, ctypes.c_void_p, ctypes.c_void_p]),
        "goat_shard_dots": (ctypes.c_int, [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, _c_double_p]),
        "goat_shard_axpby": (ctypes.c_int, [H, ctypes.c_double, ctypes.c_void_p, ctypes.c_double,
                                            ctypes.c_void_p]),
        "goat_shard_fill": (ctypes.c_int, [H, ctypes.c_double, ctypes.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


#: Every symbol include/goat.h declares (checked by tests/test_abi.py).
EXPORTS = ("goat_create", "goat_destroy", "goat_last_error", "goat_version", "goat_reserve",
           "goat_fw_core", "goat_fw_core_device", "goat_fw_core_seeded", "goat_fw_core_csr", "goat_fw_core_csr_device",
           "goat_gradient_csr", "goat_bench_gradient_csr", "goat_gradient", "goat_lot", "goat_lot_device",
           "goat_sinkhorn_knopp", "goat_line_search_coeffs", "goat_lap",
           "goat_qap_objective_perm", "goat_set_stream", "goat_bench_sweep",
           "goat_bench_gradient", "goat_lap_device", "goat_shard_setup", "goat_shard_setup_csr", "goat_shard_gradient",
           "goat_shard_minmax", "goat_shard_lot_begin", "goat_shard_lot_pass", "goat_shard_lot_merge",
           "goat_shard_lot_status", "goat_shard_lot_refine", "goat_shard_lot_repair_pass", "goat_shard_lot_repair_merge",
           "goat_shard_lot_emit", "goat_shard_dots", "goat_shard_axpby",
           "goat_shard_fill")


def load():
    """Load and bind libgoat.so; raise if it is absent (no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"libgoat.so not found at {LIB_PATH}; build it with "
                    "`python -m paper_2111_05366_b200.build` (nvcc, sm_100a)")
            _lib = _bind(ctypes.CDLL(LIB_PATH))
        return _lib


def check(rc):
    if rc == GOAT_OK:
        return
    msg = load().goat_last_error().decode(errors="replace")
    if rc == GOAT_EINVAL:
        raise ValueError(msg)
    if rc == GOAT_EOOM:
        raise MemoryError(msg)
    raise RuntimeError(f"libgoat error {rc}: {msg}")


class Handle:
    """Owns one goat_handle (one device, one stream, one precision)."""

    def __init__(self, device=0, precision="fp64", gemm="auto", split_terms=0):
        lib = load()
        prec = {"fp32": GOAT_FP32, "fp64": GOAT_FP64}[precision]
        g = {"auto": GOAT_GEMM_AUTO, "simt": GOAT_GEMM_SIMT, "tcgen05": GOAT_GEMM_TCGEN05}[gemm]
        cfg = GoatConfig(device, prec, g, split_terms)
        h = ctypes.c_void_p()
        check(lib.goat_create(ctypes.byref(h), ctypes.byref(cfg)))
        self._h = h
        self.precision = precision
        self.device = device
        self.lock = threading.Lock()

    @property
    def ptr(self):
        return self._h

    def close(self):
        if self._h:
            load().goat_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


_handles: dict = {}
_handles_lock = threading.Lock()


def handle(device=0, precision="fp64", gemm="auto") -> Handle:
    key = (os.getpid(), device, precision, gemm)
    with _handles_lock:
        h = _handles.get(key)
        if h is None:
            h = Handle(device, precision, gemm)
            _handles[key] = h
        return h


def release_handles() -> None:
    """Destroy this process's cached handles (frees their device workspace)."""
    with _handles_lock:
        for h in _handles.values():
            h.close()
        _handles.clear()


def stream_handle(torch_stream) -> ctypes.c_void_p:
    """cudaStream_t for goat_set_stream from a torch.cuda.Stream.  torch's default
    stream has handle 0, which goat_set_stream reads as "the handle's own stream";
    map it to cudaStreamLegacy (0x1) so the library really shares torch's stream."""
    s = int(torch_stream.cuda_stream)
    return ctypes.c_void_p(s if s != 0 else 1)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_c_double_p)


def f64(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 2 and a.strides[1] == 8 and a.strides[0] % 8 == 0 and a.strides[0] >= 8 * a.shape[1]:
        return a
    return np.ascontiguousarray(a)


def ld_of(a: np.ndarray) -> int:
    return a.strides[0] // 8 if a.shape[0] > 1 else max(1, a.shape[1])


def csr_struct(indptr, indices, values=None):
    """goat_csr over numpy arrays (kept alive by the caller): int64 rowptr, int32
    column indices, optional float64 values (None = every stored entry is 1)."""
    c = GoatCsr()
    c.rowptr = indptr.ctypes.data_as(_c_i64_p)
    c.colidx = indices.ctypes.data_as(_c_i32_p)
    c.values = ctypes.c_void_p(values.ctypes.data) if values is not None else None
    c.nnz = int(indices.size)
    return c


def csr_struct_device(indptr, indices, values=None):
    """goat_csr over torch CUDA tensors (rowptr int64, colidx int32, values of the
    handle's element type or None)."""
    c = GoatCsr()
    c.rowptr = ctypes.cast(ctypes.c_void_p(indptr.data_ptr()), _c_i64_p)
    c.colidx = ctypes.cast(ctypes.c_void_p(indices.data_ptr()), _c_i32_p)
    c.values = ctypes.c_void_p(values.data_ptr()) if values is not None else None
    c.nnz = int(indices.numel())
    return c
