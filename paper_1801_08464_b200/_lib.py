"""ctypes binding of libmgrgpu.so (the C-ABI in include/mgrgpu.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmgrgpu.so")
LIB_PATH_CHECKED = os.path.join(_HERE, "libmgrgpu_checked.so")

c_int, c_double, c_void_p, c_int64 = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64
P = c_void_p


class AmgOpts(ctypes.Structure):
    _fields_ = [("strength_theta", c_double), ("max_levels", c_int), ("coarse_size_cutoff", c_int),
                ("pre_sweeps", c_int), ("post_sweeps", c_int), ("cycles", c_int), ("max_elmts", c_int),
                ("seed", ctypes.c_uint64)]


class LevelSpec(ctypes.Structure):
    _fields_ = [("f_mask", P), ("rp_kind", c_int), ("frelax_kind", c_int), ("frelax_sweeps", c_int),
                ("frelax_pre", c_int), ("frelax_post", c_int), ("frelax_max_levels", c_int),
                ("global_relax", c_int)]


class GmresOpts(ctypes.Structure):
    _fields_ = [("rel_tol", c_double), ("max_iter", c_int), ("restart", c_int),
                ("reorthogonalize", c_int), ("check_every", c_int)]


class GmresRes(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("converged", c_int), ("residual_norm", c_double),
                ("rhs_norm", c_double), ("cycles", c_int), ("first_cycle_iterations", c_int)]


class Timing(ctypes.Structure):
    _fields_ = [("setup_ms", c_double), ("solve_ms", c_double), ("spmv_ms", c_double),
                ("spmv_calls", c_int64), ("vcycle_ms", c_double), ("vcycle_calls", c_int64),
                ("vcycle_bytes", c_double), ("spmv_bytes", c_double), ("phase_ms", c_double * 8),
                ("k0_ms", c_double), ("k0_calls", c_int64), ("k0_bytes", c_double),
                ("frelax_calls", c_int64), ("frelax_bytes", c_double)]


_SIGS = {
    "mg_ctx_create": [c_int, ctypes.POINTER(P)],
    "mg_ctx_destroy": [P],
    "mg_ctx_sync": [P],
    "mg_mat_upload_csr": [P, c_int, c_int, P, P, P, ctypes.POINTER(P)],
    "mg_mat_upload_bsr": [P, c_int, c_int, c_int, P, P, P, ctypes.POINTER(P)],
    "mg_mat_upload_bsr_async": [P, c_int, c_int, c_int, P, P, P, ctypes.POINTER(P)],
    "mg_mat_upload_csr_varmajor": [P, c_int, c_int, P, P, P, ctypes.POINTER(P)],
    "mg_strength": [P, P, ctypes.c_double, P, P],
    "mg_mat_info": [P, P, ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int64),
                    ctypes.POINTER(c_int)],
    "mg_mat_download": [P, P, P, P, P],
    "mg_mat_free": [P, P],
    "mg_spmv": [P, P, P, P],
    "mg_spmv_dev": [P, P, P, P],
    "mg_spmv_layout": [P, P, ctypes.POINTER(c_int), ctypes.POINTER(c_int), ctypes.POINTER(c_int)],
    "mg_matmul": [P, P, P, ctypes.POINTER(P)],
    "mg_triple_product": [P, P, P, P, ctypes.POINTER(P)],
    "mg_transpose": [P, P, ctypes.POINTER(P)],
    "mg_extract": [P, P, P, c_int, P, c_int, ctypes.POINTER(P)],
    "mg_block_scale": [P, P, c_int, ctypes.POINTER(P), ctypes.POINTER(P)],
    "mg_block_apply": [P, P, P, P],
    "mg_equilibrate": [P, P, ctypes.POINTER(P), P, P],
    "mg_abs_row_sum_max": [P, P, ctypes.POINTER(c_double)],
    "mg_build_rp": [P, P, P, c_int, ctypes.POINTER(P), ctypes.POINTER(P)],
    "mg_amg_setup": [P, P, ctypes.POINTER(AmgOpts), ctypes.POINTER(P)],
    "mg_amg_vcycle": [P, P, P, P, P],
    "mg_amg_apply": [P, P, P, P],
    "mg_amg_nlevels": [P, P, ctypes.POINTER(c_int), ctypes.POINTER(c_int)],
    "mg_amg_level_mat": [P, P, c_int, c_int, ctypes.POINTER(P)],
    "mg_amg_splitting": [P, P, c_int, P],
    "mg_amg_row_sign": [P, P, P],
    "mg_amg_free": [P, P],
    "mg_mgr_setup": [P, P, ctypes.POINTER(LevelSpec), c_int, ctypes.POINTER(AmgOpts), c_int, c_int, P,
                     ctypes.POINTER(P)],
    "mg_mgr_set_prescale": [P, P, P],
    "mg_mgr_apply": [P, P, P, P],
    "mg_mgr_apply_dev": [P, P, P, P],
    "mg_mgr_nlevels": [P, P, ctypes.POINTER(c_int)],
    "mg_mgr_level_mat": [P, P, c_int, c_int, ctypes.POINTER(P)],
    "mg_mgr_level_amg": [P, P, c_int, ctypes.POINTER(P)],
    "mg_mgr_free": [P, P],
    "mg_gmres": [P, P, P, P, P, ctypes.POINTER(GmresOpts), c_double, ctypes.POINTER(GmresRes)],
    "mg_gmres_dev": [P, P, P, P, P, ctypes.POINTER(GmresOpts), c_double, ctypes.POINTER(GmresRes)],
    "mg_gmres_ilu": [P, P, P, P, P, ctypes.POINTER(GmresOpts), c_double, ctypes.POINTER(GmresRes)],
    "mg_ilu_factor": [P, P, c_int, ctypes.POINTER(P)],
    "mg_ilu_matrix": [P, P, ctypes.POINTER(P)],
    "mg_ilu_apply": [P, P, P, P],
    "mg_ilu_free": [P, P],
    "mg_asm_create": [P, P, ctypes.POINTER(P)],
    "mg_asm_assemble": [P, P, P, P, P, P, P, P, c_double, P, P, ctypes.POINTER(P)],
    "mg_asm_free": [P, P],
    "mg_dev_alloc": [P, c_int64, ctypes.POINTER(P)],
    "mg_dev_free": [P, P],
    "mg_memcpy_h2d": [P, P, P, c_int64],
    "mg_memcpy_d2h": [P, P, P, c_int64],
    "mg_get_timing": [P, ctypes.POINTER(Timing)],
    "mg_set_profiling": [P, c_int],
    "mg_timer_start": [P],
    "mg_timer_stop": [P, ctypes.POINTER(c_double)],
}

EXPORTED = sorted(list(_SIGS) + ["mg_last_error", "mg_last_error_row", "mg_ctx_launches",
                                 "mg_ctx_device_bytes"])

_lib = None
_lock = threading.Lock()


def load(path: str | None = None):
    """Load libmgrgpu.so (no CUDA call is made here).  MG_LIB=checked loads
    libmgrgpu_checked.so instead: the same kernels built with device-side bounds
    checks (-DMG_BOUNDS_CHECK), for test runs only."""
    global _lib
    if path is None:
        path = LIB_PATH_CHECKED if os.environ.get("MG_LIB") == "checked" else LIB_PATH
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libmgrgpu.so not found at {path}: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_1801_08464_b200/csrc). There is no CPU fallback.")
        L = ctypes.CDLL(path)
        for name, args in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = c_int
        L.mg_last_error.argtypes = [P]
        L.mg_last_error.restype = ctypes.c_char_p
        L.mg_last_error_row.argtypes = [P]
        L.mg_last_error_row.restype = c_int64
        L.mg_ctx_launches.argtypes = [P]
        L.mg_ctx_launches.restype = c_int64
        L.mg_ctx_device_bytes.argtypes = [P]
        L.mg_ctx_device_bytes.restype = c_int64
        _lib = L
        return L


class Context:
    """One CUDA device + stream of libmgrgpu."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = P()
        st = self.lib.mg_ctx_create(int(device), ctypes.byref(h))
        if st != 0:
            raise RuntimeError(f"libmgrgpu: cannot create a CUDA context on device {device} (status {st}); "
                               "a B200 GPU is required — there is no CPU fallback")
        self.h = h
        self.device = device

    def check(self, st):
        if st == 0:
            return
        msg = self.lib.mg_last_error(self.h).decode(errors="replace")
        row = int(self.lib.mg_last_error_row(self.h))
        raise errors.from_status(st, msg, row)

    def call(self, name, *args):
        self.check(getattr(self.lib, name)(self.h, *args))

    @property
    def launches(self):
        return int(self.lib.mg_ctx_launches(self.h))

    @property
    def device_bytes(self):
        return int(self.lib.mg_ctx_device_bytes(self.h))

    def timing(self):
        t = Timing()
        self.check(self.lib.mg_get_timing(self.h, ctypes.byref(t)))
        return t

    def set_profiling(self, on=True):
        self.check(self.lib.mg_set_profiling(self.h, int(bool(on))))

    def sync(self):
        self.call("mg_ctx_sync")

    def close(self):
        if getattr(self, "h", None):
            self.lib.mg_ctx_destroy(self.h)
            self.h = None

    def __del__(self):  # objects built on a context keep a reference to it
        try:
            self.close()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass


_tls = threading.local()


def ctx(device: int | None = None) -> Context:
    """This thread's context for ``device`` (default: the thread's current one, else
    device 0).  One context per (thread, device), kept for the thread's lifetime:
    switching devices does not drop (and leak) the previous device's context."""
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device is None:
        device = getattr(_tls, "current", 0)
    c = ctxs.get(device)
    if c is None or c.h is None:
        c = ctxs[device] = Context(device)
    _tls.current = device
    return c


def ptr(a: np.ndarray):
    return a.ctypes.data_as(c_void_p)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)
