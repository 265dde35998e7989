"""ctypes binding of oracle/lib/liboracle.so (built by oracle/Makefile)."""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "lib", "liboracle.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i = ctypes.c_int
        L.pmis.argtypes = [i, P, P, P, ctypes.c_uint64, i, P]
        L.pmis.restype = i
        L.pmis_u.argtypes = [ctypes.c_uint64, i, ctypes.c_int64]
        L.pmis_u.restype = ctypes.c_double
        L.ext_interp_count.argtypes = [i, P, P, P, P, P, i, P]
        L.ext_interp_count.restype = i
        L.ext_interp_fill.argtypes = [i, P, P, P, P, P, i, P, P, P]
        L.ext_interp_fill.restype = i
        L.spgemm_count.argtypes = [i, i, P, P, P, P, P, P, P]
        L.spgemm_fill.argtypes = [i, i, P, P, P, P, P, P, P, P, P]
        _lib = L
    return _lib


def ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def c32(a):
    return np.ascontiguousarray(a, dtype=np.int32)
