"""ctypes binding of libcronus_b200.so (include/cronus_capi.h, include/cronus_ck.h).

The library is built in-tree (`python -m paper_2509_17357_b200.build`). There is no
fallback: if the library is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcronus_b200.so")
_lib = None

i32p = ctypes.POINTER(ctypes.c_int)
f64p = ctypes.POINTER(ctypes.c_double)
vpp = ctypes.POINTER(ctypes.c_void_p)


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2509_17357_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    L.cronus_last_error.restype = ctypes.c_char_p
    L.cronus_version.restype = ctypes.c_char_p
    L.cronus_free.argtypes = [ctypes.c_void_p]
    L.cronus_synth_trace.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                     ctypes.c_double, ctypes.c_longlong, i32p, f64p, i32p, i32p,
                                     ctypes.c_char_p, ctypes.c_int]
    L.cronus_trace_hash.argtypes = [ctypes.c_int, i32p, f64p, i32p, i32p]
    L.cronus_trace_hash.restype = ctypes.c_ulonglong
    L.cronus_run_virtual.argtypes = [ctypes.c_char_p, ctypes.c_int, i32p, f64p, i32p, i32p,
                                     ctypes.c_char_p, ctypes.c_int, ctypes.c_int, vpp, vpp, vpp]
    L.cronus_choose_split.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_longlong,
                                      ctypes.c_longlong, ctypes.c_int, ctypes.c_int, i32p, f64p,
                                      f64p, i32p]
    L.cronus_fit.argtypes = [ctypes.c_int, ctypes.c_int, f64p, f64p, f64p, f64p, f64p, f64p]
    L.cronus_percentile.argtypes = [f64p, ctypes.c_int, ctypes.c_double, f64p]
    L.cronus_config_roundtrip.argtypes = [ctypes.c_char_p, vpp]
    _bind_gpu(L)
    _lib = L
    return L


def _bind_gpu(L):
    """Signatures of the GPU-side entry points (present in the same library)."""
    try:
        from . import _gpu_sigs
        _gpu_sigs.bind(L)
    except ImportError:
        pass


def take_string(p: ctypes.c_void_p) -> str:
    s = ctypes.string_at(p.value).decode()
    lib().cronus_free(p)
    return s


def check(rc: int):
    if rc == 0:
        return
    msg = lib().cronus_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)
