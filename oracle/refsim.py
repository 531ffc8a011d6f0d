"""TEST INFRASTRUCTURE ONLY — ctypes wrapper over oracle/_ref/libcronus_ref.so.

The library is the unmodified reference simulator (/root/reference/proj/src/*.cpp)
compiled out-of-tree by oracle/Makefile plus oracle/ref_shim.cpp. It is the
schedule oracle: split points (balancer.cpp:23-76), per-iteration batches
(engine.cpp:437-520), the KV ledger (engine.cpp:522-531) and the report writers
(metrics.cpp:95-156) all come from the reference itself.

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline leg
may import this module; the product never does.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libcronus_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"schedule oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = ctypes.CDLL(LIB_PATH)
        i32p = ctypes.POINTER(ctypes.c_int)
        f64p = ctypes.POINTER(ctypes.c_double)
        cpp = ctypes.POINTER(ctypes.c_void_p)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_run.argtypes = [ctypes.c_char_p, ctypes.c_int, i32p, f64p, i32p, i32p,
                              ctypes.c_char_p, ctypes.c_int, ctypes.c_int, cpp, cpp, cpp]
        L.ref_run.restype = ctypes.c_int
        L.ref_synth_trace.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_int, ctypes.c_double, ctypes.c_longlong,
                                      i32p, f64p, i32p, i32p, ctypes.c_char_p, ctypes.c_int]
        L.ref_trace_hash.argtypes = [ctypes.c_int, i32p, f64p, i32p, i32p]
        L.ref_trace_hash.restype = ctypes.c_ulonglong
        L.ref_choose_split.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_longlong,
                                       ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                                       i32p, f64p, f64p, i32p]
        L.ref_fit.argtypes = [ctypes.c_int, ctypes.c_int, f64p, f64p, f64p, f64p, f64p, f64p]
        L.ref_percentile.argtypes = [f64p, ctypes.c_int, ctypes.c_double]
        L.ref_percentile.restype = ctypes.c_double
        _lib = L
    return _lib


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


@dataclass
class Trace:
    ids: np.ndarray
    arrival_ms: np.ndarray
    input_len: np.ndarray
    output_len: np.ndarray
    name: str = ""

    def __len__(self):
        return len(self.ids)


def synth_trace(n, mean_in, mean_out, fixed_interval=False, interval_ms=0.0, seed=1) -> Trace:
    L = lib()
    ids = np.zeros(n, np.int32); arr = np.zeros(n, np.float64)
    ins = np.zeros(n, np.int32); outs = np.zeros(n, np.int32)
    name = ctypes.create_string_buffer(256)
    rc = L.ref_synth_trace(n, mean_in, mean_out, 1 if fixed_interval else 0, interval_ms, seed,
                           _p(ids, ctypes.c_int), _p(arr, ctypes.c_double), _p(ins, ctypes.c_int),
                           _p(outs, ctypes.c_int), name, 256)
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return Trace(ids, arr, ins, outs, name.value.decode())


def trace_hash(t: Trace) -> int:
    ids, arr, ins, outs = _i32(t.ids), _f64(t.arrival_ms), _i32(t.input_len), _i32(t.output_len)
    return lib().ref_trace_hash(len(ids), _p(ids, ctypes.c_int), _p(arr, ctypes.c_double),
                                _p(ins, ctypes.c_int), _p(outs, ctypes.c_int))


def run(cfg_text: str, t: Trace, events=True, utilization=False):
    """Returns (json_text, event_log_text, csv_row) exactly as the reference writes them."""
    L = lib()
    ids, arr, ins, outs = _i32(t.ids), _f64(t.arrival_ms), _i32(t.input_len), _i32(t.output_len)
    j = ctypes.c_void_p(); e = ctypes.c_void_p(); c = ctypes.c_void_p()
    rc = L.ref_run(cfg_text.encode(), len(ids), _p(ids, ctypes.c_int), _p(arr, ctypes.c_double),
                   _p(ins, ctypes.c_int), _p(outs, ctypes.c_int), t.name.encode(),
                   1 if events else 0, 1 if utilization else 0,
                   ctypes.byref(j), ctypes.byref(e), ctypes.byref(c))
    if rc == 1:
        raise ValueError(L.ref_last_error().decode())
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    out = []
    for p in (j, e, c):
        out.append(ctypes.string_at(p.value).decode())
        L.ref_free(p)
    return tuple(out)


def choose_split(cfg_text, n_decode, decode_ctx_sum, free_kv_blocks, max_batched_tokens, input_len):
    L = lib()
    lp = ctypes.c_int(); tp = ctypes.c_double(); tc = ctypes.c_double(); fl = ctypes.c_int()
    rc = L.ref_choose_split(cfg_text.encode(), n_decode, decode_ctx_sum, free_kv_blocks,
                            max_batched_tokens, input_len, ctypes.byref(lp), ctypes.byref(tp),
                            ctypes.byref(tc), ctypes.byref(fl))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return lp.value, tp.value, tc.value, fl.value


def fit(kind, x0, x1, y):
    """kind 0 = fit_prefill(len), 1 = fit_chunked(prefill_ctx, decode_ctx_sum)."""
    L = lib()
    x0 = _f64(x0); x1 = _f64(x1 if x1 is not None else np.zeros_like(x0)); y = _f64(y)
    coef = np.zeros(3); r2 = ctypes.c_double(); mape = ctypes.c_double()
    rc = L.ref_fit(kind, len(y), _p(x0, ctypes.c_double), _p(x1, ctypes.c_double),
                   _p(y, ctypes.c_double), _p(coef, ctypes.c_double), ctypes.byref(r2),
                   ctypes.byref(mape))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return coef[: 2 if kind == 0 else 3].copy(), r2.value, mape.value
