"""Python mirror of the reference's public API for the serving path.

Names and argument meaning follow proj/include/cronus/*.hpp (`run`, `synth_trace`,
`trace_hash`, `choose_split`, `fit_prefill`, `fit_chunked`, `percentile`); every
call goes through libcronus_b200.so (C++ host + CUDA engine). `run(..., gpu=...)`
serves the trace on B200 workers; without `gpu` it is the virtual-clock drop-in
for the CPU simulator.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from ._lib import check, lib, take_string

FIXED_INTERVAL = "fixed-interval"
ALL_AT_ZERO = "all-at-zero"


@dataclass
class Trace:
    """reference trace.hpp:11-14 (struct-of-arrays)."""
    ids: np.ndarray
    arrival_ms: np.ndarray
    input_len: np.ndarray
    output_len: np.ndarray
    name: str = ""

    def __len__(self):
        return int(len(self.ids))

    def subset(self, mask_or_idx, name=None) -> "Trace":
        idx = np.asarray(mask_or_idx)
        return Trace(self.ids[idx].copy(), self.arrival_ms[idx].copy(), self.input_len[idx].copy(),
                     self.output_len[idx].copy(), self.name if name is None else name)

    def arrays(self):
        return (np.ascontiguousarray(self.ids, np.int32), np.ascontiguousarray(self.arrival_ms, np.float64),
                np.ascontiguousarray(self.input_len, np.int32), np.ascontiguousarray(self.output_len, np.int32))


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def synth_trace(n, mean_in, mean_out, arrival=ALL_AT_ZERO, interval_ms=0.0, seed=0) -> Trace:
    """reference trace.hpp:24 synth_trace (identical draws)."""
    ids = np.zeros(n, np.int32); arr = np.zeros(n, np.float64)
    ins = np.zeros(n, np.int32); outs = np.zeros(n, np.int32)
    name = ctypes.create_string_buffer(256)
    check(lib().cronus_synth_trace(n, float(mean_in), float(mean_out), 1 if arrival == FIXED_INTERVAL else 0,
                                   float(interval_ms), int(seed), _p(ids, ctypes.c_int), _p(arr, ctypes.c_double),
                                   _p(ins, ctypes.c_int), _p(outs, ctypes.c_int), name, 256))
    return Trace(ids, arr, ins, outs, name.value.decode())


def trace_hash(t: Trace) -> int:
    ids, arr, ins, outs = t.arrays()
    return lib().cronus_trace_hash(len(ids), _p(ids, ctypes.c_int), _p(arr, ctypes.c_double),
                                   _p(ins, ctypes.c_int), _p(outs, ctypes.c_int))


@dataclass
class RunResult:
    json: str
    events: str
    csv: str
    extra: dict = field(default_factory=dict)


def run(cfg_text: str, trace: Trace, events: bool = True, utilization: bool = False) -> RunResult:
    """reference engine.hpp:18 run() on the virtual clock (no device work)."""
    ids, arr, ins, outs = trace.arrays()
    j = ctypes.c_void_p(); e = ctypes.c_void_p(); c = ctypes.c_void_p()
    check(lib().cronus_run_virtual(cfg_text.encode(), len(ids), _p(ids, ctypes.c_int), _p(arr, ctypes.c_double),
                                   _p(ins, ctypes.c_int), _p(outs, ctypes.c_int), trace.name.encode(),
                                   1 if events else 0, 1 if utilization else 0,
                                   ctypes.byref(j), ctypes.byref(e), ctypes.byref(c)))
    return RunResult(take_string(j), take_string(e), take_string(c))


def choose_split(cfg_text, n_decode, decode_ctx_sum, free_kv_blocks, max_batched_tokens, input_len):
    """reference balancer.hpp:31 choose_split -> (L_p, t_prefill, t_chunked, flags)."""
    lp = ctypes.c_int(); tp = ctypes.c_double(); tc = ctypes.c_double(); fl = ctypes.c_int()
    check(lib().cronus_choose_split(cfg_text.encode(), n_decode, decode_ctx_sum, free_kv_blocks,
                                    max_batched_tokens, input_len, ctypes.byref(lp), ctypes.byref(tp),
                                    ctypes.byref(tc), ctypes.byref(fl)))
    return lp.value, tp.value, tc.value, fl.value


def _fit(kind, x0, x1, y):
    x0 = np.ascontiguousarray(x0, np.float64)
    x1 = np.ascontiguousarray(x1 if x1 is not None else np.zeros_like(x0), np.float64)
    y = np.ascontiguousarray(y, np.float64)
    coef = np.zeros(3); r2 = ctypes.c_double(); mape = ctypes.c_double()
    check(lib().cronus_fit(kind, len(y), _p(x0, ctypes.c_double), _p(x1, ctypes.c_double), _p(y, ctypes.c_double),
                           _p(coef, ctypes.c_double), ctypes.byref(r2), ctypes.byref(mape)))
    return coef[: 2 if kind == 0 else 3].copy(), r2.value, mape.value


def fit_prefill(lens, times_ms):
    """reference costmodel.hpp:38 -> ((k, b), r2, mape)."""
    return _fit(0, lens, None, times_ms)


def fit_chunked(prefill_ctx, decode_ctx_sum, times_ms):
    """reference costmodel.hpp:39 -> ((k_ctxp, k_ctxd, b), r2, mape)."""
    return _fit(1, prefill_ctx, decode_ctx_sum, times_ms)


def percentile(samples, p):
    v = np.ascontiguousarray(samples, np.float64)
    out = ctypes.c_double()
    check(lib().cronus_percentile(_p(v, ctypes.c_double), len(v), p, ctypes.byref(out)))
    return out.value


def config_roundtrip(cfg_text: str) -> str:
    out = ctypes.c_void_p()
    check(lib().cronus_config_roundtrip(cfg_text.encode(), ctypes.byref(out)))
    return take_string(out)
