"""Python mirror of cronus::GpuEngine (include/cronus/gpu.hpp, include/cronus_gpu.h).

    eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=40)
    res = eng.serve(cfg_text, trace)                # RunResult: reference-format json/events/csv
    res = eng.serve(cfg_text, trace, host_prompt=p)  # e2e: prompts H2D, tokens D2H inside the call

Every call goes to libcronus_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import json

import numpy as np

from ._lib import check, lib, take_string
from .engine import RunResult, Trace


def _p(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


class GpuEngine:
    def __init__(self, **options):
        text = "".join(f"{k} = {v}\n" for k, v in options.items())
        h = ctypes.c_void_p()
        check(lib().cronus_engine_create(text.encode(), ctypes.byref(h)))
        self._h = h
        self.options = options

    def close(self):
        if self._h:
            lib().cronus_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stage(self, cfg_text: str, trace: Trace):
        """Synthesize the trace's prompts on the device before a timed serve()."""
        ids, arr, ins, outs = trace.arrays()
        check(lib().cronus_engine_stage(self._h, cfg_text.encode(), len(ids), _p(ids, ctypes.c_int),
                                        _p(arr, ctypes.c_double), _p(ins, ctypes.c_int), _p(outs, ctypes.c_int)))

    def serve_logits(self, cfg_text: str, trace: Trace, vocab: int) -> RunResult:
        """serve() that also returns, per request, the fp32 logits [output_len, vocab] each
        generated token was sampled from (test hook; co-located pairs)."""
        ids, arr, ins, outs = trace.arrays()
        toks = np.empty(int(outs.sum()), np.int32)
        lg = np.empty((int(outs.sum()), vocab), np.float32)
        j = ctypes.c_void_p()
        check(lib().cronus_engine_serve_logits(
            self._h, cfg_text.encode(), len(ids), _p(ids, ctypes.c_int), _p(arr, ctypes.c_double),
            _p(ins, ctypes.c_int), _p(outs, ctypes.c_int), trace.name.encode(), _p(toks, ctypes.c_int),
            _p(lg, ctypes.c_float), ctypes.byref(j)))
        res = RunResult(take_string(j), "", "")
        offs = np.concatenate([[0], np.cumsum(outs)])
        res.extra["tokens"] = [toks[offs[i]:offs[i + 1]] for i in range(len(outs))]
        res.extra["logits"] = [lg[offs[i]:offs[i + 1]] for i in range(len(outs))]
        return res

    def prompts(self, cfg_text: str, trace: Trace) -> np.ndarray:
        """Host copy of the trace's prompt tokens (stages the trace first): the host
        buffers an end-to-end serve(host_prompt=...) starts from."""
        self.stage(cfg_text, trace)
        out = np.empty(int(trace.arrays()[2].sum()), np.int32)
        check(lib().cronus_engine_staged_prompts(self._h, _p(out, ctypes.c_int), len(out)))
        return out

    def time_pass(self, cfg_text: str, worker: int, n_dec=0, dec_ctx=0, chunk_len=0, chunk_pos0=0, reps=5) -> float:
        """Median ms of one forward pass on the PPI (0) or CPI (1) worker (calibration)."""
        ms = ctypes.c_double()
        check(lib().cronus_engine_time_pass(self._h, cfg_text.encode(), worker, n_dec, dec_ctx, chunk_len, chunk_pos0,
                                            reps, ctypes.byref(ms)))
        return ms.value

    def describe(self, probe=False) -> dict:
        out = ctypes.c_void_p()
        check(lib().cronus_engine_describe(self._h, 1 if probe else 0, ctypes.byref(out)))
        return json.loads(take_string(out))

    def serve(self, cfg_text: str, trace: Trace, host_prompt=None, want_tokens=False, events=True,
              profile=False) -> RunResult:
        ids, arr, ins, outs = trace.arrays()
        hp = None
        if host_prompt is not None:
            host_prompt = np.ascontiguousarray(host_prompt, np.int32)
            assert len(host_prompt) == int(ins.sum())
            hp = _p(host_prompt, ctypes.c_int)
        toks = np.empty(int(outs.sum()), np.int32) if want_tokens else None
        j, e, c, s = (ctypes.c_void_p() for _ in range(4))
        check(lib().cronus_engine_serve(
            self._h, cfg_text.encode(), len(ids), _p(ids, ctypes.c_int), _p(arr, ctypes.c_double),
            _p(ins, ctypes.c_int), _p(outs, ctypes.c_int), trace.name.encode(), hp,
            _p(toks, ctypes.c_int) if toks is not None else None, (1 if events else 0) | (2 if profile else 0),
            ctypes.byref(j), ctypes.byref(e), ctypes.byref(c), ctypes.byref(s)))
        res = RunResult(take_string(j), take_string(e), take_string(c))
        res.extra["stats"] = json.loads(take_string(s))
        if toks is not None:
            offs = np.concatenate([[0], np.cumsum(outs)])
            res.extra["tokens"] = [toks[offs[i]:offs[i + 1]] for i in range(len(outs))]
        return res


def plan_decode(lens, n_kv_heads: int, slots: int):
    """The engine's decode-attention plan (gpu::Batch::plan_decode) for these context lengths:
    (work list, seq_item0, cluster) as ck_attn_decode_tma takes them."""
    lens = np.ascontiguousarray(lens, np.int32)
    cap = 4 * len(lens) + 64 + int(((lens + 15) // 16).sum() // 8) + 1
    work = np.zeros(cap, np.int32)
    item0 = np.zeros(len(lens), np.int32)
    nw, cl = ctypes.c_int(), ctypes.c_int()
    check(lib().cronus_plan_decode(_p(lens, ctypes.c_int), len(lens), n_kv_heads, slots, _p(work, ctypes.c_int), cap,
                                   _p(item0, ctypes.c_int), ctypes.byref(nw), ctypes.byref(cl)))
    return work[:nw.value].copy(), item0, cl.value
