"""TEST / BASELINE INFRASTRUCTURE ONLY — the CPU serving baseline.

The reference's own implementation of this path is a discrete-event simulator whose
"GPU work" is three cost formulas (proj/src/costmodel.cpp:9-15); it has no model
arithmetic to run on a CPU. The CPU baseline therefore follows the paper's own
methodology (reference costmodel.cpp:94-113):

  1. time the CPU fp32 forward (oracle/numerics.py arithmetic, numpy BLAS on all
     host cores) of ONE LLaMA3-8B decoder layer on a bounded set of shapes —
     prefill lengths and mixed chunk+decode batches — and extrapolate to all
     layers plus the LM head;
  2. fit a CPU GpuProfile with the REFERENCE's fit_prefill / fit_chunked (through
     oracle/_ref, the unmodified reference library);
  3. run the REFERENCE's simulator (oracle/_ref) with that profile for both roles on
     the benchmark trace -> CPU req/s, TTFT P99, TBT P99.

Only bench.py's cpu_baseline leg / --impl reference arm and tests may import this.
"""
from __future__ import annotations

import json
import os
import re
import time

import numpy as np

from . import numerics as NUM
from . import refsim


class _Layer:
    """fp32 weights of one decoder layer of `spec` (constant-filled: BLAS timing depends
    on shapes only, and filling 0.9 GB with random numbers would dominate the budget)."""

    def __init__(self, spec: NUM.Spec):
        H, F, Q = spec.hidden, spec.ffn, spec.qkv_n
        f = lambda *s: np.full(s, 0.01, dtype=np.float32)
        self.s = spec
        self.wqkv, self.wo = f(Q, H), f(H, spec.n_heads * 128)
        self.wgu, self.wd = f(2 * F, H), f(H, F)
        self.g = np.ones(H, np.float32)

    def forward(self, x, k_cache, v_cache, seqs):
        """x [n, H]; seqs = [(row0, rows, pos0)] — a sequence's rows sit at positions
        pos0.. and attend causally to keys [0, pos0 + rows) of k/v_cache [T, nkv, 128].
        Linear layers run batched over all rows (as the GPU engine does)."""
        s = self.s
        n = x.shape[0]
        h = NUM.rmsnorm(x, self.g, s.rms_eps)
        qkv = h @ self.wqkv.T
        q = qkv[:, : s.n_heads * 128].reshape(n, s.n_heads, 128)
        G = s.n_heads // s.n_kv_heads
        out = np.empty((n, s.n_heads, 128), np.float32)
        scale = np.float32(1 / np.sqrt(128.0))
        for (r0, rows, pos0) in seqs:
            T = pos0 + rows
            K, V = k_cache[:T], v_cache[:T]
            mask = np.arange(T)[None, :] > (pos0 + np.arange(rows))[:, None]
            for kv in range(s.n_kv_heads):
                qq = q[r0:r0 + rows, kv * G:(kv + 1) * G, :].transpose(1, 0, 2)  # [G, rows, 128]
                sc = (qq @ K[:, kv, :].T) * scale
                sc = np.where(mask[None], -np.inf, sc)
                sc = np.exp(sc - sc.max(axis=-1, keepdims=True))
                sc /= sc.sum(axis=-1, keepdims=True)
                out[r0:r0 + rows, kv * G:(kv + 1) * G, :] = (sc @ V[:, kv, :]).transpose(1, 0, 2)
        x = x + out.reshape(n, -1) @ self.wo.T
        h = NUM.rmsnorm(x, self.g, s.rms_eps)
        gu = h @ self.wgu.T
        g, u = gu[:, 0::2], gu[:, 1::2]
        return x + (g / (1 + np.exp(-g)) * u) @ self.wd.T


def _time(fn, reps=2):
    fn()
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best * 1000.0


def cpu_profile(model: str = "llama3-8b", budget_s: float = 20.0, seed: int = 0):
    """Measure the CPU forward on bounded samples; returns (prefill fit, chunked fit, samples)."""
    spec = NUM.PRESETS[model]
    rng = np.random.default_rng(seed)
    layer = _Layer(spec)
    lm = np.full((spec.vocab, spec.hidden), 0.01, dtype=np.float32)
    T = 4096
    kc = rng.standard_normal((T, spec.n_kv_heads, 128), dtype=np.float32)
    vc = rng.standard_normal((T, spec.n_kv_heads, 128), dtype=np.float32)
    H = spec.hidden
    t_start = time.perf_counter()

    def full(rows, seqs, sampled_rows):
        # one layer timed, x layers, + LM head on the sampled rows
        x = rng.standard_normal((rows, H), dtype=np.float32)
        t_layer = _time(lambda: layer.forward(x, kc, vc, seqs))
        t_lm = _time(lambda: x[:sampled_rows] @ lm.T, reps=1)
        return spec.layers * t_layer + t_lm

    prefill = []
    for L in (32, 128, 256, 512):
        prefill.append((float(L), full(L, [(0, L, 0)], 1)))
        if len(prefill) >= 2 and time.perf_counter() - t_start > budget_s * 0.4:
            break
    chunked = []
    for (chunk, pos0, n_dec, ctx) in ((128, 0, 0, 0), (0, 0, 16, 1024), (256, 256, 8, 512), (64, 1024, 32, 1024),
                                      (0, 0, 64, 512), (448, 0, 64, 512)):
        seqs = [(i, 1, ctx - 1) for i in range(n_dec)]
        if chunk:
            seqs.append((n_dec, chunk, pos0))
        ms = full(n_dec + chunk, seqs, n_dec + (1 if chunk else 0))
        chunked.append((float(pos0 + chunk), float(n_dec * ctx), ms))
        # fit_chunked needs >= 3 samples (costmodel.cpp:105): the budget never cuts below that
        if len(chunked) >= 3 and time.perf_counter() - t_start > budget_s:
            break
    pf = refsim.fit(0, [p[0] for p in prefill], None, [p[1] for p in prefill])
    cf = refsim.fit(1, [c[0] for c in chunked], [c[1] for c in chunked], [c[2] for c in chunked])
    return pf, cf, {"prefill": prefill, "chunked": chunked, "seconds": time.perf_counter() - t_start,
                    "threads": os.cpu_count()}


def cpu_config(base_cfg_text: str, pf, cf) -> str:
    """The base config with both profiles replaced by the fitted CPU profile."""
    (kp, bp), (kc, kd, bc) = pf[0], cf[0]
    vals = {"prefill_k": max(kp, 0.0), "prefill_b": max(bp, 0.0), "chunked_k_ctxp": max(kc, 0.0),
            "chunked_k_ctxd": max(kd, 0.0), "chunked_b": max(bc, 0.0)}
    out = []
    for line in base_cfg_text.splitlines():
        m = re.match(r"\s*(high|low)\.(\w+)\s*=", line)
        if m and m.group(2) in vals:
            line = f"{m.group(1)}.{m.group(2)} = {float(vals[m.group(2)])!r}"
        elif m and m.group(2) == "name":
            line = f"{m.group(1)}.name = CPU-{m.group(1)}"
        out.append(line)
    return "\n".join(out) + "\n"


def run(base_cfg_text: str, trace: refsim.Trace, model: str = "llama3-8b", budget_s: float = 20.0):
    """Full CPU baseline: bounded CPU timing -> reference fit -> reference DES."""
    t0 = time.perf_counter()
    pf, cf, samples = cpu_profile(model, budget_s)
    cfg = cpu_config(base_cfg_text, pf, cf)
    t1 = time.perf_counter()
    rep = json.loads(refsim.run(cfg, trace, events=False)[0])
    t2 = time.perf_counter()
    return {
        "rps": rep["throughput_rps"], "ttft_p99_ms": rep["ttft_p99_ms"], "tbt_p99_ms": rep["tbt_p99_ms"],
        "completed": rep["completed"], "fit_prefill": {"coef": list(pf[0]), "r2": pf[1], "mape": pf[2]},
        "fit_chunked": {"coef": list(cf[0]), "r2": cf[1], "mape": cf[2]}, "samples": samples,
        "cpu_seconds": t1 - t0, "des_seconds": t2 - t1, "config": cfg,
    }
