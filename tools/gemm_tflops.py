"""Tensor-regime projection GEMM alone (ck_gemm, bf16 -> fp32), CUDA-event timed over
back-to-back launches, LLaMA3-8B projection shapes at prefill token counts; prints one JSON line
per (M, shape, CTA cap) with TFLOP/s and the fraction of MEASURED_PEAKS.json's bf16 peaks
(device burst / sustained, and scaled to the CTA cap's share of the SMs).

    python tools/gemm_tflops.py [--m 512,1024,4096] [--ctas 0,108,40] [--reps 20]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200._lib import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", default="512,1024,4096")
ap.add_argument("--ctas", default="0,108,40")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
L = lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
sms = torch.cuda.get_device_properties(0).multi_processor_count
try:
    pk = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
except Exception:
    pk = {"bf16_tflops": 1664.9, "bf16_tflops_sustained": 1390.0}
SHAPES = {"qkv": (6144, 4096), "o": (4096, 4096), "gate_up": (28672, 4096), "down": (4096, 14336)}
for M in (int(x) for x in a.m.split(",")):
    for ctas in (int(x) for x in a.ctas.split(",")):
        tot_f = tot_us = 0.0
        for name, (N, K) in SHAPES.items():
            W = torch.randn(N, K, device="cuda").bfloat16()
            X = torch.randn(M, K, device="cuda").bfloat16()
            out = torch.zeros(M, N, device="cuda")
            # the engine's epilogues: residual red.add (auto split) for O / down, fp32 stores else
            epi, splits = (2, 0) if name in ("o", "down") else (1, 1)
            for _ in range(3):
                assert L.ck_gemm(P(W), P(X), P(out), None, M, N, K, N, epi, splits, ctas, st) == 0
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                assert L.ck_gemm(P(W), P(X), P(out), None, M, N, K, N, epi, splits, ctas, st) == 0
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / a.reps
            fl = 2.0 * M * N * K
            tot_f += fl
            tot_us += us
            share = (ctas or sms) / sms
            print(json.dumps({"M": M, "gemm": name, "N": N, "K": K, "ctas": ctas or sms, "us": round(us, 2),
                              "TFLOPs": round(fl / us / 1e6, 1),
                              "frac_burst": round(fl / us / 1e6 / pk["bf16_tflops"], 4),
                              "frac_partition_sustained": round(fl / us / 1e6 / (pk["bf16_tflops_sustained"] * share), 4)}),
                  flush=True)
            del W, X, out
        print(json.dumps({"M": M, "gemm": "layer", "ctas": ctas or sms, "TFLOPs": round(tot_f / tot_us / 1e6, 1)}), flush=True)
