"""Dev probe: prefill / chunk attention kernel alone at serve shapes (LLaMA3-8B heads:
32 q / 8 kv, head dim 128), CUDA-event timed over back-to-back launches.

    python tools/prefill_probe.py [--shapes 448x1024,200x0,...] [--reps N] [--nq 32 --nkv 8]

Shape QxP = a chunk of Q query rows at prefix P (keys [0, P+Q), causal). Prints one JSON
line per shape: us per launch, algorithmic TFLOP/s (4 * nq * 128 * sum of keys), and the
fraction of the device's measured bf16 peak.
"""
import argparse
import ctypes
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200._lib import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="448x1024,448x0,448x3072,200x0,1024x0,2048x0,64x1024,4096x0")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--nq", type=int, default=32)
ap.add_argument("--nkv", type=int, default=8)
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--ctas", type=int, default=0, help="partition CTAs for key splitting (0: the device's SMs; -1: never split)")
a = ap.parse_args()

L = lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["bf16_tflops"]
except Exception:
    peak = 1590.0
for shape in a.shapes.split(","):
    q_len, pos0 = (int(x) for x in shape.split("x"))
    T = pos0 + q_len
    nblk = (T + 15) // 16
    pool = torch.randn(nblk + 2, a.layers, 2, a.nkv, 16, 128, device="cuda").bfloat16()
    bt = torch.randperm(nblk, device="cuda").int()
    q = torch.randn(q_len, a.nq * 128, device="cuda").bfloat16()
    out = torch.empty_like(q)
    ctas = torch.cuda.get_device_properties(0).multi_processor_count if a.ctas == 0 else max(a.ctas, 0)
    ws = torch.empty(max(1, L.ck_attn_prefill_ws_floats(ctas)), device="cuda")
    tickets = torch.zeros(max(1, ctas), dtype=torch.int32, device="cuda")

    def launch():
        rc = L.ck_attn_prefill_pp(P(q), q_len, P(pool), pool.shape[0], P(bt), 0, q_len, pos0, P(out), a.nq, a.nkv, 0,
                                  a.layers, 1 / math.sqrt(128), P(ws) if ctas else None, P(tickets), ctas, st)
        assert rc == 0, rc

    for _ in range(5):
        launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        launch()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    keys = q_len * pos0 + q_len * (q_len + 1) / 2
    flops = 4.0 * a.nq * 128 * keys
    print(json.dumps({"ctas": ctas, "q_len": q_len, "pos0": pos0, "us": round(us, 2), "TFLOPs": round(flops / us / 1e6, 1),
                      "frac_peak": round(flops / us / 1e6 / peak, 4)}), flush=True)
    del pool
    torch.cuda.empty_cache()
