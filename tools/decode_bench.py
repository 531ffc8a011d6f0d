"""Dev probe: decode paged attention alone, GB/s of algorithmic K/V bytes.

    python tools/decode_bench.py [--reps N] [--cluster C] [--trace-lens] [--planner engine|r1]

--trace-lens: context lengths of S random requests of the C2 trace (synth 1000/1014/247,
seed 1; input + a uniform share of the output) instead of S x ctx; --planner r1: the round-1
plan (parts of up to 2 x share x C blocks, sequence order) for comparison.

LLaMA3-8B layout (32 layers, 8 kv heads, 32 q heads, 16-token blocks, random block
tables over a zero-filled pool); each launch reads one layer, the layer rotates so
consecutive launches never hit data left in L2. Cluster plan = Batch::plan_decode (one
wave over 2 CTAs/SM). Prints one JSON line per shape.
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
ap.add_argument("--reps", type=int, default=64)
ap.add_argument("--shapes", default="1x1024,8x1024,8x2560,32x1024,64x1024,128x1024,32x4096,64x4096,16x16384")
ap.add_argument("--cluster", type=int, default=0, help="force the cluster size (0 = planner)")
ap.add_argument("--trace-lens", action="store_true")
ap.add_argument("--planner", default="engine", choices=["engine", "r1"])
ap.add_argument("--slots-per-sm", type=int, default=0, help="0: the engine's rule (3 from 64 pairs, else 2)")
ap.add_argument("--graph", action="store_true", help="time a captured CUDA graph of the launches (no host launch cost)")
a = ap.parse_args()

L = lib()
LAYERS, NKV, NQ = 32, 8, 32
SMS = torch.cuda.get_device_properties(0).multi_processor_count
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def plan(lens, slots):
    """The engine's plan (gpu::Batch::plan_decode through the C-ABI), or the round-1 rule."""
    if a.planner == "engine" and not a.cluster:
        from paper_2509_17357_b200.serving import plan_decode
        work, item0, C = plan_decode(lens, NKV, slots)
        return C, [int(x) for x in work], [int(x) for x in item0]
    total = sum((n + 15) // 16 for n in lens)
    work, item0 = [], []
    pairs = len(lens) * NKV
    C = 1
    while C < 16 and pairs * C * 2 <= slots and total * NKV >= pairs * C * 2 * 4:
        C *= 2
    C = a.cluster or C
    share = max(8, -(-total * NKV // slots))
    cap = 2 * share * C
    for s, n in enumerate(lens):
        item0.append(len(work))
        parts = max(1, -(-((n + 15) // 16) // cap))
        work += [(s << 16) | (parts << 8) | i for i in range(parts)]
    return C, work, item0


for shape in a.shapes.split(","):
    S, ctx = (int(x) for x in shape.split("x"))
    if a.trace_lens:
        import numpy as np
        from paper_2509_17357_b200 import engine as E
        tr = E.synth_trace(1000, 1014, 247, E.ALL_AT_ZERO, 0, 1)
        rng = np.random.default_rng(S)
        idx = rng.choice(1000, S, replace=False)
        lens = [int(x) for x in tr.input_len[idx] + (rng.random(S) * tr.output_len[idx]).astype(int)]
        ctx = int(np.mean(lens))
    else:
        lens = [ctx] * S
    nblk = sum((n + 15) // 16 for n in lens)
    pool = torch.zeros(nblk + 1, LAYERS, 2, NKV, 16, 128, dtype=torch.bfloat16, device="cuda")
    bt = torch.randperm(nblk, device="cuda").int()
    off = torch.tensor([0] + list(__import__("itertools").accumulate((n + 15) // 16 for n in lens))[:-1],
                       dtype=torch.int32, device="cuda")
    rows = torch.arange(S, dtype=torch.int32, device="cuda")
    lens_t = torch.tensor(lens, dtype=torch.int32, device="cuda")
    per_sm = a.slots_per_sm or (3 if S * NKV >= 64 else 2)
    bps, work, item0 = plan(lens, per_sm * SMS)
    work_t = torch.tensor(work, dtype=torch.int32, device="cuda")
    item0_t = torch.tensor(item0, dtype=torch.int32, device="cuda")
    q = torch.randn(S, NQ * 128, device="cuda").bfloat16()
    out = torch.empty_like(q)
    ws = torch.empty(len(work) * NQ * 130, device="cuda")
    tickets = torch.zeros(S * NKV, dtype=torch.int32, device="cuda")

    def launch(layer):
        rc = L.ck_attn_decode_tma(P(q), P(pool), pool.shape[0], P(bt), P(rows), P(lens_t), P(off), P(item0_t),
                                  P(work_t), len(work), S, bps, P(ws), P(tickets), P(out), NQ, NKV, layer, LAYERS,
                                  1 / math.sqrt(128), None, st)
        assert rc == 0, rc

    for i in range(8):
        launch(i % LAYERS)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.graph:  # the engine replays decode passes as graphs: time the device side alone
        cs = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cs):
            st = ctypes.c_void_p(cs.cuda_stream)
            for i in range(4):  # plain launches on the capture stream first (per-stream caches)
                launch(i % LAYERS)
            cs.synchronize()
            with torch.cuda.graph(g, stream=cs):
                for i in range(a.reps):
                    launch(i % LAYERS)
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
    else:
        e0.record()
        for i in range(a.reps):
            launch(i % LAYERS)
        e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    byts = sum(lens) * NKV * 2 * 128 * 2
    print(json.dumps({"planner": a.planner, "trace_lens": a.trace_lens, "max_len": max(lens),
                      "stages": os.environ.get("CRONUS_DEC_STAGES", "auto"), "seqs": S, "ctx": ctx,
                      "bps_or_cluster": bps, "ctas": len(work) * NKV * bps, "us": round(us, 2), "MB": round(byts / 1e6, 1),
                      "GBps": round(byts / us / 1e3, 1)}), flush=True)
    del pool
    torch.cuda.empty_cache()
