"""Dev probe: decode paged attention alone, GB/s of algorithmic K/V bytes.

    python tools/decode_bench.py [--reps N] [--cluster C]

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
a = ap.parse_args()

L = lib()
LAYERS, NKV, NQ = 32, 8, 32
SMS = torch.cuda.get_device_properties(0).multi_processor_count
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def plan(lens, slots):
    """Batch::plan_decode (cluster plan)."""
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
        work += [(s << 16) | i for i in range(parts)]
    item0.append(len(work))
    return C, work, item0


for shape in a.shapes.split(","):
    S, ctx = (int(x) for x in shape.split("x"))
    lens = [ctx] * S
    nblk = sum((n + 15) // 16 for n in lens)
    pool = torch.zeros(nblk + 1, LAYERS, 2, NKV, 16, 128, dtype=torch.bfloat16, device="cuda")
    bt = torch.randperm(nblk, device="cuda").int()
    off = torch.tensor([i * (ctx // 16) for i in range(S)], dtype=torch.int32, device="cuda")
    rows = torch.arange(S, dtype=torch.int32, device="cuda")
    lens_t = torch.tensor(lens, dtype=torch.int32, device="cuda")
    bps, work, item0 = plan(lens, 2 * SMS)
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
    e0.record()
    for i in range(a.reps):
        launch(i % LAYERS)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    byts = S * ctx * NKV * 2 * 128 * 2
    print(json.dumps({"stages": os.environ.get("CRONUS_DEC_STAGES", "3"), "seqs": S, "ctx": ctx,
                      "bps_or_cluster": bps, "ctas": len(work) * NKV * bps, "us": round(us, 2), "MB": round(byts / 1e6, 1),
                      "GBps": round(byts / us / 1e3, 1)}), flush=True)
    del pool
    torch.cuda.empty_cache()
