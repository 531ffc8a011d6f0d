"""Dev probe: device timeline of one forward pass via CUPTI (torch.profiler).

    python tools/timeline.py [--n-dec 8] [--ctx 1024] [--chunk 0] [--worker 1] [--json out.json]

Runs EngineHandle.time_pass under torch.profiler (CUPTI kernel activity sees every
kernel our library launches), then prints, per kernel class, launches, mean duration
and mean gap to the previous kernel's end, plus the pass's busy/idle split. Kernel
"duration" includes time spent resident at griddepcontrol.wait under PDL.
"""
import argparse
import collections
import json
import os
import re
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200.serving import GpuEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n-dec", type=int, default=8)
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--pos0", type=int, default=0)
ap.add_argument("--worker", type=int, default=1)
ap.add_argument("--ppi-sms", type=int, default=40)
ap.add_argument("--json", default=None)
a = ap.parse_args()

cfg = open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "configs", "b200_llama8b_coloc.cfg")).read()
eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=a.ppi_sms)
kw = dict(worker=a.worker, n_dec=a.n_dec, dec_ctx=a.ctx, chunk_len=a.chunk, chunk_pos0=a.pos0)
eng.time_pass(cfg, reps=3, **kw)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ms = eng.time_pass(cfg, reps=1, **kw)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = []
for e in evs:
    name = e.name
    if "memcpy" in name.lower() or "memset" in name.lower():
        cls = "memcpy/memset"
    else:
        m = re.search(r"(\w+_kernel)(<[^>]*>)?", name)
        cls = (m.group(1) + (m.group(2) or "")) if m else name[:40]
    ks.append((e.time_range.start, e.time_range.end, cls))
ks.sort()
# keep the last pass only: time_pass(reps=1) may run warm-up passes too; split on big gaps
t0, t1 = ks[0][0], max(k[1] for k in ks)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
crit = collections.defaultdict(float)
prev_end = ks[0][0]
busy = 0.0
cur_s, cur_e = ks[0][0], ks[0][1]
for s, e, c in ks:
    agg[c][0] += 1
    agg[c][1] += e - s
    agg[c][2] += max(0.0, s - prev_end)
    crit[c] += max(0.0, e - max(prev_end, s))  # time this launch adds to the chain
    prev_end = max(prev_end, e)
    if s > cur_e:
        busy += cur_e - cur_s
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
span = t1 - t0
out = {"pass_ms_reported": ms, "span_us": round(span, 1), "busy_us": round(busy, 1), "idle_us": round(span - busy, 1),
       "kernels": len(ks), "classes": {}}
for c, (n, d, g) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out["classes"][c] = {"n": n, "mean_us": round(d / n, 2), "total_us": round(d, 1), "mean_gap_us": round(g / n, 2),
                         "crit_us_per_launch": round(crit[c] / n, 2), "crit_total_us": round(crit[c], 1)}
print(json.dumps(out, indent=1))
if a.json:
    json.dump({"summary": out, "kernels": [(round(s - t0, 2), round(e - t0, 2), c) for s, e, c in ks]},
              open(a.json, "w"))
