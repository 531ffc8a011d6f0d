"""Dev probe: time single forward passes of chosen shapes (cheap target for ncu).

    python tools/kernel_probe.py [--reps N] [--only decode|chunk|ppi]
"""
import argparse, os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200.serving import GpuEngine

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--only", default=None)
ap.add_argument("--ppi-sms", type=int, default=40)
a = ap.parse_args()
cfg = open("tests/golden/configs/b200_llama8b_coloc.cfg").read()
eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=a.ppi_sms)
cases = {
    "decode": [dict(worker=1, n_dec=n, dec_ctx=c) for n in (8, 32, 64, 128) for c in (1024, 2048)],
    "chunk": [dict(worker=1, n_dec=n, dec_ctx=1024, chunk_len=512 - n, chunk_pos0=p) for n in (0, 32) for p in (0, 2048)],
    "ppi": [dict(worker=0, chunk_len=L) for L in (256, 1024, 2048, 4096)],
}
for name, lst in cases.items():
    if a.only and name != a.only:
        continue
    for kw in lst:
        ms = eng.time_pass(cfg, reps=a.reps, **kw)
        print(name, json.dumps(kw), f"{ms:.3f} ms", flush=True)
