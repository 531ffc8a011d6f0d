"""Dev: per-pass time of decode-only CPI passes (run with CRONUS_MEGA=0/1).

    python tools/pass_sweep.py [model] [NxCTX ...]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200.serving import GpuEngine
cfg = open("tests/golden/configs/b200_llama8b_coloc.cfg").read()
model = sys.argv[1] if len(sys.argv) > 1 else "llama3-8b"
shapes = sys.argv[2:] or [f"{n}x{c}" for c in (512, 2048) for n in (1, 8, 16, 32, 48, 64)]
eng = GpuEngine(model=model, clock="wall", ppi_sms=int(os.environ.get("PPI_SMS", "40")),
                decode_forward="persistent" if os.environ.get("CRONUS_MEGA") == "1" else "layered")
out = {}
for sh in shapes:
    n, ctx = map(int, sh.split("x"))
    out[sh] = round(eng.time_pass(cfg, 1, n_dec=n, dec_ctx=ctx, chunk_len=0, chunk_pos0=0, reps=20), 3)
print("mega", os.environ.get("CRONUS_MEGA", "0"), "pf", os.environ.get("CRONUS_MEGA_PF", "-"), json.dumps(out), flush=True)
eng.close()
