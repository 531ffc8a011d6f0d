"""Dev: per-pass time of mixed CPI passes (prefill chunk + decoders); CRONUS_PASS_STATS=1 for the split."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200.serving import GpuEngine
cfg = open("tests/golden/configs/b200_llama8b_coloc.cfg").read()
eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=40)
out = {}
for (nd, ctx, cl, p0) in [(0, 0, 512, 0), (0, 0, 512, 2048), (32, 1024, 480, 512), (96, 1024, 416, 512), (64, 1500, 448, 1024)]:
    out[f"{nd}x{ctx}+{cl}@{p0}"] = round(eng.time_pass(cfg, 1, n_dec=nd, dec_ctx=ctx, chunk_len=cl, chunk_pos0=p0, reps=10), 3)
print(json.dumps(out), flush=True)
eng.close()
