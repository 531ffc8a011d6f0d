"""Dev: run exactly one warm + one measured forward pass of a given shape (ncu target)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200.serving import GpuEngine
ap = argparse.ArgumentParser()
ap.add_argument("--worker", type=int, default=1)
ap.add_argument("--n-dec", type=int, default=32)
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--pos0", type=int, default=0)
a = ap.parse_args()
cfg = open("tests/golden/configs/b200_llama8b_coloc.cfg").read()
eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=40)
print(eng.time_pass(cfg, a.worker, n_dec=a.n_dec, dec_ctx=a.ctx, chunk_len=a.chunk, chunk_pos0=a.pos0, reps=1))
