"""Dev: fixed cost vs size of weight-sized streams (ck_bw_probe TMA mode, 108 CTAs)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_17357_b200._lib import lib
L = lib()
buf = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
buf.uniform_(-1, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for mb in (8, 16, 34, 50, 120, 240, 960):
    for mode in (1, 2):
        nbytes = mb << 20
        ts = []
        for r in range(8):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = L.ck_bw_probe(ctypes.c_void_p(buf.data_ptr()), nbytes, mode, 108, ctypes.c_void_p(s.cuda_stream))
            b.record()
            torch.cuda.synchronize()
            if r:
                ts.append(a.elapsed_time(b))
        ts.sort()
        t = ts[len(ts) // 2]
        print(f"mode={mode} {mb:5d} MB  {t*1e3:8.1f} us  {nbytes / (t / 1e3) / 1e9:7.1f} GB/s", flush=True)
