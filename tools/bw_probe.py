"""Dev: HBM read bandwidth by access pattern and CTA count (ck_bw_probe)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_17357_b200._lib import lib
L = lib()
nbytes = 4 << 30
buf = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda")
buf.uniform_(-1, 1)
s = torch.cuda.current_stream()
for mode, name in ((0, "ldg128"), (1, "tma2d_128x64"), (2, "bulk16k")):
    for ctas in (40, 108, 148, 296):
        ts = []
        for r in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = L.ck_bw_probe(ctypes.c_void_p(buf.data_ptr()), nbytes, mode, ctas, ctypes.c_void_p(s.cuda_stream))
            b.record()
            torch.cuda.synchronize()
            assert rc == 0, rc
            if r:
                ts.append(a.elapsed_time(b))
        ts.sort()
        print(f"{name:14s} ctas={ctas:4d} {nbytes / (ts[len(ts)//2] / 1e3) / 1e9:8.1f} GB/s", flush=True)
