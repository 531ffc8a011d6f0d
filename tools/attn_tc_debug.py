"""Dev: run one tcgen05 prefill-attention case and report (watchdog prints on deadlock)."""
import ctypes, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_17357_b200._lib import lib
L = lib()
pos0, qlen, nq, nkv = (int(x) for x in sys.argv[1:5])
layers, layer = 2, 0
T = pos0 + qlen
nb = (T + 15) // 16 + 5
pool = torch.zeros(nb, layers, 2, nkv, 16, 128, dtype=torch.bfloat16, device="cuda")
pool.normal_()
table = torch.randperm(nb, device="cuda")[: (T + 15) // 16].int()
q = torch.randn(qlen + 5, nq * 128, device="cuda").bfloat16()
out = torch.zeros_like(q)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
rc = L.ck_attn_prefill_tc(ctypes.c_void_p(q.data_ptr()), q.shape[0], ctypes.c_void_p(pool.data_ptr()), nb,
                          ctypes.c_void_p(table.data_ptr()), 2, qlen, pos0, ctypes.c_void_p(out.data_ptr()), nq, nkv,
                          layer, layers, 1 / math.sqrt(128), s)
print("rc", rc, flush=True)
torch.cuda.synchronize()
print("ok", out.float().abs().mean().item())
