"""Dev: per-CTA timeline of the weight-streaming GEMM (CRONUS_GEMM_PROBE=1), LLaMA3-8B shapes."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("CRONUS_GEMM_PROBE", "1")
import torch
from paper_2509_17357_b200._lib import lib
L = lib()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 108
p = lambda t: ctypes.c_void_p(t.data_ptr())
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, N, K in [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]:
    W = torch.randn(N, K, device="cuda").bfloat16()
    X = torch.randn(M, K, device="cuda").bfloat16()
    out = torch.zeros(M, N, device="cuda")
    for _ in range(3):
        assert L.ck_gemm(p(W), p(X), p(out), None, M, N, K, N, 2, 0, ctas, s) == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert L.ck_gemm(p(W), p(X), p(out), None, M, N, K, N, 2, 0, ctas, s) == 0
    e1.record()
    torch.cuda.synchronize()
    print(name, f"{e0.elapsed_time(e1)*1e3:.1f} us (event, incl. probe copy)", flush=True)
