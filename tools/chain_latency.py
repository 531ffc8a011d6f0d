"""Dev probe: per-boundary latency of a PDL-chained sequence of tiny dependent kernels
(ck_rmsnorm on 1 or 148 rows of 128 floats), i.e. the floor each kernel boundary adds. The
stream is held by a spin kernel while the host enqueues, so host launch cost is excluded."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200._lib import lib

L = lib()
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for rows in (1, 148):
    x = torch.randn(rows, 128, device="cuda")
    g = torch.ones(128, device="cuda").bfloat16()
    out = torch.empty(rows, 128, device="cuda").bfloat16()
    for _ in range(10):
        L.ck_rmsnorm(P(x), P(g), P(out), None, rows, 128, 1e-5, None, 0, st)
    n = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    L.ck_spin(30000, st)  # hold the stream while the host enqueues the whole chain
    e0.record()
    for _ in range(n):
        L.ck_rmsnorm(P(x), P(g), P(out), None, rows, 128, 1e-5, None, 0, st)
    e1.record()
    torch.cuda.synchronize()
    print(f"rows={rows}: {e0.elapsed_time(e1) * 1e3 / n:.2f} us per chained kernel "
          f"(PDL {'off' if os.environ.get('CRONUS_NO_PDL') == '1' else 'on'})")

# the same chain captured in a CUDA graph (programmatic edges kept), replayed
for rows in (1, 148):
    x = torch.randn(rows, 128, device="cuda")
    g = torch.ones(128, device="cuda").bfloat16()
    out = torch.empty(rows, 128, device="cuda").bfloat16()
    n = 500
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        sp = ctypes.c_void_p(s.cuda_stream)
        L.ck_rmsnorm(P(x), P(g), P(out), None, rows, 128, 1e-5, None, 0, sp)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            for _ in range(n):
                L.ck_rmsnorm(P(x), P(g), P(out), None, rows, 128, 1e-5, None, 0, sp)
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"graph rows={rows}: {e0.elapsed_time(e1) * 1e3 / (4 * n):.2f} us per chained kernel")
