"""tcgen05 GEMM (ck_gemm) against a torch fp32 reference of the same op.

Tolerance: inputs are bf16, accumulation fp32 in both; differences come only from
summation order (and the final bf16 rounding for CK_EPI_BF16):
    |got - ref| <= 1e-3 * sqrt(K) * rms(ref) + 1e-2 * |ref|   (bf16 output)
    |got - ref| <= 1e-4 * sqrt(K) * rms(ref) + 1e-5 * |ref|   (fp32 output)
"""
import ctypes

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EPI_BF16, EPI_F32, EPI_RED = 0, 1, 2


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_17357_b200._lib import lib
    return lib()


def p(t):
    return ctypes.c_void_p(t.data_ptr())


def run_gemm(L, W, X, out, M, N, K, epi, splits=1, bias=None, max_ctas=0):
    s = torch.cuda.current_stream().cuda_stream
    rc = L.ck_gemm(p(W), p(X), p(out), p(bias) if bias is not None else None, M, N, K, N, epi, splits, max_ctas,
                   ctypes.c_void_p(s))
    assert rc == 0, f"ck_gemm rc={rc}"
    torch.cuda.synchronize()


def check(got, ref, K, bf16_out):
    err = (got.float() - ref).abs()
    rms = ref.pow(2).mean().sqrt().item() + 1e-6
    tol = (1e-3 if bf16_out else 1e-4) * (K ** 0.5) * rms + (1e-2 if bf16_out else 1e-5) * ref.abs()
    bad = (err > tol)
    assert not bad.any(), f"max err {err.max().item():.4g} (rms {rms:.4g}), {bad.sum().item()} bad"


@pytest.mark.parametrize("M", [1, 7, 32, 33, 64, 100, 128, 129, 256, 300, 512, 1000])
@pytest.mark.parametrize("N,K", [(128, 64), (384, 256), (1024, 1024)])
def test_gemm_store(L, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    ref = X.float() @ W.float().t()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    run_gemm(L, W, X, out, M, N, K, EPI_BF16)
    check(out, ref, K, True)
    out32 = torch.empty(M, N, device="cuda", dtype=torch.float32)
    run_gemm(L, W, X, out32, M, N, K, EPI_F32)
    check(out32, ref, K, False)


@pytest.mark.parametrize("M", [1, 16, 48, 128, 200])
@pytest.mark.parametrize("splits", [0, 1, 3, 8])
def test_gemm_splitk_red(L, M, splits):
    N, K = 768, 2048
    g = torch.Generator(device="cuda").manual_seed(M + splits)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    base = torch.randn(M, N, device="cuda", generator=g)
    ref = base + X.float() @ W.float().t()
    out = base.clone()
    run_gemm(L, W, X, out, M, N, K, EPI_RED, splits=splits)
    check(out, ref, K, False)


def test_gemm_bias_and_llama_shapes(L):
    # LLaMA3-8B QKV projection at a decode batch and a chunk batch, with a bias vector.
    N, K = 6144, 4096
    g = torch.Generator(device="cuda").manual_seed(5)
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.02).bfloat16()
    bias = (torch.randn(N, device="cuda", generator=g) * 0.1).bfloat16()
    for M in (40, 512):
        X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
        ref = X.float() @ W.float().t() + bias.float()
        out = torch.empty(M, N, device="cuda", dtype=torch.float32)
        run_gemm(L, W, X, out, M, N, K, EPI_F32, bias=bias)
        check(out, ref, K, False)


def test_gemm_capped_grid(L):
    # the PPI runs on an SM subset: persistence must cover every unit with a small grid
    N, K, M = 1024, 512, 300
    W = (torch.randn(N, K, device="cuda") * 0.05).bfloat16()
    X = torch.randn(M, K, device="cuda").bfloat16()
    ref = X.float() @ W.float().t()
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    run_gemm(L, W, X, out, M, N, K, EPI_F32, max_ctas=5)
    check(out, ref, K, False)


class Fuse(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("zero_after", ctypes.c_int), ("tickets", ctypes.c_void_p),
                ("q_out", ctypes.c_void_p), ("kv_pool", ctypes.c_void_p), ("bt", ctypes.c_void_p),
                ("row_bt", ctypes.c_void_p), ("row_pos", ctypes.c_void_p), ("cos_tab", ctypes.c_void_p),
                ("sin_tab", ctypes.c_void_p), ("nq", ctypes.c_int), ("nkv", ctypes.c_int), ("layer", ctypes.c_int),
                ("n_layers", ctypes.c_int), ("act", ctypes.c_void_p), ("gamma", ctypes.c_void_p),
                ("norm_out", ctypes.c_void_p), ("eps", ctypes.c_float), ("zero_cols", ctypes.c_int),
                ("zero", ctypes.c_void_p), ("row_tickets", ctypes.c_void_p)]


@pytest.mark.parametrize("M", [3, 32, 100, 300])
def test_gemm_fused_silu_matches_unfused(L, M):
    """gate_up GEMM + SiLU*up finalized by the last CTA of each tile (tickets)."""
    F, K = 512, 1024
    W = (torch.randn(2 * F, K, device="cuda") * 0.05).bfloat16()
    X = torch.randn(M, K, device="cuda").bfloat16()
    small = M <= 128
    acc = torch.zeros(M, 2 * F, device="cuda")
    act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    tickets = torch.zeros(4096, dtype=torch.int32, device="cuda")
    f = Fuse(kind=2, zero_after=1 if small else 0, tickets=tickets.data_ptr(), act=act.data_ptr())
    s = torch.cuda.current_stream().cuda_stream
    rc = L.ck_gemm_fused(p(W), p(X), p(acc), None, M, 2 * F, K, EPI_RED if small else EPI_F32, 0 if small else 1, 0,
                         ctypes.byref(f), ctypes.c_void_p(s))
    assert rc == 0
    torch.cuda.synchronize()
    gu = X.float() @ W.float().t()
    ref = torch.nn.functional.silu(gu[:, 0::2]) * gu[:, 1::2]
    assert torch.allclose(act.float(), ref, rtol=2e-2, atol=2e-2)
    assert tickets.abs().sum() == 0
    if small:
        assert acc.abs().sum() == 0  # accumulator cleared for reuse


@pytest.mark.parametrize("M", [5, 64, 200])
def test_gemm_fused_qkv_rope_matches_unfused(L, M):
    nq, nkv, H, layers, layer = 4, 2, 512, 2, 1
    Q = (nq + 2 * nkv) * 128
    g = torch.Generator(device="cuda").manual_seed(M)
    W = (torch.randn(Q, H, device="cuda", generator=g) * 0.05).bfloat16()
    X = torch.randn(M, H, device="cuda", generator=g).bfloat16()
    bias = (0.1 * torch.randn(Q, device="cuda", generator=g)).bfloat16()
    small = M <= 128
    nb = 64
    pos = torch.randperm(1000, device="cuda", generator=g)[:M].int()
    perm = torch.randperm(nb, device="cuda", generator=g).int()
    bt = perm.repeat(M)
    row_bt = torch.arange(M, device="cuda", dtype=torch.int32) * nb
    c = torch.empty(2048 * 64, device="cuda"); sn = torch.empty(2048 * 64, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.ck_rope_table(p(c), p(sn), 2048, 10000.0, st) == 0
    outs = []
    for fused in (False, True):
        pool = torch.zeros(nb, layers, 2, nkv, 16, 128, dtype=torch.bfloat16, device="cuda")
        acc = torch.zeros(M, Q, device="cuda")
        q_out = torch.empty(M, nq * 128, dtype=torch.bfloat16, device="cuda")
        epi = EPI_RED if small else EPI_F32
        if fused:
            tickets = torch.zeros(4096, dtype=torch.int32, device="cuda")
            f = Fuse(kind=1, zero_after=1 if small else 0, tickets=tickets.data_ptr(), q_out=q_out.data_ptr(),
                     kv_pool=pool.data_ptr(), bt=bt.data_ptr(), row_bt=row_bt.data_ptr(), row_pos=pos.data_ptr(),
                     cos_tab=c.data_ptr(), sin_tab=sn.data_ptr(), nq=nq, nkv=nkv, layer=layer, n_layers=layers)
            assert L.ck_gemm_fused(p(W), p(X), p(acc), p(bias), M, Q, H, epi, 0 if small else 1, 0, ctypes.byref(f),
                                   st) == 0
        else:
            assert L.ck_gemm(p(W), p(X), p(acc), p(bias), M, Q, H, Q, epi, 0 if small else 1, 0, st) == 0
            assert L.ck_qkv_rope_append(p(acc), None, p(q_out), p(pool), p(bt), p(row_bt), p(pos), p(c), p(sn), M,
                                        nq, nkv, layer, layers, 1 if small else 0, st) == 0
        torch.cuda.synchronize()
        outs.append((q_out.float(), pool.float()))
    assert torch.allclose(outs[0][0], outs[1][0], rtol=1e-2, atol=1e-2)
    assert torch.allclose(outs[0][1], outs[1][1], rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M", [129, 300, 512, 1000])
def test_gemm_silu_epilogue(L, M):
    """CK_EPI_SILU_BF16: interleaved gate/up weight rows -> bf16 silu(gate) * up, written
    straight from the accumulator (tensor regime, whole tiles per CTA)."""
    g = torch.Generator(device="cuda").manual_seed(M)
    F, K = 640, 512
    W = (torch.randn(2 * F, K, device="cuda", generator=g) * 0.05).bfloat16()
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    act = torch.full((M, F), float("nan"), device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    assert L.ck_gemm_fused(p(W), p(X), p(act), None, M, 2 * F, K, 3, 1, 0, None, ctypes.c_void_p(s)) == 0
    torch.cuda.synchronize()
    ref = X.float() @ W.float().t()
    want = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
    assert torch.allclose(act.float(), want, rtol=2e-2, atol=2e-2), (act.float() - want).abs().max().item()
    bad = L.ck_gemm_fused(p(W), p(X), p(act), None, M, 2 * F, K, 3, 0, 0, None, ctypes.c_void_p(s))
    assert bad != 0  # split-K / stream-K cannot fuse the gate-up pairing


@pytest.mark.parametrize("M,F,K,ctas", [(200, 1024, 512, 12), (512, 1024, 4096, 13), (300, 640, 1024, 7),
                                        (512, 14336, 4096, 148), (512, 14336, 4096, 108)])
def test_gemm_silu_hybrid(L, M, F, K, ctas):
    """Hybrid SiLU GEMM (splits 0 + CK_FUSE_SILU): whole tiles write silu(gate) * up from
    TMEM, the tiles of a sparse last wave run as stream-K pieces red.added into the zeroed
    fp32 accumulator and finalized by the tile's last piece; the accumulator is left zero.
    Cases: pieces of whole tiles (K=512), pieces straddling tiles (K=4096), LLaMA3-8B gate_up
    at 512 rows on 148 and 108 SMs (448 tiles: last waves of 4 and 16 tiles)."""
    g = torch.Generator(device="cuda").manual_seed(M + F)
    W = (torch.randn(2 * F, K, device="cuda", generator=g) * 0.05).bfloat16()
    X = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    acc = torch.zeros(M, 2 * F, device="cuda")
    act = torch.full((M, F), float("nan"), device="cuda", dtype=torch.bfloat16)
    tickets = torch.zeros(8192, dtype=torch.int32, device="cuda")
    f = Fuse(kind=2, zero_after=1, tickets=tickets.data_ptr(), act=act.data_ptr())
    s = torch.cuda.current_stream().cuda_stream
    assert L.ck_gemm_fused(p(W), p(X), p(acc), None, M, 2 * F, K, 3, 0, ctas, ctypes.byref(f), ctypes.c_void_p(s)) == 0
    torch.cuda.synchronize()
    ref = X.float() @ W.float().t()
    ref = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
    assert torch.allclose(act.float(), ref, rtol=2e-2, atol=2e-2), (act.float() - ref).abs().max().item()
    assert tickets.abs().sum() == 0
    assert acc.abs().sum() == 0


@pytest.mark.parametrize("M,H,K,ctas", [(1, 4096, 4096, 0), (8, 4096, 4096, 108), (16, 4096, 14336, 148),
                                        (13, 3584, 18944, 108), (5, 256, 512, 7), (100, 4096, 4096, 0)])
def test_gemm_residual_rmsnorm_fuse(L, M, H, K, ctas):
    """CK_FUSE_RMSNORM: residual stream-K GEMM x += A W^T whose m-tile's last finished tile
    writes rmsnorm(x) * gamma (bf16) — the next norm without a launch; each tile clears
    its slice of the `zero` accumulator. Shapes: LLaMA3-8B O / down at 1-16 decode rows,
    Qwen2-7B down (H = 3584), tiny, and 100 rows. Tickets are left zero, and a second
    call on the same tickets gives the same result (self-resetting)."""
    g = torch.Generator(device="cuda").manual_seed(M * 7 + K)
    W = (torch.randn(H, K, device="cuda", generator=g) * 0.02).bfloat16()
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    x0 = torch.randn(M, H, device="cuda", generator=g)
    gamma = (1.0 + 0.1 * torch.randn(H, device="cuda", generator=g)).bfloat16()
    ref_x = x0 + A.float() @ W.float().t()
    ref_h = ref_x * torch.rsqrt(ref_x.pow(2).mean(-1, keepdim=True) + 1e-5) * gamma.float()
    tickets = torch.zeros(4096, dtype=torch.int32, device="cuda")
    rows = torch.zeros(64, dtype=torch.int32, device="cuda")
    Z = 6144
    for _ in range(2):
        x = x0.clone()
        h = torch.full((M, H), float("nan"), device="cuda", dtype=torch.bfloat16)
        zero = torch.ones(M, Z, device="cuda")
        f = Fuse(kind=3, tickets=tickets.data_ptr(), gamma=gamma.data_ptr(), norm_out=h.data_ptr(), eps=1e-5,
                 zero=zero.data_ptr(), zero_cols=Z, row_tickets=rows.data_ptr())
        s = torch.cuda.current_stream().cuda_stream
        assert L.ck_gemm_fused(p(W), p(A), p(x), None, M, H, K, EPI_RED, 0, ctas, ctypes.byref(f),
                               ctypes.c_void_p(s)) == 0
        torch.cuda.synchronize()
        check(x, ref_x, K, False)
        assert torch.allclose(h.float(), ref_h, rtol=1.6e-2, atol=1e-2), (h.float() - ref_h).abs().max().item()
        assert zero.abs().sum() == 0
        assert tickets.abs().sum() == 0 and rows.abs().sum() == 0
    # the fuse needs the residual stream-K epilogue and rows of <= 4096
    bad = Fuse(kind=3, tickets=tickets.data_ptr(), gamma=gamma.data_ptr(), norm_out=h.data_ptr(), eps=1e-5,
               row_tickets=rows.data_ptr())
    assert L.ck_gemm_fused(p(W), p(A), p(x), None, M, H, K, EPI_RED, 1, ctas, ctypes.byref(bad), None) != 0
