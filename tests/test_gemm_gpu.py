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
