"""ctypes signatures of the C-ABI kernel layer (include/cronus_ck.h) and the GPU
engine entry points (include/cronus_gpu.h)."""
import ctypes

V = ctypes.c_void_p
I = ctypes.c_int
LL = ctypes.c_longlong
ULL = ctypes.c_ulonglong
F = ctypes.c_float
D = ctypes.c_double

CK = {
    "ck_gemm": [V, V, V, V, I, I, I, I, I, I, I, V],
    "ck_gemm_fused": [V, V, V, V, I, I, I, I, I, I, V, V],
    "ck_init_uniform": [V, LL, ULL, ULL, F, F, V],
    "ck_prompt_tokens": [V, V, V, I, ULL, I, V],
    "ck_rope_table": [V, V, I, D, V],
    "ck_embed": [V, V, V, V, V, V, V, V, I, I, V],
    "ck_rmsnorm": [V, V, V, V, I, I, F, V, I, V],
    "ck_qkv_rope_append": [V, V, V, V, V, V, V, V, V, I, I, I, I, I, I, V],
    "ck_attn_decode_tma": [V, V, LL, V, V, V, V, V, V, I, I, I, V, V, V, I, I, I, I, F, V, V],
    "ck_attn_prefill_pp": [V, I, V, LL, V, I, I, I, V, I, I, I, I, F, V, V, I, V],
    "ck_silu_mul": [V, V, I, I, I, V],
    "ck_argmax_emit": [V, I, I, V, V, V, V, V, V, I, V, V],
    "ck_kv_copy": [V, V, V, V, I, LL, V],
    "ck_copy_token": [V, LL, V, LL, V, LL, V],
    "ck_device_sms": [],
    "ck_smid_probe": [V, I, V],
    "ck_bw_probe": [V, LL, I, I, V],
}


def bind(L):
    for name, args in CK.items():
        fn = getattr(L, name, None)
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = I
    if hasattr(L, "ck_attn_prefill_ws_floats"):
        L.ck_attn_prefill_ws_floats.argtypes = [I]
        L.ck_attn_prefill_ws_floats.restype = LL
    try:
        from . import _engine_sigs
        _engine_sigs.bind(L)
    except ImportError:
        pass
