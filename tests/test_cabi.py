"""The C-ABI library (libcronus_b200.so) loads on a CPU-only machine and exports every
entry point declared in include/*.h (no device calls here)."""
import ctypes
import glob
import os
import re

from conftest import ROOT


def declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[\w\s\*]+?\b(\w+)\s*\(", text, flags=re.M):
            if m.group(1) not in ("if", "defined"):
                names.add(m.group(1))
    return names


def test_every_declared_symbol_is_exported():
    from paper_2509_17357_b200._lib import lib
    L = lib()
    names = declared()
    assert {"ck_gemm", "ck_attn_decode_tma", "ck_attn_prefill_pp", "cronus_run_virtual", "cronus_engine_serve"} <= names
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, missing


def test_version_and_errors_without_gpu():
    from paper_2509_17357_b200._lib import lib
    L = lib()
    assert b"sm_100a" in L.cronus_version()
    out = ctypes.c_void_p()
    rc = L.cronus_config_roundtrip(b"bogus = 1\n", ctypes.byref(out))
    assert rc == 2 and b"unknown key" in L.cronus_last_error()


def test_kernel_layer_is_sm100a_only():
    # the library carries sm_100a SASS (tcgen05 / TMA) and nothing for other targets
    import subprocess
    so = os.path.join(ROOT, "paper_2509_17357_b200", "libcronus_b200.so")
    r = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True)
    if r.returncode != 0:
        return  # cuobjdump unavailable
    assert "sm_100a" in r.stdout and "sm_90" not in r.stdout
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass and "UTMALDG" in sass  # tcgen05.mma and TMA tensor loads


def test_gemm_fuse_argument_checks_without_gpu():
    """ck_gemm_fused rejects fused-finalize requests it cannot honour before any device call
    (include/cronus_ck.h): the fp32 finalize needs tickets and a non-bf16 epilogue; the fused
    RMSNorm needs the residual stream-K epilogue (CK_EPI_RED_F32, splits 0), its row tickets,
    gamma and output, and rows of at most 4096."""
    from paper_2509_17357_b200._lib import lib

    class Fuse(ctypes.Structure):
        _fields_ = [("kind", ctypes.c_int), ("zero_after", ctypes.c_int), ("tickets", ctypes.c_void_p),
                    ("q_out", ctypes.c_void_p), ("kv_pool", ctypes.c_void_p), ("bt", ctypes.c_void_p),
                    ("row_bt", ctypes.c_void_p), ("row_pos", ctypes.c_void_p), ("cos_tab", ctypes.c_void_p),
                    ("sin_tab", ctypes.c_void_p), ("nq", ctypes.c_int), ("nkv", ctypes.c_int),
                    ("layer", ctypes.c_int), ("n_layers", ctypes.c_int), ("act", ctypes.c_void_p),
                    ("gamma", ctypes.c_void_p), ("norm_out", ctypes.c_void_p), ("eps", ctypes.c_float),
                    ("zero_cols", ctypes.c_int), ("zero", ctypes.c_void_p), ("row_tickets", ctypes.c_void_p)]

    L = lib()
    d = ctypes.c_void_p(1 << 20)  # never dereferenced: every case fails validation first
    EINVAL = 1  # cudaErrorInvalidValue
    ok = dict(kind=3, tickets=d.value, gamma=d.value, norm_out=d.value, eps=1e-5, row_tickets=d.value)

    def call(f, N=4096, epi=2, splits=0):
        return L.ck_gemm_fused(d, d, d, None, 8, N, 4096, epi, splits, 0, ctypes.byref(f), None)

    assert call(Fuse(**ok), epi=0) == EINVAL                      # bf16 epilogue cannot be finalized
    assert call(Fuse(**{**ok, "tickets": None})) == EINVAL        # no tile tickets
    assert call(Fuse(**ok), splits=1) == EINVAL                   # not stream-K
    assert call(Fuse(**ok), epi=1) == EINVAL                      # not the residual red.add
    assert call(Fuse(**{**ok, "row_tickets": None})) == EINVAL
    assert call(Fuse(**{**ok, "gamma": None})) == EINVAL
    assert call(Fuse(**ok), N=8192) == EINVAL                     # rows longer than 4096
    assert call(Fuse(**{**ok, "zero": d.value, "zero_cols": 6}), N=4096) == EINVAL
