"""B200 calibration: measure the workers, fit the paper's linear cost models, emit a config.

Mirror of the reference's `cronus_sim calibrate` (proj/tools/cronus_sim.cpp:186-244) and
of the paper's methodology: samples of PPI prefill time vs length and
CPI iteration time vs (prefill context, decode context sum) are timed with CUDA events on
the real workers (GpuEngine.time_pass), fitted with fit_prefill / fit_chunked (costmodel.cpp:
94-113 semantics, here through libcronus_b200.so), and written as a ClusterConfig whose
profiles the balancer then uses on the wall clock.

    python -m paper_2509_17357_b200.calibrate --model llama3-8b --ppi-sms 40 \\
        --out tests/golden/configs/b200_llama8b_coloc.cfg
"""
from __future__ import annotations

import argparse
import json
import os
import sys

from . import engine as E


def samples(eng, cfg_text, max_prefill=4096):
    pre = []
    for L in (16, 64, 128, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096):
        if L > max_prefill:
            break
        pre.append((L, eng.time_pass(cfg_text, 0, chunk_len=L, reps=3)))
    chk = []
    for n_dec in (0, 8, 32, 64, 128):
        for ctx in (512, 1536):
            if n_dec == 0 and ctx != 512:
                continue
            for chunk in (0, 128, 512 - n_dec):
                for pos0 in (0, 1024):
                    if chunk == 0 and (n_dec == 0 or pos0):
                        continue
                    ms = eng.time_pass(cfg_text, 1, n_dec=n_dec, dec_ctx=ctx, chunk_len=chunk, chunk_pos0=pos0, reps=3)
                    chk.append((pos0 + chunk if chunk else 0, n_dec * ctx, ms, n_dec, chunk))
    return pre, chk


def build_config(base_cfg: str, pre_fit, chk_fit, names, caps, link) -> str:
    (kp, bp), _, _ = pre_fit
    (kc, kd, bc), _, _ = chk_fit
    vals = {
        "low": {"name": names[0], "kv_blocks_capacity": caps[0], "prefill_k": kp, "prefill_b": bp},
        "high": {"name": names[1], "kv_blocks_capacity": caps[1], "chunked_k_ctxp": kc, "chunked_k_ctxd": kd,
                 "chunked_b": bc},
    }
    out = []
    for line in base_cfg.splitlines():
        key = line.split("=")[0].strip()
        side, _, field = key.partition(".")
        if side in vals and field in vals[side]:
            v = vals[side][field]
            v = max(float(v), 0.0) if isinstance(v, float) else v
            line = f"{key} = {v!r}" if isinstance(v, float) else f"{key} = {v}"
        elif key in ("link.bandwidth", "link.latency"):
            line = f"{key} = {link[key]!r}"
        out.append(line)
    return "\n".join(out) + "\n"


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--ppi-sms", type=int, default=40)
    ap.add_argument("--base", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                   "tests", "golden", "configs", "a100_a10_llama8b.cfg"))
    ap.add_argument("--cpi-blocks", type=int, default=56000)
    ap.add_argument("--ppi-blocks", type=int, default=8192)
    ap.add_argument("--out", default=None)
    ap.add_argument("--samples-out", default=None, help="write the raw samples (reference calibrate format) here")
    a = ap.parse_args(argv)
    from .serving import GpuEngine
    base = open(a.base).read()
    eng = GpuEngine(model=a.model, clock="wall", ppi_sms=a.ppi_sms)
    part = eng.describe()
    # size the pools for sampling under the base config's capacities
    pre, chk = samples(eng, base)
    pf = E.fit_prefill([p[0] for p in pre], [p[1] for p in pre])
    cf = E.fit_chunked([c[0] for c in chk], [c[1] for c in chk], [c[2] for c in chk])
    kv_tok = {"llama3-8b": 131072, "qwen2-7b": 57344}.get(a.model, 16384)
    # co-located handoff = D2D block copy (read + write) at HBM speed; measured peak copy
    # bandwidth 6545 GB/s (MEASURED_PEAKS.json) -> tokens per ms
    link = {"link.bandwidth": 6545e9 / (2 * kv_tok) / 1000.0, "link.latency": 0.01}
    names = (f"B200-PPI{part['ppi_sms']}", f"B200-CPI{part['cpi_sms']}")
    cfg = build_config(base, pf, cf, names, (a.ppi_blocks, a.cpi_blocks), link)
    header = (f"# B200 co-located operating point, calibrated on the GPU by paper_2509_17357_b200.calibrate\n"
              f"# model {a.model}; SM partition {json.dumps(part)}\n"
              f"# prefill fit r2={pf[1]:.4f} mape={pf[2]:.4f}; chunked fit r2={cf[1]:.4f} mape={cf[2]:.4f}\n")
    cfg = header + cfg
    E.config_roundtrip(cfg)  # validates with the drop-in parser
    if a.out:
        with open(a.out, "w") as f:
            f.write(cfg)
    if a.samples_out:
        with open(a.samples_out, "w") as f:
            json.dump({"prefill": pre, "chunked": chk, "fit_prefill": [list(pf[0]), pf[1], pf[2]],
                       "fit_chunked": [list(cf[0]), cf[1], cf[2]], "partition": part}, f, indent=1)
    print(cfg)
    for p in pre:
        print(f"prefill L={p[0]:5d} {p[1]:8.3f} ms  ({2 * 6.98e9 * p[0] / p[1] / 1e9:7.1f} TFLOP/s linear)")
    for c in chk:
        print(f"iter pctx={c[0]:5d} ctxd={c[1]:7d} n_dec={c[3]:3d} chunk={c[4]:3d}: {c[2]:8.3f} ms")
    eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
