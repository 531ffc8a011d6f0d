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


def _peaks():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
    except (OSError, ValueError):
        d = {}
    hbm = d.get("hbm_gbs") or 6545.0
    tf = d.get("bf16_tflops_sustained") or d.get("bf16_tflops") or 1390.0
    return {"hbm_GBps": float(hbm), "bf16_tflops": float(tf)}


def samples(eng, cfg_text, max_prefill=4096, budget_high=512, budget_low=256):
    """Samples in the regime each fitted model is evaluated in.

    prefill_time(low, L) is asked for PPI serial prefills of L tokens (engine.cpp:551);
    chunked_iter_time(high, pctx, ctxd) is asked by the balancer for iterations that carry a
    FULL chunk of n_p = max_batched_tokens - n_decode prompt tokens at growing prefill
    contexts (balancer.cpp:53-63) and by the engine for the same iterations (engine.cpp:473).
    Iterations of a fixed token budget are therefore sampled over prefill context (the chunk's
    start position) and decode context sum, with the chunk filling the rest of the budget."""
    pre = []
    for L in (16, 64, 128, 256, 384, 512, 768, 1024, 1536, 2048, 3072, 4096):
        if L > max_prefill:
            break
        pre.append((L, eng.time_pass(cfg_text, 0, chunk_len=L, reps=3)))
    chk = chunked_samples(eng, cfg_text, 1, budget_high)
    return pre, chk


def chunked_samples(eng, cfg_text, worker, budget, pos0s=(0, 1024, 2048, 3072), n_decs=(0, 8, 32, 64, 128),
                    ctxs=(512, 1536)):
    """(pctx, ctxd, ms, n_dec, chunk) of full-budget iterations on `worker` (0 PPI, 1 CPI)."""
    out = []
    for n_dec in n_decs:
        if n_dec >= budget:
            continue
        chunk = budget - n_dec
        for ctx in (ctxs if n_dec else ctxs[:1]):
            for pos0 in pos0s:
                ms = eng.time_pass(cfg_text, worker, n_dec=n_dec, dec_ctx=ctx if n_dec else 0, chunk_len=chunk,
                                   chunk_pos0=pos0, reps=3)
                out.append((pos0 + chunk, n_dec * ctx, ms, n_dec, chunk))
    return out


def prefill_samples(eng, cfg_text, worker, lengths=(64, 128, 256, 384, 512)):
    """Serial prefills on `worker` (the CPI's rows are sized for its token budget: <= 512)."""
    return [(L, eng.time_pass(cfg_text, worker, chunk_len=L, reps=3)) for L in lengths]


def build_config(base_cfg: str, fits, names, caps, link, tflops) -> str:
    """fits: {"low": {"prefill": fit, "chunked": fit}, "high": {...}} (coef, r2, mape)."""
    vals = {}
    for side in ("low", "high"):
        (kp, bp), _, _ = fits[side]["prefill"]
        (kc, kd, bc), _, _ = fits[side]["chunked"]
        vals[side] = {"name": names[side], "kv_blocks_capacity": caps[side], "prefill_k": kp, "prefill_b": bp,
                      "chunked_k_ctxp": kc, "chunked_k_ctxd": kd, "chunked_b": bc, "bf16_tflops": tflops[side]}
    out = []
    for line in base_cfg.splitlines():
        if line.startswith("#"):
            continue  # the base config's commentary describes other hardware
        key = line.split("=")[0].strip()
        side, _, field = key.partition(".")
        if side in vals and field in vals[side]:
            v = vals[side][field]
            v = max(float(v), 0.0) if isinstance(v, float) else v
            line = f"{key} = {v!r}" if isinstance(v, float) else f"{key} = {v}"
        elif key in ("link.bandwidth", "link.latency"):
            line = f"{key} = {link[key]!r}"
        out.append(line)
    while out and not out[0].strip():
        out.pop(0)
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
    budget_high = budget_low = None
    for line in base.splitlines():
        k, _, v = line.partition("=")
        if k.strip() == "max_batched_tokens_high":
            budget_high = int(v)
        elif k.strip() == "max_batched_tokens_low":
            budget_low = int(v)
    pre, chk = samples(eng, base, budget_high=budget_high)
    # the other two models of each profile (DP and disaggregated baselines run them)
    pre_hi = prefill_samples(eng, base, 1)
    # the PPI worker runs chunked iterations only under the DP policy: size it for that role
    base_dp = "\n".join("policy = dp" if ln.split("=")[0].strip() == "policy" else ln for ln in base.splitlines())
    chk_lo = chunked_samples(eng, base_dp, 0, budget_low, pos0s=(0, 1024, 2048), n_decs=(0, 8, 32, 64))
    fits = {"low": {"prefill": E.fit_prefill([p[0] for p in pre], [p[1] for p in pre]),
                    "chunked": E.fit_chunked([c[0] for c in chk_lo], [c[1] for c in chk_lo], [c[2] for c in chk_lo])},
            "high": {"prefill": E.fit_prefill([p[0] for p in pre_hi], [p[1] for p in pre_hi]),
                     "chunked": E.fit_chunked([c[0] for c in chk], [c[1] for c in chk], [c[2] for c in chk])}}
    kv_tok = {"llama3-8b": 131072, "qwen2-7b": 57344}.get(a.model, 16384)
    # co-located handoff = D2D block copy (read + write) at HBM speed; measured peak copy
    # bandwidth (MEASURED_PEAKS.json) -> tokens per ms
    peaks = _peaks()
    link = {"link.bandwidth": peaks["hbm_GBps"] * 1e9 / (2 * kv_tok) / 1000.0, "link.latency": 0.01}
    names = {"low": f"B200-PPI{part['ppi_sms']}", "high": f"B200-CPI{part['cpi_sms']}"}
    # dense bf16 peak of each partition (the measured device figure scaled by its SMs)
    tflops = {"low": round(peaks["bf16_tflops"] * part["ppi_sms"] / part["device_sms"], 1),
              "high": round(peaks["bf16_tflops"] * part["cpi_sms"] / part["device_sms"], 1)}
    cfg = build_config(base, fits, names, {"low": a.ppi_blocks, "high": a.cpi_blocks}, link, tflops)
    fl = " ".join(f"{side}.{m} r2={fits[side][m][1]:.4f} mape={fits[side][m][2]:.4f}"
                  for side in ("low", "high") for m in ("prefill", "chunked"))
    header = (f"# B200 co-located operating point, calibrated on the GPU by paper_2509_17357_b200.calibrate\n"
              f"# model {a.model}; SM partition {json.dumps(part)}\n"
              f"# fits (reference OLS, costmodel.cpp:94-113): {fl}\n"
              f"# chunked samples: full-budget iterations (chunk = max_batched_tokens - n_decode) over prefill\n"
              f"# context and decode context sum, the regime balancer.cpp:53-63 evaluates\n\n")
    cfg = header + cfg
    E.config_roundtrip(cfg)  # validates with the drop-in parser
    if a.out:
        with open(a.out, "w") as f:
            f.write(cfg)
    if a.samples_out:
        with open(a.samples_out, "w") as f:
            json.dump({"prefill_low": pre, "chunked_high": chk, "prefill_high": pre_hi, "chunked_low": chk_lo,
                       "fits": {s: {m: [list(v[0]), v[1], v[2]] for m, v in d.items()} for s, d in fits.items()},
                       "partition": part}, f, indent=1)
    print(cfg)
    for p in pre:
        print(f"PPI prefill L={p[0]:5d} {p[1]:8.3f} ms")
    for c in chk:
        print(f"CPI iter pctx={c[0]:5d} ctxd={c[1]:7d} n_dec={c[3]:3d} chunk={c[4]:3d}: {c[2]:8.3f} ms")
    eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
