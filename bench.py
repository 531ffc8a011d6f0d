"""Benchmark: Cronus partial-prefill serving of LLaMA3-8B shapes on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1] at N=1): LLaMA3-8B shapes (bf16, random init),
one B200 with the partial-prefill worker (PPI, 40 SMs) and the chunked-prefill/decode
worker (CPI, 108 SMs) co-located via green-context SM partitioning; synthetic trace of
the paper's shape (synth_trace(1000, 1014, 247, seed 1), lognormal
lengths), all requests at t = 0 (the paper's max-throughput protocol);
scheduler on the wall clock with B200-calibrated cost profiles (tests/golden/configs/
b200_llama8b_coloc.cfg, produced by paper_2509_17357_b200.calibrate).

A step = serving the whole 1000-request trace to completion. `value` = requests
completed / step time with prompts already resident in HBM; `e2e` = the same through the
C-ABI with host buffers (prompt tokens H2D and generated tokens D2H inside the timed
region). `latency` = the same trace with fixed-interval arrivals offered at 0.7 x the
measured max req/s: TTFT / TBT P99 under load. N > 1 GPUs form N/2
worker pairs (PPI GPU 2p, CPI GPU 2p+1, NVLink handoff); pair p serves the requests with
id % pairs == p (static rule); weak scaling; P99s over the samples
pooled across pairs (metrics.cpp:35-57).

--impl reference: the CPU path on this host (oracle port of the decoder on all cores,
fitted with the reference's own fit_* and scheduled by the reference's own simulator,
oracle/_ref, on a trace synthesized by the reference's own synth_trace) for the same
metric; each step is one bounded CPU profile + fit + simulation.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG_DIR = os.path.join(ROOT, "tests", "golden", "configs")
DEFAULT_CFG = os.path.join(CFG_DIR, "b200_llama8b_coloc.cfg")
FALLBACK_CFG = os.path.join(CFG_DIR, "a100_a10_llama8b.cfg")
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--requests", type=int, default=1000, help="requests per worker pair per step (C2: 1000)")
    ap.add_argument("--warmup-requests", type=int, default=24)
    ap.add_argument("--model", default="llama3-8b")
    ap.add_argument("--config", default=None)
    ap.add_argument("--policy", default="cronus", choices=["cronus", "dp", "disagg-lh", "disagg-hl"],
                    help="serving policy on the pair (the paper's baselines besides cronus)")
    ap.add_argument("--ppi-sms", type=int, default=40)
    ap.add_argument("--arrival", default="all-at-zero", choices=["all-at-zero", "fixed-interval"])
    ap.add_argument("--interval-ms", type=float, default=0.0)
    ap.add_argument("--mean-in", type=float, default=1014, help="trace mean input tokens (paper: 1014; long: 4056)")
    ap.add_argument("--mean-out", type=float, default=247, help="trace mean output tokens (paper: 247; long: 988)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--profile-requests", type=int, default=8, help="trace prefix profiled with CUPTI")
    ap.add_argument("--cupti-timeout-s", type=float, default=120.0, help="deadlock guard of the CUPTI prefix")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget-s", type=float, default=20.0)
    ap.add_argument("--latency-load", type=float, default=0.7,
                    help="fixed-interval point at this fraction of the measured max req/s (0: off)")
    ap.add_argument("--time-budget-s", type=float, default=1500.0,
                    help="wall budget of the whole run: optional legs are skipped to stay inside it")
    ap.add_argument("--one-gpu-pairs", action="store_true",
                    help="test hook: every rank on GPU 0 (gloo), pairs as separate-device engines")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_cfg(path, policy="cronus"):
    """The cluster config text, with its `policy` line set to `policy` (the paper's
    baselines dp / disagg-lh / disagg-hl run on the same pair and profiles)."""
    path = path or (DEFAULT_CFG if os.path.exists(DEFAULT_CFG) else FALLBACK_CFG)
    lines = open(path).read().splitlines()
    lines = [f"policy = {policy}" if ln.split("=")[0].strip() == "policy" else ln for ln in lines]
    return path, "\n".join(lines) + "\n"


def make_trace(args, pairs):
    from paper_2509_17357_b200 import engine as E
    arrival = E.FIXED_INTERVAL if args.arrival == "fixed-interval" else E.ALL_AT_ZERO
    return E.synth_trace(args.requests * pairs, args.mean_in, args.mean_out, arrival, args.interval_ms, 1)


def pair_trace(trace, pair, pairs):
    return trace.subset(np.nonzero(trace.ids % pairs == pair)[0], name=f"{trace.name}[pair {pair}/{pairs}]")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [l.strip().split(", ") for l in self.f.read().splitlines() if l.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        for r in rows:
            if len(r) > 8:
                for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                                   r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(name)
        mx = float(rows[0][2]) if rows and len(rows[0]) > 2 and rows[0][2].replace(".", "").isdigit() else None
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    try:
        p = json.load(open(PEAKS))
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


TRAFFIC = os.path.join(ROOT, "profiles", "r2_ncu_after.json")
if not os.path.exists(TRAFFIC):
    TRAFFIC = os.path.join(ROOT, "profiles", "r1_ncu_traffic.json")


def traffic_ratios():
    """DRAM bytes / algorithmic bytes per kernel class from the committed ncu --set full
    captures (tools/scripts/ncu_full.sh -> tools/ncu_traffic.py); latest capture wins."""
    try:
        caps = json.load(open(TRAFFIC))["captures"]
    except Exception:
        return {}
    out = {}
    for name, c in caps.items():
        if c.get("traffic_ratio"):
            out[c["class"]] = (c["traffic_ratio"], f"{os.path.relpath(TRAFFIC, ROOT)}:{name}")
    return out


def kernel_class(name):
    """Kernel name (CUPTI, demangled) -> the engine's kernel-time class."""
    if "gemm_tc_kernel" in name:
        return "gemm_tc" if "<256" in name else "gemm_stream"  # BN <= 128 <=> M <= 128 rows
    if "attn_decode" in name:
        return "decode_attn"
    if "attn_prefill" in name:
        return "prefill_attn"
    return "other"


def cupti_profile(eng, cfg, sample):
    """Critical-path time per kernel class from CUPTI kernel records (torch.profiler) over a
    bounded sample of the trace, with the PDL launch chains intact (no per-launch events).

    Per worker (its streams: stream ids from the engine), kernels are ordered by end time and
    each is charged end_i - max(end_{i-1}, start_i): the time it adds to the worker's chain,
    so a kernel resident early at griddepcontrol.wait is not charged for waiting. Returns
    the stats shape of GpuEngine (per worker/class: launches, ms, bytes, flops)."""
    import tempfile
    from collections import defaultdict

    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        res = eng.serve(cfg, sample, events=False)
        torch.cuda.synchronize()
    fd, path = tempfile.mkstemp(suffix=".json")
    os.close(fd)
    try:
        prof.export_chrome_trace(path)
        tr = json.load(open(path))
    finally:
        os.remove(path)
    st = res.extra["stats"]
    sids = st["partition"].get("stream_ids", {})
    worker_of = {sids.get("ppi"): "ppi", sids.get("cpi"): "cpi", sids.get("cpi_full"): "cpi"}
    per_worker = defaultdict(list)
    copy_us = 0.0
    for e in tr.get("traceEvents", []):
        if e.get("cat") == "kernel" and "args" in e:
            w = worker_of.get(e["args"].get("stream"))
            if w:
                per_worker[w].append((e["ts"] + e["dur"], e["ts"], kernel_class(e["name"])))
            elif "kv_copy" in e["name"]:
                copy_us += e["dur"]
    out = {"cpi": {}, "ppi": {}, "partition": st["partition"], "sample_requests": len(sample)}
    if copy_us > 0 and st.get("handoff_bytes"):
        # KV handoff (co-located: D2D block copies read + write; NVLink pull between GPUs)
        out["handoff"] = {"handoffs": st["handoffs"], "bytes": st["handoff_bytes"], "kernel_ms": copy_us / 1e3,
                          "GBps": round((1 if not st.get("colocated", True) else 2) * st["handoff_bytes"]
                                        / (copy_us * 1e3), 1),
                          "what": "read+write bytes / kv_copy kernel time" if st.get("colocated", True)
                          else "bytes pulled over NVLink / kv_copy kernel time"}
    for w, ks in per_worker.items():
        ks.sort()
        prev = -1e30
        ms = defaultdict(float)
        for end, start, cls in ks:
            ms[cls] += (end - max(prev, start)) / 1e3
            prev = end
        for cls, tally in st[w].items():
            if cls in ms and tally.get("launches"):
                out[w][cls] = dict(tally, ms=ms[cls])
    return out


def decode_attn_probe(seqs=64, ctx=1024, layers=4, reps=40):
    """The decode-attention kernel alone at a larger batch than the serve's tail (the
    north-star shape class: HBM-bound paged attention), timed with CUDA events over
    back-to-back launches on its stream: LLaMA3-8B heads (8 kv / 32 q), random block
    tables, the layer rotated per launch so consecutive launches never hit L2 (each
    layer's K/V = seqs x ctx x 4 KiB > L2). Same planner as the engine (1 wave, clusters)."""
    import ctypes
    import math

    import torch
    from paper_2509_17357_b200._lib import lib
    L = lib()
    nkv, nq, sms = 8, 32, torch.cuda.get_device_properties(0).multi_processor_count
    slots = 2 * sms
    nblk = ctx // 16
    pairs = seqs * nkv
    C = 1
    while C < 16 and pairs * C * 2 <= slots and seqs * nblk * nkv >= pairs * C * 2 * 4:
        C *= 2
    pool = torch.zeros(seqs * nblk + 1, layers, 2, nkv, 16, 128, dtype=torch.bfloat16, device="cuda")
    bt = torch.randperm(seqs * nblk, device="cuda").int()
    off = torch.arange(seqs, dtype=torch.int32, device="cuda") * nblk
    rows = torch.arange(seqs, dtype=torch.int32, device="cuda")
    lens = torch.full((seqs,), ctx, dtype=torch.int32, device="cuda")
    work = ((torch.arange(seqs, dtype=torch.int32, device="cuda") << 16) | (1 << 8)).contiguous()  # 1 part each
    item0 = torch.arange(seqs, dtype=torch.int32, device="cuda")
    q = torch.randn(seqs, nq * 128, device="cuda").bfloat16()
    out = torch.empty_like(q)
    ws = torch.empty(seqs * nq * 130, device="cuda")
    tickets = torch.zeros(seqs * nkv, dtype=torch.int32, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    st = torch.cuda.current_stream()
    sp = ctypes.c_void_p(st.cuda_stream)

    def launch(layer):
        rc = L.ck_attn_decode_tma(P(q), P(pool), pool.shape[0], P(bt), P(rows), P(lens), P(off), P(item0), P(work),
                                  seqs, seqs, C, P(ws), P(tickets), P(out), nq, nkv, layer, layers,
                                  1 / math.sqrt(128), None, sp)
        assert rc == 0, rc

    for i in range(8):
        launch(i % layers)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for i in range(reps):
        launch(i % layers)
    e1.record(st)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    alg = seqs * ctx * nkv * 2 * 128 * 2
    hbm = peaks()[0]
    del pool
    torch.cuda.empty_cache()
    return {"kernel": "attn_decode_tma (alone)", "shape": f"{seqs} seqs x {ctx} keys, 8 kv / 32 q heads, cluster {C}",
            "bound": "hbm", "achieved": round(alg / us / 1e3, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(alg / us / 1e3 / hbm, 4), "us_per_launch": round(us, 2), "algorithmic_per_launch": alg}


def roofline(stats, partition=None, critical=None):
    """Kernel classes of a profiled serve -> (dominant class's roofline object, all classes).

    Dominant = the largest time share on the `critical` worker (the one busy the whole
    step: the CPI), or overall when None. Tensor-bound classes also get `frac_partition`:
    the fraction of the peak scaled to the SMs the worker owns (PPI 40 / CPI 108 of 148
    in the co-located split; CPI iterations on lent SMs make the CPI figure conservative)."""
    hbm, tf_burst, tf_sus, src = peaks()
    ratios = traffic_ratios()
    sms = {"ppi": (partition or {}).get("ppi_sms"), "cpi": (partition or {}).get("cpi_sms")}
    dev_sms = (partition or {}).get("device_sms") or 148
    classes = []
    for worker in ("cpi", "ppi"):
        for name, k in stats[worker].items():
            if name in ("forward", "other") or not k["launches"] or k["ms"] <= 0:
                continue
            bound = "hbm" if name in ("gemm_stream", "decode_attn") else "tensor"
            ms_avg = k["ms"] / k["launches"]
            if bound == "hbm":
                ach = k["bytes"] / k["launches"] / (ms_avg / 1e3) / 1e9
                peak, unit = hbm, "GB/s"
            else:
                ach = k["flops"] / k["launches"] / (ms_avg / 1e3) / 1e12
                peak, unit = tf_sus, "TFLOP/s"
            ent = {"kernel": f"{worker}.{name}", "bound": bound, "achieved": round(ach, 1), "peak": peak,
                   "unit": unit, "frac": round(ach / peak, 4), "launches": k["launches"],
                   "share_ms": round(k["ms"], 2), "avg_us": round(1e3 * ms_avg, 2),
                   "algorithmic_per_launch": (k["bytes"] if bound == "hbm" else k["flops"]) / k["launches"]}
            if bound == "tensor" and sms.get(worker):
                ent["frac_partition"] = round(ach / (peak * sms[worker] / dev_sms), 4)
            if f"{worker}.{name}" in ratios:
                r, src_t = ratios[f"{worker}.{name}"]
                ent["traffic"] = round(r * k["bytes"] / k["launches"])
                ent["traffic_ratio"] = r
                ent["traffic_source"] = src_t
            classes.append(ent)
    classes.sort(key=lambda c: -c["share_ms"])
    pool = [c for c in classes if critical is None or c["kernel"].startswith(critical + ".")]
    top = dict(pool[0]) if pool else {}
    if top:
        top.setdefault("traffic", None)
        top["peak_source"] = f"MEASURED_PEAKS.json ({src}; {'sustained' if top['bound'] == 'tensor' else 'copy'})"
        # committed ncu cross-check of the same class (tools/roofline_check.py: one serve, its
        # algorithmic work over ncu's kernel durations vs over CUDA-event class time)
        try:
            chk = json.load(open(os.path.join(ROOT, "profiles", "r2_roofline_check.json")))
            for c in chk["classes"]:
                if c["kernel"] == top["kernel"]:
                    top["ncu_crosscheck"] = {"frac_ncu": c["frac_ncu"], "frac_events_same_serve": c["frac_events"],
                                             "share_ncu": c["share_ncu"], "share_events": c["share_events"],
                                             "source": "profiles/r2_roofline_check.json"}
        except (OSError, ValueError, KeyError):
            pass
    return top, classes


def pass_rooflines(stats):
    """Pass-level HBM figures from the timed serve's own iteration records (wall-clock
    events per CPI iteration, PDL chains intact): decode-only passes stream every layer's
    weights + the LM head once plus each decoder's KV, so bytes / pass time is their
    achieved HBM rate (SURVEY.md 8(d) 'small-M GEMM: HBM', 'decode attention: HBM')."""
    hbm = peaks()[0]
    wb, kvb = stats.get("pass_weight_bytes"), stats.get("kv_bytes_per_token")
    out = {}
    for key, (n, ms, rows, ctx) in (stats.get("iteration_shapes") or {}).items():
        if not key.startswith("decode ") or not n or not wb:
            continue
        per = wb + rows * ctx * kvb
        us = 1e3 * ms / n
        out[key.split(" ", 1)[1] + " decoders"] = {
            "passes": n, "us_per_pass": round(us, 1), "mean_decoders": round(rows, 2), "mean_ctx": round(ctx, 1),
            "bytes_per_pass": per, "achieved_GBps": round(per / us / 1e3, 1), "frac": round(per / us / 1e3 / hbm, 4)}
    return out


class Comm:
    """The few collectives bench needs (NCCL on GPUs; gloo for the one-GPU test hook)."""

    def __init__(self, world, gloo):
        self.world, self.gloo = world, gloo
        if world > 1:
            import torch
            import torch.distributed as dist
            dist.init_process_group("gloo" if gloo or not torch.cuda.is_available() else "nccl")

    def _dev(self):
        import torch
        return "cpu" if self.gloo or not torch.cuda.is_available() else "cuda"

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def reduce(self, vals, op="max"):
        if self.world == 1:
            return list(vals)
        import torch
        import torch.distributed as dist
        t = torch.tensor(list(vals), dtype=torch.float64, device=self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return t.cpu().tolist()

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out


def nearest_rank(samples, p=0.99):
    """metrics.cpp:13-20 (nearest rank)."""
    v = np.sort(np.asarray(samples, np.float64))
    return float(v[max(1, int(np.ceil(p * len(v)))) - 1]) if len(v) else None


def pooled(reports):
    """TTFT / TBT P99 and means over the request records of every pair (metrics.cpp:35-57:
    TBT samples pooled across requests, here across pairs too)."""
    recs = [r for rep in reports for r in rep["records"] if r.get("ttft_ms", -1) >= 0]
    ttft = [r["ttft_ms"] for r in recs]
    tbt = [x for r in recs for x in r["tbt_samples_ms"]]
    return {"ttft_p99_ms": nearest_rank(ttft), "tbt_p99_ms": nearest_rank(tbt),
            "ttft_mean_ms": float(np.mean(ttft)) if ttft else None, "tbt_mean_ms": float(np.mean(tbt)) if tbt else None,
            "requests": len(recs), "tbt_samples": len(tbt)}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_ours(args, rank, world):
    import torch
    from paper_2509_17357_b200.serving import GpuEngine

    t_run0 = time.perf_counter()
    pairs = max(1, world // 2)
    colocated = world == 1
    cfg_path, cfg = load_cfg(args.config, args.policy)
    trace = make_trace(args, pairs)
    comm = Comm(world, args.one_gpu_pairs)
    driver = colocated or rank % 2 == 0  # even ranks drive a pair; odd ranks host its CPI GPU
    pair = rank // 2
    dev = 0 if colocated or args.one_gpu_pairs else rank
    torch.cuda.set_device(dev)
    eng = sub = None
    if driver:
        opts = dict(model=args.model, clock="wall")
        opts["ppi_sms"] = args.ppi_sms  # the low-end worker: an SM partition (its own GPU when N > 1)
        if args.one_gpu_pairs and not colocated:
            opts.update(ppi_device=0, cpi_device=0, separate=1)
        elif not colocated:
            opts.update(ppi_device=rank, cpi_device=rank + 1)
        eng = GpuEngine(**opts)
        sub = pair_trace(trace, pair, pairs)
        warm = sub.subset(np.arange(min(args.warmup_requests, len(sub))), name="warmup")

    def left():
        return args.time_budget_s - (time.perf_counter() - t_run0)

    def phase(name):  # progress on stderr (the JSON line is printed only at the end)
        if rank == 0:
            print(f"[bench] {time.perf_counter() - t_run0:7.1f} s  {name}", file=sys.stderr, flush=True)

    phase("engine ready")
    # ---- warm-up: W untimed serves (short trace: every kernel shape class, graphs of streams)
    for _ in range(args.warmup):
        if driver:
            eng.serve(cfg, warm, events=False)
    if driver:
        eng.stage(cfg, sub)  # prompts resident in HBM before the timed region
    # ---- timed: K serves of the full trace, device-timed, max over ranks
    times, reports = [], []
    clocks = None
    steps_run = 0
    for i in range(args.steps):
        comm.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(dev) as cs:
            s0.record()
            res = eng.serve(cfg, sub, events=False) if driver else None
            s1.record()
            torch.cuda.synchronize()
        clocks = cs.summary()
        ms = s0.elapsed_time(s1)
        if driver:
            ms = max(ms, res.extra["stats"]["gpu_ms"])  # engine streams' own event span
            reports.append(res)
        times.append(ms)
        steps_run += 1
        # guard: a step count that cannot finish inside the budget would lose the whole run
        # (after the next step there must still be room for the e2e and latency legs)
        proj = comm.reduce([(time.perf_counter() - t_run0) + np.mean(times) / 1e3 * (1.05 + 1.0 + 1.5)])[0]
        if i + 1 < args.steps and proj > args.time_budget_s:
            print(f"[bench] time budget: stopping after {steps_run} of {args.steps} steps", file=sys.stderr)
            break
    local = comm.reduce(times)
    step_ms = float(np.mean(local))
    n_done = json.loads(reports[-1].json)["completed"] if driver else 0
    n_done = int(comm.reduce([n_done], "sum")[0])
    value = n_done / (step_ms / 1e3)
    reps = comm.gather(json.loads(reports[-1].json) if driver else None)
    reps = [r for r in reps if r is not None]
    lat_max = pooled(reps)
    stats_all = comm.gather(reports[-1].extra["stats"] if driver else None)
    stats_all = [s for s in stats_all if s is not None]

    # ---- e2e: host prompt buffers in, generated tokens out, through the C-ABI
    e2e = None
    if not args.no_e2e:
        prompts = eng.prompts(cfg, sub) if driver else None  # host copy of the staged prompt tokens
        comm.barrier()
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        r = eng.serve(cfg, sub, host_prompt=prompts, want_tokens=True, events=False) if driver else None
        s1.record()
        torch.cuda.synchronize()
        ems = comm.reduce([s0.elapsed_time(s1)])[0]
        h2d, d2h = comm.reduce([r.extra["stats"]["h2d_bytes"] if driver else 0,
                                r.extra["stats"]["d2h_bytes"] if driver else 0], "sum")
        e2e = {"value": round(n_done / (ems / 1e3), 4), "unit": "req/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms": round(ems, 2)}

    phase("timed steps + e2e done")
    # ---- latency under load: fixed-interval arrivals at latency_load x the measured max req/s
    latency = None
    # every rank takes the same decision (a collective), so the legs below stay in step
    est = np.mean(times) / 1e3 / max(args.latency_load, 1e-9)
    short = comm.reduce([1.0 if left() < 1.2 * est + 1.3 * step_ms / 1e3 else 0.0])[0] > 0
    if args.latency_load > 0 and not short:
        iv = 1000.0 / (args.latency_load * value)  # ms between arrivals (all pairs' requests interleaved)
        from paper_2509_17357_b200 import engine as E
        fi = E.synth_trace(args.requests * pairs, args.mean_in, args.mean_out, E.FIXED_INTERVAL, iv, 1)
        fsub = pair_trace(fi, pair, pairs) if driver else None
        if driver:
            eng.stage(cfg, fsub)
        comm.barrier()
        torch.cuda.synchronize()
        r = eng.serve(cfg, fsub, events=False) if driver else None
        torch.cuda.synchronize()
        freps = [x for x in comm.gather(json.loads(r.json) if driver else None) if x is not None]
        span = max(x["t_end_ms"] for x in freps) - min(x["t_start_ms"] for x in freps)
        latency = dict(offered_load=args.latency_load, interval_ms=round(iv, 4), offered_rps=round(1000.0 / iv, 4),
                       value=round(sum(x["completed"] for x in freps) / (span / 1e3), 4), unit="req/s",
                       **{k: (round(v, 3) if isinstance(v, float) else v) for k, v in pooled(freps).items()},
                       trace=f"synth(n={args.requests * pairs}, mean_in={args.mean_in:g}, mean_out={args.mean_out:g}, "
                             f"seed=1, fixed-interval {iv:.4f} ms)")
    elif args.latency_load > 0:
        print("[bench] time budget: latency leg skipped", file=sys.stderr)

    phase("latency leg done")
    # ---- kernel rooflines: a profiled serve of the SAME trace (CUDA events around every
    # launch on its worker's stream; events between kernels serialise the PDL chain, so the
    # per-kernel figures are conservative), plus pass-level figures from the timed serve
    # and CUPTI critical-path times on a bounded prefix (chains intact) as a cross-check.
    roof, classes, crit, attn_probe, handoff, prof_stats = {}, [], [], None, None, None
    short = comm.reduce([1.0 if left() < 1.3 * step_ms / 1e3 + 60 else 0.0])[0] > 0
    if not args.no_profile and driver and not short:
        pr = eng.serve(cfg, sub, events=False, profile=True)
        prof_stats = pr.extra["stats"]
        roof, classes = roofline(prof_stats, prof_stats.get("partition"), critical="cpi")
        if roof:
            roof["timing"] = (f"CUDA events around each launch over the whole {len(sub)}-request trace "
                              "(average launch of the CPI worker's largest-share kernel class)")
        phase("profiled serve done")
        try:
            attn_probe = decode_attn_probe()
        except Exception as ex:
            print(f"[bench] decode attention probe failed ({ex})", file=sys.stderr)
        # CUPTI kernel records of a short prefix (PDL chains intact; handoff copy times): a
        # cross-check run last, in a thread with a deadlock guard — the CUPTI-traced serve has
        # been seen to stall on some boxes, and nothing after it may depend on it
        import threading
        box = {}

        def _cupti():
            try:
                sample = sub.subset(np.arange(min(args.profile_requests, len(sub))), name="profile-sample")
                box["cp"] = cupti_profile(eng, cfg, sample)
            except Exception as ex:  # noqa: BLE001
                box["err"] = str(ex)

        th = threading.Thread(target=_cupti, daemon=True)
        th.start()
        th.join(args.cupti_timeout_s)
        if "cp" in box:
            _, crit = roofline(box["cp"], box["cp"]["partition"])
            handoff = box["cp"].get("handoff")
        else:
            CUPTI_STUCK.append(th.is_alive())
            print(f"[bench] CUPTI prefix {'timed out' if th.is_alive() else 'failed: ' + box.get('err', '?')}",
                  file=sys.stderr)
        phase("CUPTI prefix done")
    elif not args.no_profile and driver:
        print("[bench] time budget: profiled serve skipped", file=sys.stderr)
    comm.barrier()

    if rank != 0:
        return None
    rep = json.loads(reports[-1].json)
    st = reports[-1].extra["stats"]
    line = {
        "metric": "req/s (Cronus partial-prefill serving, paper-shape trace; TTFT/TBT P99 alongside)",
        "value": round(value, 4), "unit": "req/s", "n_gpus": world, "steps": steps_run, "warmup": args.warmup,
        "ms_per_step": round(step_ms, 2), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (lognormal trace of the paper's shape; random-init weights)",
        "ttft_p99_ms": round(lat_max["ttft_p99_ms"], 3), "tbt_p99_ms": round(lat_max["tbt_p99_ms"], 3),
        "ttft_mean_ms": round(lat_max["ttft_mean_ms"], 3), "tbt_mean_ms": round(lat_max["tbt_mean_ms"], 3),
        "p99_pooled_requests": lat_max["requests"], "latency": latency,
        "config": {"workload": ("LLaMA3-8B shapes, 1 B200, PPI+CPI co-located (green-context SM split)"
                                if colocated else f"LLaMA3-8B shapes, {pairs} PPI/CPI pair(s) over NVLink"),
                   "model": args.model, "policy": args.policy, "requests_per_pair": len(sub), "pairs": pairs,
                   "trace": (f"synth(n={args.requests * pairs}, mean_in={args.mean_in:g}, mean_out={args.mean_out:g}, "
                             f"seed=1, {args.arrival}"
                             + (f" {args.interval_ms:g} ms)" if args.arrival == "fixed-interval" else ")")),
                   "cluster_config": os.path.relpath(cfg_path, ROOT), "clock": "wall (CUDA events)",
                   "partition": st.get("partition"), "l2": "inputs > L2 (15 GB of weights streamed per iteration)",
                   "parallelism": "replicas of worker pairs" if pairs > 1 else "co-located pair",
                   "p99": "nearest rank over samples pooled across pairs"},
        "gpu_launches": int(sum(s.get("gpu_launches", 0) for s in stats_all)),
        "cpi_iterations": st["cpi_iterations"], "violations": sum(len(r["violations"]) for r in reps),
        "cpi_busy_ms": round(st.get("cpi_busy_ms", 0.0), 2),
        "cpi_lent_iterations": st.get("cpi_lent_iterations"),
        "iteration_shapes_count_ms_rows_ctx": st.get("iteration_shapes"),
        "clocks": clocks, "e2e": e2e, "roofline": roof, "kernels": classes[:8],
        "decode_pass_hbm": pass_rooflines(st), "kernels_critical_path_prefix": crit[:8],
        "handoff": handoff, "decode_attn_kernel": attn_probe,
    }
    if CUPTI_STUCK:
        line["kernels_critical_path_prefix_note"] = "CUPTI-traced prefix did not finish within the guard; omitted"
    if steps_run < args.steps:
        line["steps_requested"] = args.steps
    if not args.no_cpu_baseline and world == 1:
        phase("CPU baseline")
        line["cpu_baseline"] = cpu_baseline(args, cfg, sub)
    phase("done")
    return line


def cpu_baseline(args, cfg, sub):
    from oracle import cpu_baseline as CB, refsim
    t = refsim.Trace(sub.ids, sub.arrival_ms, sub.input_len, sub.output_len, sub.name)
    r = CB.run(cfg, t, model=args.model, budget_s=args.cpu_budget_s)
    return {"value": round(r["rps"], 6), "unit": "req/s", "cores": r["samples"]["threads"], "kind": "port",
            "cpu": cpu_model(),
            "sample": ("1 of 32 decoder layers (numpy fp32, oracle restatement) timed on "
                       f"{len(r['samples']['prefill'])} prefill lengths + {len(r['samples']['chunked'])} mixed "
                       "batches, x32 + LM head; fitted with the reference's fit_prefill/fit_chunked and scheduled "
                       f"by the reference simulator (oracle/_ref) on the same {len(sub)}-request trace"),
            "ttft_p99_ms": round(r["ttft_p99_ms"], 1), "tbt_p99_ms": round(r["tbt_p99_ms"], 1),
            "seconds": round(r["cpu_seconds"] + r["des_seconds"], 2)}


def run_reference(args, rank, world):
    """The reference's own CPU path on this host: each step = a bounded CPU profile of the
    decoder (oracle port, all cores) -> the reference's fit_prefill / fit_chunked -> the
    reference's simulator on a trace from the reference's own synth_trace (oracle/_ref:
    nothing from this repo's package is loaded). Rank 0 only."""
    if rank != 0:
        return None
    from oracle import cpu_baseline as CB, refsim
    _, cfg = load_cfg(args.config, args.policy)
    pairs = max(1, world // 2)
    full = refsim.synth_trace(args.requests * pairs, args.mean_in, args.mean_out,
                              args.arrival == "fixed-interval", args.interval_ms, 1)
    keep = np.nonzero(full.ids % pairs == 0)[0]
    t = refsim.Trace(full.ids[keep], full.arrival_ms[keep], full.input_len[keep], full.output_len[keep], full.name)
    # per-step CPU budget: the whole --steps K --warmup W run stays within a few minutes
    budget = max(2.0, min(args.cpu_budget_s, 240.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        CB.run(cfg, t, model=args.model, budget_s=budget)
    vals, lat, last = [], [], None
    t0 = time.perf_counter()
    for _ in range(args.steps):
        last = CB.run(cfg, t, model=args.model, budget_s=budget)
        vals.append(last["rps"])
    wall = (time.perf_counter() - t0) / max(1, args.steps)
    v = float(np.mean(vals))
    threads = last["samples"]["threads"]
    return {"metric": "req/s (Cronus partial-prefill serving, paper-shape trace; TTFT/TBT P99 alongside)",
            "impl": "reference", "value": round(v, 6), "unit": "req/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall * 1e3, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "ttft_p99_ms": round(last["ttft_p99_ms"], 1), "tbt_p99_ms": round(last["tbt_p99_ms"], 1),
            "config": {"workload": "same trace and cluster config as the ours arm", "model": args.model,
                       "requests": len(t), "trace": t.name, "cluster_config": "same as ours (CPU-fitted profiles)"},
            "fit_chunked": last["fit_chunked"], "fit_prefill": last["fit_prefill"],
            "cpu_baseline": {"value": round(v, 6), "unit": "req/s", "cores": threads, "kind": "port",
                             "cpu": cpu_model(),
                             "sample": (f"per step: 1 of 32 decoder layers (numpy fp32 oracle port, {threads} threads) "
                                        f"timed on {len(last['samples']['prefill'])} prefill lengths + "
                                        f"{len(last['samples']['chunked'])} mixed batches within {budget:.1f} s, "
                                        "x32 + LM head -> reference fit_prefill/fit_chunked -> reference simulator "
                                        f"(oracle/_ref) on the {len(t)}-request trace")},
            "e2e": {"value": round(v, 6), "unit": "req/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


CUPTI_STUCK = []  # a CUPTI prefix thread that never returned (the process must not wait for it)


def main():
    args = parse()
    rank, world, _ = dist_env()
    if world != args.gpus and world == 1 and args.gpus > 1:
        print(json.dumps({"error": f"--gpus {args.gpus} must be launched with torchrun (one rank per GPU)"}))
        return 2
    if world > 1 and world % 2:
        print(json.dumps({"error": "N > 1 GPUs must be even (PPI/CPI pairs)"}))
        return 2
    line = run_reference(args, rank, world) if args.impl == "reference" else run_ours(args, rank, world)
    if line is not None:
        print(json.dumps(line), flush=True)
    if any(CUPTI_STUCK):
        sys.stderr.flush()
        os._exit(0)  # the stalled profiler thread holds the engine: exit without tearing it down
    return 0


if __name__ == "__main__":
    sys.exit(main())
