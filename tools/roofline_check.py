"""Cross-check of bench.py's roofline against Nsight Compute (round 2).

    # 1) the serve under ncu (metrics-only launch list; PDL off: ncu replay cannot coexist with it;
    #    no green-context partition: ncu fails on green-context streams, so both runs use ppi_sms 0)
    CRONUS_NO_PDL=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/roof_launches.csv python tools/roofline_check.py serve --requests 24 \
        --stats gpurun_out/roof_stats_ncu.json
    # 2) the same serve without ncu (CUDA-event class timings, as bench.py measures them)
    python tools/roofline_check.py serve --requests 24 --stats gpurun_out/roof_stats_events.json
    # 3) compare
    python tools/roofline_check.py compare gpurun_out/roof_launches.csv gpurun_out/roof_stats_ncu.json \
        gpurun_out/roof_stats_events.json > profiles/r2_roofline_check.json

Per (worker, kernel class): algorithmic work of the serve (the engine's own tally, the same
numbers bench.py divides) over (a) the summed ncu kernel durations of that worker's streams
(kernels serialised and alone on the GPU) and (b) the CUDA-event class time of the same serve
(kernels concurrent with the other worker, as in bench.py's roofline), plus each class's share
of its worker's kernel time under both clocks.
"""
import argparse
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def serve(a):
    import numpy as np
    import bench
    from paper_2509_17357_b200 import engine as E
    from paper_2509_17357_b200.serving import GpuEngine
    _, cfg = bench.load_cfg(None, "cronus")  # bench.py's default cluster config and trace shape
    t = E.synth_trace(a.requests, 1014, 247, E.ALL_AT_ZERO, 0.0, 1)
    if a.max_out > 0:  # bounded decode tails (ncu times every launch: keep the launch count small)
        t = E.Trace(t.ids, t.arrival_ms, t.input_len, np.minimum(t.output_len, a.max_out).astype(np.int32), t.name)
    eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=a.ppi_sms)
    if not a.no_warm:
        eng.serve(cfg, t.subset(np.arange(4), name="warm"), events=False)  # lazy init
    res = eng.serve(cfg, t, events=False, profile=True)
    st = res.extra["stats"]
    json.dump({"stats": st, "describe": eng.describe()}, open(a.stats, "w"))
    eng.close()


def ncu_classes(csv_path, stream_ids):
    from bench import kernel_class
    text = open(csv_path).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    worker_of = {str(stream_ids.get("ppi")): "ppi", str(stream_ids.get("cpi")): "cpi",
                 str(stream_ids.get("cpi_full")): "cpi"}
    out = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        w = worker_of.get(r.get("Stream"))
        if w is None:
            continue
        us = float(r["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                                                          "msecond": 1e3, "ms": 1e3}.get(r.get("Metric Unit"), 1.0)
        c = kernel_class(r["Kernel Name"])
        d = out.setdefault(w, {}).setdefault(c, {"launches": 0, "us": 0.0})
        d["launches"] += 1
        d["us"] += us
    return out


def compare(a):
    from bench import peaks
    hbm, _, tf_sus, src = peaks()
    ncu_run = json.load(open(a.stats_ncu))
    ev_run = json.load(open(a.stats_events))
    sids = ncu_run["stats"]["partition"].get("stream_ids", {})
    nc = ncu_classes(a.launches, sids)
    res = {"how": __doc__.strip().splitlines()[0], "peaks": {"hbm_GBps": hbm, "bf16_tflops_sustained": tf_sus,
                                                              "source": src}, "classes": []}
    for w in ("cpi", "ppi"):
        tot_ncu = sum(v["us"] for v in nc.get(w, {}).values())
        tot_ev = sum(v["ms"] for k, v in ev_run["stats"][w].items() if k not in ("forward",) and v.get("launches"))
        for cls, tally in ev_run["stats"][w].items():
            if cls in ("forward", "other") or not tally.get("launches") or cls not in nc.get(w, {}):
                continue
            alg = ncu_run["stats"][w][cls]
            bound = "hbm" if cls in ("gemm_stream", "decode_attn") else "tensor"
            work = alg["bytes"] if bound == "hbm" else alg["flops"]
            peak = hbm if bound == "hbm" else tf_sus
            scale = 1e9 if bound == "hbm" else 1e12
            a_ncu = work / (nc[w][cls]["us"] * 1e-6) / scale
            work_ev = tally["bytes"] if bound == "hbm" else tally["flops"]
            a_ev = work_ev / (tally["ms"] * 1e-3) / scale
            res["classes"].append({
                "kernel": f"{w}.{cls}", "bound": bound, "unit": "GB/s" if bound == "hbm" else "TFLOP/s",
                "launches_ncu": nc[w][cls]["launches"], "launches_engine": alg["launches"],
                "achieved_ncu": round(a_ncu, 1), "frac_ncu": round(a_ncu / peak, 4),
                "achieved_events": round(a_ev, 1), "frac_events": round(a_ev / peak, 4),
                "share_ncu": round(nc[w][cls]["us"] / max(tot_ncu, 1e-9), 4),
                "share_events": round(tally["ms"] * 1e3 / max(tot_ev * 1e3, 1e-9), 4)})
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("serve")
    s.add_argument("--requests", type=int, default=24)
    s.add_argument("--stats", required=True)
    s.add_argument("--max-out", type=int, default=0, help="clip output lengths (0: the trace's own)")
    s.add_argument("--no-warm", action="store_true",
                   help="no warm-up serve (under ncu: the launch list then holds exactly the measured serve)")
    s.add_argument("--ppi-sms", type=int, default=0,
                   help="0 (default): no green-context partition (ncu cannot profile kernels on green-context streams)")
    c = sub.add_parser("compare")
    c.add_argument("launches")
    c.add_argument("stats_ncu")
    c.add_argument("stats_events")
    a = ap.parse_args()
    serve(a) if a.cmd == "serve" else compare(a)
