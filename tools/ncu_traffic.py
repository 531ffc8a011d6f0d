"""Summarise `ncu --set full` captures (tools/scripts/ncu_full.sh) into profiles/.

    python tools/ncu_traffic.py gpurun_out/ncu_*.ncu-rep > profiles/rNN_ncu_traffic.json

Per captured launch: duration, DRAM read+write bytes, the kernel's ALGORITHMIC bytes for
the captured shape (passed in the capture's name, see SHAPES) and their ratio (traffic
well above 1 = wasted re-reads), tensor-pipe and DRAM utilisation. bench.py scales the
per-class ratio by its live algorithmic bytes per launch to report `traffic`.
"""
import csv
import io
import json
import os
import subprocess
import sys

MB = 1e6
L = dict(H=4096, Q=6144, NQ=4096, F=14336, KVTOK=8 * 2 * 128 * 2)  # LLaMA3-8B; KV bytes per token per layer
# capture name -> (class, [algorithmic bytes or flops per captured launch, in launch order], unit)
SHAPES = {
    "ncu_gemm_stream_dec8": ("cpi.gemm_stream", [2 * (L["Q"] * L["H"] + 8 * L["H"]) + 4 * 8 * L["Q"],
                                                 2 * (L["H"] * L["NQ"] + 8 * L["NQ"]) + 4 * 8 * L["H"],
                                                 2 * (2 * L["F"] * L["H"] + 8 * L["H"]) + 4 * 8 * 2 * L["F"],
                                                 2 * (L["H"] * L["F"] + 8 * L["F"]) + 4 * 8 * L["H"]], "bytes"),
    "ncu_decode_attn_dec8": ("cpi.decode_attn", [8 * 2048 * L["KVTOK"]], "bytes"),
    "ncu_decode_attn_dec64": ("cpi.decode_attn", [64 * 1024 * L["KVTOK"]], "bytes"),
    "ncu_gemm_tc_ppi1024": ("ppi.gemm_tc", [2 * 1024 * L["Q"] * L["H"], 2 * 1024 * L["H"] * L["NQ"],
                                            2 * 1024 * 2 * L["F"] * L["H"], 2 * 1024 * L["H"] * L["F"]], "flops"),
    "ncu_prefill_attn_chunk": ("cpi.prefill_attn", [4 * 32 * 128 * sum(2048 + i + 1 for i in range(480))], "flops"),
    "ncu_prefill_attn_v2": ("cpi.prefill_attn", [4 * 32 * 128 * sum(2048 + i + 1 for i in range(480))], "flops"),
    # round 2: the C2 serve's mixed pass (97 decoders x 1395 keys + a 415-token chunk at 1024) and a PPI prefill
    "ncu_prefill_pp_mixed": ("cpi.prefill_attn", [4 * 32 * 128 * sum(1024 + i + 1 for i in range(415))], "flops"),
    "ncu_decode_mixed": ("cpi.decode_attn", [97 * 1395 * L["KVTOK"]], "bytes"),
    "ncu_gemm_tc_mixed": ("cpi.gemm_tc", [2 * 512 * L["Q"] * L["H"], 2 * 512 * L["H"] * L["NQ"],
                                          2 * 512 * 2 * L["F"] * L["H"], 2 * 512 * L["H"] * L["F"]], "flops"),
    "ncu_prefill_pp_ppi": ("ppi.prefill_attn", [4 * 32 * 128 * sum(i + 1 for i in range(512))], "flops"),
    # round 2, final kernels: mixed pass of 80 decoders x 1440 keys + a 415-token chunk at 1024
    "ncu2_prefill_pp_mixed": ("cpi.prefill_attn", [4 * 32 * 128 * sum(1024 + i + 1 for i in range(415))], "flops"),
    "ncu2_decode_mixed": ("cpi.decode_attn", [80 * 1440 * L["KVTOK"]], "bytes"),
    "ncu2_gemm_tc_mixed": ("cpi.gemm_tc", [2 * 495 * L["Q"] * L["H"], 2 * 495 * L["H"] * L["NQ"],
                                           2 * 495 * 2 * L["F"] * L["H"], 2 * 495 * L["H"] * L["F"]], "flops"),
    "ncu2_gemm_stream_dec8": ("cpi.gemm_stream", [2 * (L["Q"] * L["H"] + 8 * L["H"]) + 4 * 8 * L["Q"],
                                                  2 * (L["H"] * L["NQ"] + 8 * L["NQ"]) + 4 * 8 * L["H"],
                                                  2 * (2 * L["F"] * L["H"] + 8 * L["H"]) + 4 * 8 * 2 * L["F"],
                                                  2 * (L["H"] * L["F"] + 8 * L["F"]) + 4 * 8 * L["H"]], "bytes"),
    "ncu2_prefill_pp_ppi": ("ppi.prefill_attn", [4 * 32 * 128 * sum(i + 1 for i in range(512))], "flops"),
}
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
           "launch__registers_per_thread"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = row[i].replace(",", "")
                try:
                    d[m] = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    d[m] = v
        d["kernel"] = row[hdr.index("Kernel Name")][:80]
        yield d


res = {"how": "ncu --set full --clock-control none, CRONUS_NO_PDL=1, tools/scripts/ncu_full.sh; bytes in B, time in us",
       "captures": {}}
for rep in sys.argv[1:]:
    name = os.path.basename(rep).replace(".ncu-rep", "")
    if name not in SHAPES:
        continue
    cls, alg, unit = SHAPES[name]
    launches = []
    for k, d in enumerate(rows(rep)):
        dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        a = alg[k] if k < len(alg) else None
        ent = {"kernel": d["kernel"], "us": round(d["gpu__time_duration.sum"], 2), "dram_bytes": int(dram),
               "grid": d.get("launch__grid_size"), "regs": d.get("launch__registers_per_thread"),
               "dram_pct": round(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"], 1),
               "tensor_pct": round(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"], 1)}
        if a is not None and unit == "bytes":
            ent.update(algorithmic_bytes=int(a), traffic_ratio=round(dram / a, 4),
                       achieved_gbs=round(a / d["gpu__time_duration.sum"] / 1e3, 1))
        elif a is not None:
            ent.update(algorithmic_flops=int(a), achieved_tflops=round(a / d["gpu__time_duration.sum"] / 1e6, 1),
                       dram_bytes_per_launch=int(dram))
        launches.append(ent)
    alg_b = sum(e.get("algorithmic_bytes", 0) for e in launches)
    dram_b = sum(e["dram_bytes"] for e in launches)
    res["captures"][name] = {"class": cls, "launches": launches,
                             "traffic_ratio": round(dram_b / alg_b, 4) if alg_b else None}
print(json.dumps(res, indent=1))
