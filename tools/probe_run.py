"""Dev probe: SM partition + a short LLaMA3-8B wall-clock serve with kernel stats."""
import json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200 import engine as E
from paper_2509_17357_b200.serving import GpuEngine

cfg = open("tests/golden/configs/a100_a10_llama8b.cfg").read()
eng = GpuEngine(model="tiny", clock="wall", ppi_sms=40)
print("partition", eng.describe(probe=True), flush=True)
eng.close()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for ppi_sms in (0, 40):
    t0 = time.time()
    eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=ppi_sms, profile=1)
    print("engine create s", round(time.time() - t0, 2), eng.describe(), flush=True)
    tr = E.synth_trace(n, 1014, 247, E.ALL_AT_ZERO, 0, 1)
    t0 = time.time()
    res = eng.serve(cfg, tr)
    dt = time.time() - t0
    rep = json.loads(res.json)
    st = res.extra["stats"]
    print(f"ppi_sms={ppi_sms} n={n} wall {dt:.2f}s rps {rep['throughput_rps']:.3f} ttft_p99 {rep['ttft_p99_ms']:.1f} "
          f"tbt_p99 {rep['tbt_p99_ms']:.2f} viol {len(rep['violations'])}", flush=True)
    cpi = st["cpi"]
    for k in ("decode_attn", "prefill_attn", "gemm", "other", "forward"):
        v = cpi[k]
        if v["launches"]:
            print(f"  cpi {k}: n={v['launches']} ms={v['ms']:.1f} avg_us={1000*v['ms']/v['launches']:.1f} "
                  f"GB/s={v['bytes']/max(v['ms'],1e-9)/1e6:.0f} TF/s={v['flops']/max(v['ms'],1e-9)/1e9:.1f}")
    for k in ("prefill_attn", "gemm", "other", "forward"):
        v = st["ppi"][k]
        if v["launches"]:
            print(f"  ppi {k}: n={v['launches']} ms={v['ms']:.1f} TF/s={v['flops']/max(v['ms'],1e-9)/1e9:.1f}")
    print("  iters", st["cpi_iterations"], "decode_rows", st["decode_rows"], "chunk_rows", st["chunk_rows"],
          "gpu_ms", round(st["gpu_ms"], 1), "instances", rep["instances"], flush=True)
    eng.close()
