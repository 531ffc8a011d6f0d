import faulthandler, sys, os, time
sys.path.insert(0, '.')
faulthandler.dump_traceback_later(90, repeat=True, file=sys.stderr)
import numpy as np, bench
from paper_2509_17357_b200 import engine as E
from paper_2509_17357_b200.serving import GpuEngine
_, cfg = bench.load_cfg(None, "cronus")
t = E.synth_trace(48, 1014, 247, E.ALL_AT_ZERO, 0.0, 1)
eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=40)
t0 = time.time()
eng.serve(cfg, t.subset(np.arange(8), name="w"), events=False)
print("warm", time.time() - t0, file=sys.stderr, flush=True)
for n in (8, 48):
    t0 = time.time()
    cp = bench.cupti_profile(eng, cfg, t.subset(np.arange(n), name="p"))
    print("cupti", n, time.time() - t0, list(cp["cpi"].keys()), file=sys.stderr, flush=True)
