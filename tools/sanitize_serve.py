"""Dev: a tiny Cronus serve (PPI partial prefill -> handoff -> CPI chunks + decode) as a
compute-sanitizer target (tools/scripts/r2_sanitize.sh). Exits non-zero on a violation or
a schedule that differs from the host scheduler's."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_17357_b200 import engine as E  # noqa: E402
from paper_2509_17357_b200.serving import GpuEngine  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "tiny"
cfg = open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "configs", "a100_a10_llama8b.cfg")).read()
t = E.synth_trace(12, 300, 12, E.FIXED_INTERVAL, 20.0, 1)
eng = GpuEngine(model=model, clock="virtual")
res = eng.serve(cfg, t, want_tokens=True)
eng.close()
rep = json.loads(res.json)
ok = rep["violations"] == [] and rep["completed"] == len(t) and res.json == E.run(cfg, t).json
print(f"sanitize_serve {model}: completed {rep['completed']}/{len(t)}, schedule parity {ok}")
sys.exit(0 if ok else 1)
