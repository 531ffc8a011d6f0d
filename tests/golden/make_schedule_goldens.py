"""Regenerate tests/golden/schedule_goldens.json from the schedule oracle.

The oracle is the unmodified reference simulator (/root/reference/proj/src/*.cpp)
compiled by oracle/Makefile. Run in the build container (needs oracle/_ref):

    python tests/golden/make_schedule_goldens.py

Digest = sha256(report_to_json(rep, true) + "\\n" + event_log), the form used in
BASELINE.md section 2; the first six entries must equal the survey's digests.
"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import refsim  # noqa: E402

CASES = {
    "zero": dict(n=1000, mean_in=1014, mean_out=247, fixed_interval=False, interval_ms=0.0),
    "fi150": dict(n=1000, mean_in=1014, mean_out=247, fixed_interval=True, interval_ms=150.0),
    "tiny": dict(n=64, mean_in=256, mean_out=32, fixed_interval=True, interval_ms=20.0),
    "long": dict(n=1000, mean_in=4056, mean_out=988, fixed_interval=True, interval_ms=400.0),
}


def main():
    out = {}
    for cfg in ("a100_a10_llama8b", "a100_a30_qwen7b"):
        text = open(os.path.join(ROOT, "tests", "golden", "configs", cfg + ".cfg")).read()
        for tag, c in CASES.items():
            t = refsim.synth_trace(c["n"], c["mean_in"], c["mean_out"], c["fixed_interval"], c["interval_ms"], seed=1)
            j, e, row = refsim.run(text, t)
            rep = json.loads(j)
            out[f"{cfg}/{tag}"] = {
                "trace": c,
                "trace_hash": f"{refsim.trace_hash(t):016x}",
                "digest": hashlib.sha256((j + "\n" + e).encode()).hexdigest(),
                "csv": row,
                "partial_prefill_len": [r["partial_prefill_len"] for r in rep["records"]],
            }
    path = os.path.join(ROOT, "tests", "golden", "schedule_goldens.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
