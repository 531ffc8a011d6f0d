"""bench.py end to end on the GPU: the N > 1 pair path (torchrun, max-over-ranks timing,
pooled P99s, the latency leg) on ONE GPU through the --one-gpu-pairs hook (every rank on
GPU 0, gloo collectives, each pair a separate-device engine), and the N = 1 line's keys.
Multi-GPU hardware numbers are not produced here."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

COMMON = ["--model", "tiny", "--steps", "1", "--warmup", "1", "--warmup-requests", "4", "--no-profile",
          "--no-cpu-baseline", "--config", os.path.join(ROOT, "tests", "golden", "configs", "a100_a10_llama8b.cfg")]


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def test_bench_world4_pairs_pool_p99():
    port = 29600 + os.getpid() % 300
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "4", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "4", "--one-gpu-pairs", "--requests", "12",
           *COMMON]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 4 and line["config"]["pairs"] == 2 and line["config"]["requests_per_pair"] == 12
    assert line["value"] > 0 and line["violations"] == 0 and line["gpu_launches"] > 0
    assert line["p99_pooled_requests"] == 24  # both pairs' records, not rank 0's alone
    lat = line["latency"]
    assert lat and lat["requests"] == 24 and lat["tbt_p99_ms"] > 0 and lat["offered_load"] == 0.7
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0


def test_bench_n1_line_keys():
    r = subprocess.run([sys.executable, "bench.py", "--requests", "16", *COMMON], cwd=ROOT, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    line = _last_json(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "clocks", "e2e", "gpu_launches", "latency", "ttft_p99_ms", "tbt_p99_ms"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["config"]["requests_per_pair"] == 16 and line["p99_pooled_requests"] == 16
    assert line["latency"]["value"] > 0
