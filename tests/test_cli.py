"""cronus_b200, the command-line driver: the reference cronus_sim's
subcommands and flags (proj/tools/cronus_sim.cpp:292-367). Its report JSON, CSV row, event log,
split decision and fits must equal the reference's own (oracle/_ref, built from the reference
sources) byte for byte; exit codes follow the reference (1 usage, 2 validation)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import CONFIG_DIR, ROOT

from oracle import refsim  # noqa: E402

CLI = os.path.join(ROOT, "paper_2509_17357_b200", "cronus_b200")
CFG = os.path.join(CONFIG_DIR, "a100_a10_llama8b.cfg")
try:
    HAVE_ORACLE = refsim.available()
except Exception:  # pragma: no cover
    HAVE_ORACLE = False
needs_oracle = pytest.mark.skipif(not HAVE_ORACLE, reason="oracle/_ref not built")
TRACE = ["--synth-n", "64", "--synth-mean-in", "256", "--synth-mean-out", "32", "--arrival", "fixed-interval",
         "--interval-ms", "20", "--synth-seed", "1"]


def cli(*args, check=True):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, timeout=120)
    if check:
        assert r.returncode == 0, r.stderr
    return r


def ref_trace():
    return refsim.synth_trace(64, 256, 32, True, 20.0, 1)


@needs_oracle
@pytest.mark.parametrize("policy", ["cronus", "dp", "disagg-hl", "disagg-lh"])
def test_run_outputs_equal_reference(tmp_path, policy):
    js, csv, ev = tmp_path / "r.json", tmp_path / "r.csv", tmp_path / "e.log"
    out = cli("run", "--config", CFG, "--policy", policy, *TRACE, "--json", str(js), "--csv", str(csv),
              "--emit-events", str(ev)).stdout
    cfg = open(CFG).read().replace("policy = cronus", f"policy = {policy}")
    want_json, want_ev, want_csv = refsim.run(cfg, ref_trace())
    assert js.read_text() == want_json + "\n"
    assert ev.read_text() == want_ev
    assert csv.read_text().splitlines()[1] == want_csv.strip()
    assert f"policy:        {policy}" in out


@needs_oracle
def test_compare_rows_equal_reference():
    pols = ["cronus", "dp", "disagg-hl", "disagg-lh"]
    rows = cli("compare", "--config", CFG, "--policies", ",".join(pols), *TRACE).stdout.splitlines()
    assert len(rows) == 1 + len(pols)
    for pol, row in zip(pols, rows[1:]):
        cfg = open(CFG).read().replace("policy = cronus", f"policy = {pol}")
        assert row == refsim.run(cfg, ref_trace(), events=False, utilization=True)[2].strip()


@needs_oracle
def test_split_equals_reference():
    for n_dec, ctxd, L in [(0, 0, 1014), (37, 41000, 2500), (500, 10**6, 300)]:
        out = cli("split", "--config", CFG, "--input-len", str(L), "--n-decode", str(n_dec), "--decode-ctx-sum",
                  str(ctxd)).stdout
        got = dict(line.split(" = ") for line in out.strip().splitlines())
        lp, tp, tc, _ = refsim.choose_split(open(CFG).read(), n_dec, ctxd, 20480, 512, L)
        assert int(got["partial_len"]) == lp
        assert abs(float(got["predicted_t_prefill_ms"]) - tp) <= 1e-9 * max(1.0, abs(tp))


@needs_oracle
def test_calibrate_equals_reference(tmp_path):
    rng = np.random.default_rng(3)
    x0 = rng.uniform(16, 4096, 20)
    x1 = rng.uniform(0, 2e5, 20)
    y = 0.003 * x0 + 2e-5 * x1 + 6 + rng.normal(0, 0.1, 20)
    f = tmp_path / "s.txt"
    f.write_text("# prefill_ctx decode_ctx_sum time_ms\n" + "".join(f"{float(a)!r},{float(b)!r},{float(c)!r}\n" for a, b, c in zip(x0, x1, y)))
    got = dict(line.split(" = ") for line in cli("calibrate", "--samples", str(f), "--kind", "chunked")
               .stdout.splitlines() if " = " in line)
    coef, _, _ = refsim.fit(1, x0, x1, y)
    assert np.allclose([float(got[k]) for k in ("chunked_k_ctxp", "chunked_k_ctxd", "chunked_b")], coef, rtol=1e-9)


def test_synth_roundtrip_and_exit_codes(tmp_path):
    out = tmp_path / "t.txt"
    msg = cli("synth", *TRACE, "--out", str(out)).stdout
    assert "e429169258cc169a" in msg  # the C1 trace hash (BASELINE.md goldens)
    assert "trace_hash:    e429169258cc169a" in cli("run", "--config", CFG, "--trace", str(out)).stdout
    assert cli("bogus", check=False).returncode == 1
    assert cli("run", "--synth-n", "4", check=False).returncode == 1  # --config missing
    assert cli("run", "--config", CFG, "--policy", "nope", "--synth-n", "4", check=False).returncode == 2
    assert cli("run", "--config", "/nonexistent.cfg", "--synth-n", "4", check=False).returncode == 2


@pytest.mark.gpu
def test_run_on_gpu_engine_matches_simulator(tmp_path):
    """--gpu serves the trace on the B200 engine; on the virtual clock its report and event
    log are the simulator's, byte for byte."""
    a, b = tmp_path / "gpu.json", tmp_path / "sim.json"
    ea, eb = tmp_path / "gpu.log", tmp_path / "sim.log"
    cli("run", "--config", CFG, *TRACE, "--gpu", "model = tiny, clock = virtual", "--json", str(a),
        "--emit-events", str(ea))
    cli("run", "--config", CFG, *TRACE, "--json", str(b), "--emit-events", str(eb))
    assert a.read_text() == b.read_text() and ea.read_text() == eb.read_text()
    r = cli("compare", "--config", CFG, "--policies", "cronus,dp", *TRACE, "--gpu", "model = tiny, clock = wall")
    assert len(r.stdout.splitlines()) == 3 and "FAILED" not in r.stdout
