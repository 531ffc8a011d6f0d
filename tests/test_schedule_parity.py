"""Schedule parity: the B200 engine's scheduler (virtual clock, no device work)
against the schedule oracle (the unmodified reference simulator, oracle/_ref) and
the committed goldens (tests/golden/schedule_goldens.json, whose first six digests
equal BASELINE.md section 2).

Mirrors the reference tests that pin the hot path:
test_balancer.cpp (brute force + guard), acceptance.cpp criteria 1/2/4/5/9,
test_engine.cpp:69/170/189/227, test_metrics.cpp:10/55, test_trace.cpp:25/49/112.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest

from conftest import ROOT, load_cfg
from paper_2509_17357_b200 import engine as E

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "schedule_goldens.json")))

try:
    from oracle import refsim
    HAVE_ORACLE = refsim.available()
except Exception:  # pragma: no cover
    HAVE_ORACLE = False
needs_oracle = pytest.mark.skipif(not HAVE_ORACLE, reason="oracle/_ref not built")

# Desk operating point of the reference unit tests (tests/helpers.hpp:11-40), as text.
DESK = """
policy = cronus
high.name = high
high.kv_blocks_capacity = 4096
high.kv_block_size = 16
high.prefill_k = 0.05
high.prefill_b = 5
high.chunked_k_ctxp = 0.002
high.chunked_k_ctxd = 0.00005
high.chunked_b = 25
high.total_layers = 32
high.bf16_tflops = 312
low.name = low
low.kv_blocks_capacity = 1024
low.kv_block_size = 16
low.prefill_k = 0.15
low.prefill_b = 10
low.chunked_k_ctxp = 0.006
low.chunked_k_ctxd = 0.00015
low.chunked_b = 40
low.total_layers = 32
low.bf16_tflops = 125
link.bandwidth = 100
link.latency = 1
link.kv_cost_per_token = 1
pp_layers_high = 23
pp_layers_low = 9
pp_comm_ms = 5
"""


def with_keys(text, **kv):
    lines = [l for l in text.strip().splitlines() if l.split("=")[0].strip() not in kv]
    lines += [f"{k.replace('__', '.')} = {v}" for k, v in kv.items()]
    return "\n".join(lines) + "\n"


def trace_of(rows, name="t"):
    rows = sorted(rows, key=lambda r: r[1])  # stable by arrival, like the reference
    a = np.array(rows, dtype=np.float64) if rows else np.zeros((0, 4))
    return E.Trace(a[:, 0].astype(np.int32), a[:, 1].copy(), a[:, 2].astype(np.int32), a[:, 3].astype(np.int32), name)


@pytest.mark.parametrize("key", sorted(GOLD))
def test_golden_digests(key):
    g = GOLD[key]
    cfg = load_cfg(key.split("/")[0])
    c = g["trace"]
    t = E.synth_trace(c["n"], c["mean_in"], c["mean_out"], E.FIXED_INTERVAL if c["fixed_interval"] else E.ALL_AT_ZERO,
                      c["interval_ms"], seed=1)
    assert f"{E.trace_hash(t):016x}" == g["trace_hash"]
    r = E.run(cfg, t)
    assert hashlib.sha256((r.json + "\n" + r.events).encode()).hexdigest() == g["digest"]
    assert r.csv == g["csv"]
    assert [x["partial_prefill_len"] for x in json.loads(r.json)["records"]] == g["partial_prefill_len"]


def test_survey_digests_pinned():
    # BASELINE.md section 2 digests (what the survey measured on the reference).
    want = {"a100_a10_llama8b/zero": "025d9156", "a100_a10_llama8b/fi150": "a7b15120",
            "a100_a10_llama8b/tiny": "0cd77a81", "a100_a30_qwen7b/zero": "8ad2e5e3",
            "a100_a30_qwen7b/fi150": "e22ebbdf", "a100_a30_qwen7b/tiny": "f14bd24d"}
    for k, v in want.items():
        assert GOLD[k]["digest"].startswith(v)


def random_trace(rng, n, max_in, max_out, bursty, max_arr=2000):
    rows = []
    for i in range(n):
        arr = 0.0 if bursty else float(rng.integers(0, max_arr))
        rows.append((i, arr, 1 + int(rng.integers(0, max_in)), 1 + int(rng.integers(0, max_out))))
    return trace_of(rows, "rand")


@needs_oracle
@pytest.mark.parametrize("policy", ["cronus", "dp", "disagg-hl", "disagg-lh"])
def test_random_traces_match_oracle(policy):
    """acceptance.cpp:189-229 sweep shape; here every output byte is compared."""
    rng = np.random.default_rng(1004)
    for trial in range(40):
        t = random_trace(rng, 2 + int(rng.integers(0, 20)), 3000, 60, trial % 2 == 0, 3000)
        kv = {"policy": policy}
        if trial % 4 == 0:
            kv["low__kv_blocks_capacity"] = 128
        if trial % 5 == 0:
            kv["high__kv_blocks_capacity"] = 512
        if trial % 7 == 0:
            kv["ppi_max_inflight"] = 1 + trial % 3
        cfg = with_keys(DESK, **kv)
        want = refsim.run(cfg, refsim.Trace(t.ids, t.arrival_ms, t.input_len, t.output_len, t.name),
                          utilization=trial % 3 == 0)
        got = E.run(cfg, t, utilization=trial % 3 == 0)
        assert got.json == want[0], (policy, trial)
        assert got.events == want[1], (policy, trial)
        assert got.csv == want[2]


@needs_oracle
def test_random_profiles_match_oracle():
    """Random GPU profiles (tests/helpers.hpp:43-54) and block sizes through the full run."""
    rng = np.random.default_rng(77)
    for trial in range(25):
        kv = {}
        for side in ("high", "low"):
            kv[f"{side}__kv_blocks_capacity"] = 64 + int(rng.uniform() * 8192)
            kv[f"{side}__kv_block_size"] = 8 << int(rng.integers(0, 3))
            kv[f"{side}__prefill_k"] = repr(0.01 + 0.3 * rng.uniform())
            kv[f"{side}__prefill_b"] = repr(20.0 * rng.uniform())
            kv[f"{side}__chunked_k_ctxp"] = repr(0.0005 + 0.01 * rng.uniform())
            kv[f"{side}__chunked_k_ctxd"] = repr(0.00001 + 0.0005 * rng.uniform())
            kv[f"{side}__chunked_b"] = repr(1.0 + 60.0 * rng.uniform())
        kv["max_batched_tokens_high"] = int(rng.choice([128, 256, 512]))
        cfg = with_keys(DESK, **kv)
        t = random_trace(rng, 3 + int(rng.integers(0, 40)), 4000, 80, trial % 2 == 0)
        want = refsim.run(cfg, refsim.Trace(t.ids, t.arrival_ms, t.input_len, t.output_len, t.name))
        got = E.run(cfg, t)
        assert (got.json, got.events, got.csv) == want, trial


def test_invariants_random_traces():
    """test_engine.cpp:189-225: no violations, every request accounted for."""
    rng = np.random.default_rng(77)
    for trial in range(20):
        n = 3 + int(rng.integers(0, 25))
        t = random_trace(rng, n, 2000, 50, trial % 2 == 0)
        for policy in ("cronus", "dp", "disagg-hl", "disagg-lh"):
            kv = {"policy": policy}
            if trial % 3 == 0:
                kv["low__kv_blocks_capacity"] = 96
            rep = json.loads(E.run(with_keys(DESK, **kv), t).json)
            assert rep["violations"] == []
            assert rep["completed"] + len(rep["failed_ids"]) == n
            for rec in rep["records"]:
                assert rec["ttft_ms"] > 0
                assert rec["completion_ms"] + 1e-9 >= rec["ttft_ms"]
                assert all(g > 0 for g in rec["tbt_samples_ms"])


def test_cronus_single_request_closed_form():
    """test_engine.cpp:69-107 / acceptance criterion 5."""
    L, out = 1000, 3
    lp, _, _, flags = E.choose_split(DESK, 0, 0, 4096, 512, L)
    assert flags == 0
    t = (0.15 * lp + 10.0) + (1.0 + 1.0 * lp / 100.0)
    done = lp
    if done == L:
        t += 0.002 * L + 25.0
    while done < L:
        done += min(512, L - done)
        t += 0.002 * done + 0.00005 * 0 + 25.0
    rep = json.loads(E.run(DESK, trace_of([(0, 0.0, L, out)])).json)
    rec = rep["records"][0]
    assert rep["violations"] == []
    assert rec["partial_prefill_len"] == lp
    assert math.isclose(rec["ttft_ms"], t, rel_tol=1e-12)
    for j, g in enumerate(rec["tbt_samples_ms"]):
        assert math.isclose(g, 0.002 * 0 + 0.00005 * (L + 1 + j) + 25.0, rel_tol=1e-12)


def test_determinism_and_event_log():
    """test_engine.cpp:170-187 (determinism) and :227-238 (event log)."""
    t = E.synth_trace(60, 400, 40, E.FIXED_INTERVAL, 20.0, 5)
    for policy in ("cronus", "dp", "disagg-hl", "disagg-lh"):
        cfg = with_keys(DESK, policy=policy)
        a, b = E.run(cfg, t), E.run(cfg, t)
        assert (a.json, a.events, a.csv) == (b.json, b.events, b.csv)
    log = E.run(DESK, trace_of([(0, 0.0, 300, 2)])).events
    assert "arrival" in log and "transfer-done" in log


def test_oversized_requests_fail_cleanly():
    """test_engine.cpp:156-168."""
    cfg = with_keys(DESK, policy="disagg-lh", low__kv_blocks_capacity=8)
    rep = json.loads(E.run(cfg, trace_of([(0, 0.0, 100, 2), (1, 0.0, 5000, 2), (2, 0.0, 50, 2)])).json)
    assert rep["violations"] == [] and rep["completed"] == 2 and rep["failed_ids"] == [1]


def test_invalid_inputs_rejected():
    with pytest.raises(ValueError):
        E.run(DESK, trace_of([]))
    with pytest.raises(ValueError):
        E.run(with_keys(DESK, link__bandwidth=0), trace_of([(0, 0.0, 10, 2)]))
    with pytest.raises(ValueError):  # pp baseline is out of scope for the B200 engine
        E.run(with_keys(DESK, policy="pp"), trace_of([(0, 0.0, 10, 2)]))
    with pytest.raises(RuntimeError):
        E.run(DESK + "bogus_key = 1\n", trace_of([(0, 0.0, 10, 2)]))


def brute_force_split(cfg_low, cfg_high, n_decode, ctx_sum, free_blocks, B, L):
    """test_balancer.cpp:16-52: every candidate straight from the formulas."""
    N = cfg_high["kv_block_size"]
    if free_blocks < (L + N - 1) // N:
        return L, 1
    n_p = B - n_decode
    if n_p <= 0:
        return L, 2
    best, best_gap = None, -1.0
    for i in range(1, 513):
        lp = (i * L + 511) // 512
        lc = L - lp
        tp = cfg_low["prefill_k"] * lp + cfg_low["prefill_b"]
        n_iter = 1 if lc == 0 else (lc + n_p - 1) // n_p
        l_last = lp + (lc // n_p) * n_p
        tc = n_iter * (cfg_high["chunked_k_ctxp"] * (L + l_last) / 2.0 + cfg_high["chunked_k_ctxd"] * float(ctx_sum)
                       + cfg_high["chunked_b"])
        gap = abs(tp - tc)
        if best_gap < 0 or gap < best_gap:
            best_gap, best = gap, lp
    return best, 0


def test_choose_split_brute_force_and_guard():
    """test_balancer.cpp:86-120, acceptance criteria 1-2 (1000 random instances)."""
    rng = np.random.default_rng(202)
    for trial in range(1000):
        prof = {}
        for side in ("high", "low"):
            prof[side] = dict(kv_blocks_capacity=64 + int(rng.uniform() * 8192), kv_block_size=8 << int(rng.integers(0, 3)),
                              prefill_k=0.01 + 0.3 * rng.uniform(), prefill_b=20.0 * rng.uniform(),
                              chunked_k_ctxp=0.0005 + 0.01 * rng.uniform(), chunked_k_ctxd=0.00001 + 0.0005 * rng.uniform(),
                              chunked_b=1.0 + 60.0 * rng.uniform())
        cfg = with_keys(DESK, **{f"{s}__{k}": repr(v) if isinstance(v, float) else v
                                 for s in prof for k, v in prof[s].items()})
        B = int(128 << int(rng.integers(0, 3)))
        n_dec = int(rng.integers(0, B + 64))
        ctx = n_dec * (100 + int(rng.integers(0, 2000)))
        L = 1 + int(rng.integers(0, 16384))
        if trial % 4 == 0:  # guard: strictly fewer free blocks than the prompt needs
            need = (L + prof["high"]["kv_block_size"] - 1) // prof["high"]["kv_block_size"]
            free = int(rng.integers(0, need))
        else:
            free = int(rng.integers(0, prof["high"]["kv_blocks_capacity"] + 1))
        lp, tp, tc, flags = E.choose_split(cfg, n_dec, ctx, free, B, L)
        want_lp, want_flags = brute_force_split(prof["low"], prof["high"], n_dec, ctx, free, B, L)
        assert (lp, flags) == (want_lp, want_flags), trial
        if HAVE_ORACLE and trial % 10 == 0:
            assert (lp, tp, tc, flags) == refsim.choose_split(cfg, n_dec, ctx, free, B, L)


def test_candidate_grid_edges():
    for L in (1, 512, 1000, 16384):
        lp, *_ = E.choose_split(DESK, 0, 0, 10**9, 512, L)
        assert 1 <= lp <= L
    with pytest.raises(ValueError):
        E.choose_split(DESK, 0, 0, 4096, 512, 0)


def test_fit_recovers_coefficients():
    """test_costmodel.cpp:48-132 / acceptance criterion 3."""
    rng = np.random.default_rng(3)
    lens = rng.uniform(1, 4000, 40)
    (k, b), r2, mape = E.fit_prefill(lens, 0.07 * lens + 3.0)
    assert abs(k - 0.07) < 1e-9 and abs(b - 3.0) < 1e-6 and r2 > 0.999999 and mape < 1e-9
    p, d = rng.uniform(0, 512, 50), rng.uniform(0, 1e5, 50)
    (kp, kd, bc), r2, _ = E.fit_chunked(p, d, 0.002 * p + 0.00005 * d + 13.0)
    assert abs(kp - 0.002) < 1e-9 and abs(kd - 0.00005) < 1e-11 and abs(bc - 13.0) < 1e-6
    with pytest.raises(RuntimeError):
        E.fit_prefill([5.0, 5.0, 5.0], [1.0, 2.0, 3.0])
    with pytest.raises(RuntimeError):
        E.fit_chunked([1.0, 2.0], [1.0, 2.0], [1.0, 2.0])
    if HAVE_ORACLE:
        y = 0.07 * lens + 3.0 + rng.normal(0, 0.5, 40)
        got = E.fit_prefill(lens, y)
        want = refsim.fit(0, lens, None, y)
        assert np.allclose(got[0], want[0], rtol=1e-12) and abs(got[1] - want[1]) < 1e-12


def test_percentile_nearest_rank():
    """test_metrics.cpp:10-45 / acceptance criterion 10."""
    assert E.percentile(list(range(1, 101)), 0.99) == 99.0
    assert E.percentile([7.5], 0.99) == 7.5
    assert E.percentile(list(range(1, 1001)), 0.99) == 990.0


@pytest.mark.parametrize("samples,p", [([], 0.99), ([1.0, 2.0], 99.0), ([1.0], 0.0), ([1.0], -0.5)])
def test_percentile_errors_cross_the_c_abi(samples, p):
    """metrics.cpp:13-15: empty sets and p outside (0, 1] throw std::invalid_argument; the
    C ABI turns it into ValueError instead of terminating the process."""
    with pytest.raises(ValueError):
        E.percentile(samples, p)


def test_config_roundtrip():
    """test_model.cpp:73-86: serialize -> parse is the identity."""
    for name in ("a100_a10_llama8b", "a100_a30_qwen7b"):
        text = load_cfg(name)
        once = E.config_roundtrip(text)
        assert E.config_roundtrip(once) == once
        if HAVE_ORACLE:
            assert refsim.run(once, refsim.synth_trace(20, 300, 20, True, 10.0, 1))[2] == \
                refsim.run(text, refsim.synth_trace(20, 300, 20, True, 10.0, 1))[2]


def test_synth_trace_properties():
    """test_trace.cpp:25-56."""
    a = E.synth_trace(200, 1014, 247, E.ALL_AT_ZERO, 0, 42)
    b = E.synth_trace(200, 1014, 247, E.ALL_AT_ZERO, 0, 42)
    c = E.synth_trace(200, 1014, 247, E.ALL_AT_ZERO, 0, 43)
    assert E.trace_hash(a) == E.trace_hash(b) != E.trace_hash(c)
    t = E.synth_trace(2000, 100, 30, E.ALL_AT_ZERO, 0, 7)
    assert t.input_len.min() >= 1 and t.input_len.max() <= 1600
    assert t.output_len.min() >= 1 and t.output_len.max() <= 480
    t = E.synth_trace(10, 50, 20, E.FIXED_INTERVAL, 25.0, 1)
    assert np.allclose(t.arrival_ms, 25.0 * np.arange(10))
