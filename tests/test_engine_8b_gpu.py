"""Token parity at the benchmarked shapes (LLaMA3-8B, Qwen2-7B): the B200 engine serves a few
requests through the Cronus split (PPI partial prefill -> handoff -> CPI chunked prefill +
decode) and every generated token is checked, teacher-forced, against a plain PyTorch fp32
reference decoder on the GPU (tests/torch_ref.py) built from bit-identical weights.

Tolerance: 0.5 logits (logit std ~3 at these shapes; bf16 activations through 28-32 layers):
each GPU token's reference logit must be within 0.5 of the reference max, and equal to the
reference argmax whenever the reference's top-1/top-2 margin exceeds 0.5.
"""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import load_cfg  # noqa: E402
from oracle import numerics as NUM  # noqa: E402
from paper_2509_17357_b200 import engine as E  # noqa: E402

TOL = 0.5
# Stated bounds at the benchmarked shapes (logit std ~3):
#  * tests/torch_ref.py in fp32 vs Hugging Face Llama/Qwen2ForCausalLM fp32 (same weights):
#    max |d logit| <= TOL_HF (GPU fp32 GEMMs, TF32 off: summation order only)
#  * the engine's sampled-row logits through the Cronus split vs the bf16-mirrored reference,
#    teacher-forced on the engine's tokens: max |d logit| <= TOL_LOGIT, rms <= TOL_LOGIT_RMS,
#    and rms no larger than the bf16 storage effect itself (bf16-mirrored vs plain fp32 reference)
TOL_HF = 2e-3
TOL_LOGIT = 0.6  # max over ~2M logits (3 requests x 5 tokens x 128k vocab), logit std ~3; measured 0.42 / 0.34
TOL_LOGIT_RMS = 0.1  # measured 0.081 (LLaMA3-8B) / 0.062 (Qwen2-7B)


@pytest.mark.parametrize("model,cfg_name", [("llama3-8b", "a100_a10_llama8b"), ("qwen2-7b", "a100_a30_qwen7b")])
def test_real_shape_tokens(model, cfg_name):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_17357_b200._lib import lib
    from paper_2509_17357_b200.serving import GpuEngine
    from torch_ref import TorchWeights, greedy_check

    spec = NUM.PRESETS[model]
    cfg = load_cfg(cfg_name)
    ins = np.array([37, 300, 700, 129], np.int32)
    t = E.Trace(np.arange(len(ins), dtype=np.int32), np.zeros(len(ins)), ins, np.full(len(ins), 6, np.int32),
                "real-shape parity")
    eng = GpuEngine(model=model, clock="virtual", ppi_sms=40)
    res = eng.serve(cfg, t, want_tokens=True)
    eng.close()
    rep = json.loads(res.json)
    assert rep["violations"] == [] and rep["completed"] == len(t)
    assert res.json == E.run(cfg, t).json  # the schedule is the reference's
    torch.cuda.empty_cache()
    w = TorchWeights(spec, lib())
    total = exact = 0
    deficit = 0.0
    for i, r in enumerate(rep["records"]):
        prompt = NUM.prompt_tokens(99, int(t.ids[i]), int(ins[i]), spec.vocab)
        n, e, _, d = greedy_check(w, prompt, res.extra["tokens"][i], TOL, split=r["partial_prefill_len"] or None)
        total += n
        exact += e
        deficit = max(deficit, d)
    print(f"{model}: {exact}/{total} tokens equal to the reference argmax, max logit deficit {deficit:.3f}")
    # every token is within TOL of the reference max (asserted per step); most are the argmax
    # (random-init models at 128-152k vocab have frequent near-ties below TOL)
    assert exact >= 0.6 * total, f"{exact}/{total} tokens equal to the reference argmax"


@pytest.mark.parametrize("policy", ["cronus", "disagg-lh"])
def test_real_shape_edge_requests(policy):
    """LLaMA3-8B edge cases through the whole pair: a 1-token prompt, a 5000-token prompt
    (cronus: long chunked prefill on the CPI; disagg-lh: the whole prompt prefilled on the PPI
    in 4096-row slices, then a staged handoff), decode over ~5k keys with cluster-split
    attention, block-boundary prompts (16, 17) and a 1-token output."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_17357_b200._lib import lib
    from paper_2509_17357_b200.serving import GpuEngine
    from torch_ref import TorchWeights, greedy_check

    spec = NUM.PRESETS["llama3-8b"]
    cfg = load_cfg("a100_a10_llama8b").replace("policy = cronus", f"policy = {policy}")
    ins = np.array([1, 5000, 16, 17], np.int32)
    outs = np.array([3, 4, 1, 5], np.int32)
    t = E.Trace(np.arange(4, dtype=np.int32) + 10, np.zeros(4), ins, outs, "edge requests")
    eng = GpuEngine(model="llama3-8b", clock="virtual", ppi_sms=40)
    res = eng.serve(cfg, t, want_tokens=True)
    eng.close()
    rep = json.loads(res.json)
    assert rep["violations"] == [] and rep["completed"] == len(t)
    assert res.json == E.run(cfg, t).json
    assert [len(x) for x in res.extra["tokens"]] == list(outs)
    torch.cuda.empty_cache()
    w = TorchWeights(spec, lib())
    total = exact = 0
    for i, r in enumerate(rep["records"]):
        prompt = NUM.prompt_tokens(99, int(t.ids[i]), int(ins[i]), spec.vocab)
        n, e, _, _ = greedy_check(w, prompt, res.extra["tokens"][i], TOL, split=r["partial_prefill_len"] or None)
        total += n
        exact += e
    print(f"edge requests ({policy}): {exact}/{total} tokens equal to the reference argmax; splits "
          f"{[r['partial_prefill_len'] for r in rep['records']]}")
    assert exact >= 0.6 * total


def test_real_shape_wall_clock_tokens():
    """The bench's mode (wall clock, co-located green-context split, SM lending) at LLaMA3-8B
    shapes: all requests complete without ledger violations, iterations were lent, and every
    token passes the reference check under each request's actual split."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_17357_b200._lib import lib
    from paper_2509_17357_b200.serving import GpuEngine
    from torch_ref import TorchWeights, greedy_check

    spec = NUM.PRESETS["llama3-8b"]
    cfg = load_cfg("b200_llama8b_coloc")
    t = E.synth_trace(6, 600, 8, E.ALL_AT_ZERO, 0.0, 7)
    eng = GpuEngine(model="llama3-8b", clock="wall", ppi_sms=40)
    res = eng.serve(cfg, t, want_tokens=True)
    st = res.extra["stats"]
    eng.close()
    rep = json.loads(res.json)
    assert rep["violations"] == [] and rep["completed"] == len(t)
    assert st["cpi_lent_iterations"] > 0
    torch.cuda.empty_cache()
    w = TorchWeights(spec, lib())
    total = exact = 0
    for i, r in enumerate(rep["records"]):
        prompt = NUM.prompt_tokens(99, int(t.ids[i]), int(t.input_len[i]), spec.vocab)
        n, e, _, _ = greedy_check(w, prompt, res.extra["tokens"][i], TOL, split=r["partial_prefill_len"] or None)
        total += n
        exact += e
    assert exact >= 0.6 * total, f"{exact}/{total}"


def test_real_shape_long_prompt():
    """A 16k-token prompt at LLaMA3-8B shapes beside a short one: the balancer's split, a long
    PPI partial prefill, a multi-chunk CPI prefill over a >10k-key prefix (pp attention) and
    decode over ~16k keys (cluster-split attention); tokens checked against the reference."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_17357_b200._lib import lib
    from paper_2509_17357_b200.serving import GpuEngine
    from torch_ref import TorchWeights, greedy_check

    spec = NUM.PRESETS["llama3-8b"]
    cfg = load_cfg("a100_a10_llama8b")
    ins = np.array([16000, 200], np.int32)
    outs = np.array([4, 4], np.int32)
    t = E.Trace(np.arange(2, dtype=np.int32) + 40, np.zeros(2), ins, outs, "long prompt")
    eng = GpuEngine(model="llama3-8b", clock="virtual", ppi_sms=40)
    res = eng.serve(cfg, t, want_tokens=True)
    eng.close()
    rep = json.loads(res.json)
    assert rep["violations"] == [] and rep["completed"] == len(t)
    assert res.json == E.run(cfg, t).json
    torch.cuda.empty_cache()
    w = TorchWeights(spec, lib())
    total = exact = 0
    for i, r in enumerate(rep["records"]):
        prompt = NUM.prompt_tokens(99, int(t.ids[i]), int(ins[i]), spec.vocab)
        n, e, _, _ = greedy_check(w, prompt, res.extra["tokens"][i], TOL, split=r["partial_prefill_len"] or None)
        total += n
        exact += e
    print(f"long prompt: {exact}/{total} tokens equal to the reference argmax; splits "
          f"{[r['partial_prefill_len'] for r in rep['records']]}")
    assert exact >= 0.6 * total


@pytest.mark.parametrize("model", ["llama3-8b", "qwen2-7b"])
def test_torch_reference_matches_hf(model):
    """Pin the GPU reference decoder against the published implementation at full shapes."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from hf_ref import hf_logits, hf_model, torch_tensors
    from paper_2509_17357_b200._lib import lib
    from torch_ref import TorchDecoder, TorchWeights

    spec = NUM.PRESETS[model]
    torch.backends.cuda.matmul.allow_tf32 = False
    w = TorchWeights(spec, lib())
    prompt = NUM.prompt_tokens(99, 7, 96, spec.vocab)
    dec = TorchDecoder(w, mirror_bf16=False)
    dec.forward(prompt[:40], 0)  # split prefill, as the pair runs it
    got = dec.logits(torch.cat([dec.forward(prompt[40:], 40)]))
    del dec
    m = hf_model(spec, torch_tensors(w), device="cuda")
    want = hf_logits(m, prompt, device="cuda")[40:]
    del m
    torch.cuda.empty_cache()
    err = float((got - want).abs().max())
    print(f"{model}: torch reference (fp32) vs HF fp32 max |d logit| = {err:.2e}, logit std {float(want.std()):.2f}")
    assert err <= TOL_HF
    assert float((got.argmax(-1) == want.argmax(-1)).float().mean()) >= 0.95


@pytest.mark.parametrize("model,cfg_name", [("llama3-8b", "a100_a10_llama8b"), ("qwen2-7b", "a100_a30_qwen7b")])
def test_real_shape_logits(model, cfg_name):
    """Sampled-row logits through PPI partial prefill -> handoff -> CPI chunks + decode at
    the benchmarked shapes, within TOL_LOGIT of the bf16-mirrored reference."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_17357_b200._lib import lib
    from paper_2509_17357_b200.serving import GpuEngine
    from torch_ref import TorchWeights, teacher_forced_logits

    spec = NUM.PRESETS[model]
    cfg = load_cfg(cfg_name)
    ins = np.array([300, 700, 129], np.int32)
    t = E.Trace(np.arange(len(ins), dtype=np.int32) + 3, np.zeros(len(ins)), ins, np.full(len(ins), 5, np.int32),
                "real-shape logits")
    eng = GpuEngine(model=model, clock="virtual", ppi_sms=40)
    res = eng.serve_logits(cfg, t, spec.vocab)
    eng.close()
    rep = json.loads(res.json)
    assert rep["violations"] == [] and res.json == E.run(cfg, t).json
    torch.cuda.empty_cache()
    w = TorchWeights(spec, lib())
    worst = rms = eff_max = eff_rms = 0.0
    n = 0
    for i, r in enumerate(rep["records"]):
        toks, got = res.extra["tokens"][i], torch.from_numpy(res.extra["logits"][i]).cuda()
        assert torch.equal(got.argmax(-1).cpu().int(), torch.from_numpy(toks).int())
        prompt = NUM.prompt_tokens(99, int(t.ids[i]), int(ins[i]), spec.vocab)
        split = r["partial_prefill_len"] or None
        want = teacher_forced_logits(w, prompt, toks, split)
        # the size of the engine's own bf16 storage effect: the same reference in plain fp32
        want32 = teacher_forced_logits(w, prompt, toks, split, mirror_bf16=False)
        d, e = (got - want).float(), (want - want32).float()
        worst, eff_max = max(worst, float(d.abs().max())), max(eff_max, float(e.abs().max()))
        rms += float((d * d).sum())
        eff_rms += float((e * e).sum())
        n += d.numel()
    rms, eff_rms = (rms / n) ** 0.5, (eff_rms / n) ** 0.5
    print(f"{model}: engine vs bf16-mirrored reference max |d logit| = {worst:.4f} rms {rms:.4f} "
          f"(tolerance {TOL_LOGIT} / rms {TOL_LOGIT_RMS}); bf16 storage effect (mirrored vs fp32 reference) "
          f"max {eff_max:.4f} rms {eff_rms:.4f}; logit std {float(want.std()):.2f}; splits "
          f"{[r['partial_prefill_len'] for r in rep['records']]}")
    assert worst <= TOL_LOGIT and rms <= TOL_LOGIT_RMS
    # the engine sits about as far from the bf16-mirrored reference as bf16 storage itself moves
    # the fp32 reference (measured 0.081 vs 0.091 and 0.062 vs 0.063): the remaining differences
    # are rounding-order effects of the same size, not a systematic error
    assert rms <= 1.25 * eff_rms
