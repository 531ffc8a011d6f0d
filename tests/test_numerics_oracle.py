"""Numerics pin (CPU): the fp32 oracle restatement (oracle/numerics.py) against published
implementations — Hugging Face LlamaForCausalLM / Qwen2ForCausalLM loaded with the engine's
bit-identical weights (tests/hf_ref.py) — and the Cronus split (PPI partial prefill + CPI
chunks + one-token decode steps) against a monolithic prefill.

Stated tolerances (fp32 everywhere, summation order the only difference):
  * oracle vs HF logits:                 max |d logit| <= 1e-4 (logit std ~4 at tiny shapes)
  * split / incremental vs monolithic:   max |d logit| <= 1e-4
  * the bf16-mirrored oracle (the engine's storage precision) vs HF fp32: <= 0.1
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytest.importorskip("transformers")

from hf_ref import hf_logits, hf_model, numpy_tensors  # noqa: E402
from oracle import numerics as NUM  # noqa: E402

TOL_FP32 = 1e-4
TOL_BF16_MIRROR = 0.1


@pytest.fixture(scope="module", params=["tiny", "tiny-qwen"])
def setup(request):
    spec = NUM.PRESETS[request.param]
    w = NUM.Weights(spec)
    return spec, w, hf_model(spec, numpy_tensors(w))


def oracle_logits(w, tokens, cuts=(), mirror=False):
    """Logits of every position, the prompt fed in pieces [0, c1), [c1, c2), ..."""
    dec = NUM.Decoder(w, mirror_bf16=mirror)
    edges = [0, *cuts, len(tokens)]
    rows = [dec.forward(tokens[a:b], a) for a, b in zip(edges[:-1], edges[1:]) if b > a]
    return dec.logits(np.concatenate(rows))


def test_oracle_matches_hf(setup):
    spec, w, m = setup
    toks = NUM.prompt_tokens(99, 3, 200, spec.vocab)
    want = hf_logits(m, toks).numpy()
    got = oracle_logits(w, toks)
    err = float(np.abs(got - want).max())
    print(f"{spec.name}: oracle vs HF max |d logit| = {err:.2e} (logit std {want.std():.2f})")
    assert err <= TOL_FP32
    assert (got.argmax(-1) == want.argmax(-1)).mean() >= 0.99


def test_bf16_mirror_close_to_hf(setup):
    """The engine-precision oracle (bf16 storage of q/k/v, normed activations, attention
    output, SiLU product) stays within a stated bound of the fp32 published model."""
    spec, w, m = setup
    toks = NUM.prompt_tokens(99, 5, 128, spec.vocab)
    want = hf_logits(m, toks).numpy()
    err = float(np.abs(oracle_logits(w, toks, mirror=True) - want).max())
    print(f"{spec.name}: bf16-mirrored oracle vs HF fp32 max |d logit| = {err:.3f}")
    assert err <= TOL_BF16_MIRROR


@pytest.mark.parametrize("cuts", [(37,), (37, 101, 165), tuple(range(16, 200, 16)), (1,), (199,)])
def test_split_prefill_equals_monolithic(setup, cuts):
    """A PPI prefix of L_p tokens followed by CPI chunks (the
    partition the scheduler picks, engine.cpp:459-463) computes the monolithic logits."""
    spec, w, _ = setup
    toks = NUM.prompt_tokens(99, 11, 200, spec.vocab)
    mono = oracle_logits(w, toks)
    split = oracle_logits(w, toks, cuts)
    assert float(np.abs(split - mono).max()) <= TOL_FP32


def test_decode_steps_match_hf(setup):
    """Teacher-forced one-token decode steps after a split prefill (the CPI decode rows)
    equal HF's full-sequence forward at those positions."""
    spec, w, m = setup
    prompt = NUM.prompt_tokens(99, 21, 90, spec.vocab)
    dec = NUM.Decoder(w, mirror_bf16=False)
    dec.forward(prompt[:30], 0)
    h = dec.forward(prompt[30:], 30)[-1:]
    seq, got = list(prompt), []
    for i in range(12):
        lg = dec.logits(h)[0]
        got.append(lg)
        tok = int(np.argmax(lg))
        seq.append(tok)
        h = dec.forward(np.array([tok]), len(prompt) + i)
    want = hf_logits(m, np.array(seq[:-1])).numpy()[len(prompt) - 1:]
    assert float(np.abs(np.stack(got) - want).max()) <= TOL_FP32
