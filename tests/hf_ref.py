"""Published implementations of the decoder the engine runs, as numerics pins (test
infrastructure only).

The reference has no model arithmetic and the paper's vLLM 0.6.1.post2
 is not vendored, so the oracle restatements (oracle/numerics.py on numpy,
tests/torch_ref.py on torch) are pinned against Hugging Face `transformers`
(LlamaForCausalLM / Qwen2ForCausalLM, the version installed in the image) loaded with the
engine's bit-identical weights: rotate-half RoPE with the default rope type (no LLaMA-3
frequency scaling), RMSNorm, GQA attention, SiLU-gated MLP, Qwen2 q/k/v bias.

Weight mapping (engine layout -> HF names):
  wqkv [(nq + 2 nkv) 128, H] rows = q | k | v  -> q_proj / k_proj / v_proj (+ bias)
  wgu  [2F, H], row 2i = gate_i, 2i+1 = up_i    -> gate_proj = wgu[0::2], up_proj = wgu[1::2]
  wo, wd, norms, embedding, lm_head             -> o_proj, down_proj, *_layernorm, embed_tokens, lm_head
"""
from __future__ import annotations

import torch

from oracle import numerics as NUM


def hf_config(spec: NUM.Spec, max_pos: int = 16384):
    common = dict(vocab_size=spec.vocab, hidden_size=spec.hidden, intermediate_size=spec.ffn,
                  num_hidden_layers=spec.layers, num_attention_heads=spec.n_heads,
                  num_key_value_heads=spec.n_kv_heads, head_dim=128, max_position_embeddings=max_pos,
                  rms_norm_eps=spec.rms_eps, rope_theta=spec.rope_theta, tie_word_embeddings=False,
                  hidden_act="silu", attn_implementation="eager")
    if spec.qkv_bias:
        from transformers import Qwen2Config
        return Qwen2Config(use_sliding_window=False, **common)
    from transformers import LlamaConfig
    return LlamaConfig(attention_bias=False, mlp_bias=False, **common)


@torch.no_grad()
def hf_model(spec: NUM.Spec, tensors, device="cpu"):
    """HF decoder in fp32 with the engine's weights. tensors(key) -> fp32 torch tensor for
    key in {"embed", "lm_head", "final_norm", (layer, "wqkv"|"bqkv"|"wo"|"wgu"|"wd"|"an"|"fn")}."""
    cfg = hf_config(spec)
    if spec.qkv_bias:
        from transformers import Qwen2ForCausalLM as Model
    else:
        from transformers import LlamaForCausalLM as Model
    with torch.device(device):
        m = Model(cfg).float().eval()
    nq, nkv = spec.n_heads * 128, spec.n_kv_heads * 128
    m.model.embed_tokens.weight.copy_(tensors("embed"))
    m.lm_head.weight.copy_(tensors("lm_head"))
    m.model.norm.weight.copy_(tensors("final_norm"))
    for l, layer in enumerate(m.model.layers):
        a, mlp = layer.self_attn, layer.mlp
        wqkv = tensors((l, "wqkv"))
        a.q_proj.weight.copy_(wqkv[:nq])
        a.k_proj.weight.copy_(wqkv[nq:nq + nkv])
        a.v_proj.weight.copy_(wqkv[nq + nkv:])
        if spec.qkv_bias:
            b = tensors((l, "bqkv"))
            a.q_proj.bias.copy_(b[:nq])
            a.k_proj.bias.copy_(b[nq:nq + nkv])
            a.v_proj.bias.copy_(b[nq + nkv:])
        a.o_proj.weight.copy_(tensors((l, "wo")))
        wgu = tensors((l, "wgu"))
        mlp.gate_proj.weight.copy_(wgu[0::2])
        mlp.up_proj.weight.copy_(wgu[1::2])
        mlp.down_proj.weight.copy_(tensors((l, "wd")))
        layer.input_layernorm.weight.copy_(tensors((l, "an")))
        layer.post_attention_layernorm.weight.copy_(tensors((l, "fn")))
        del wqkv, wgu
    return m


def numpy_tensors(w: NUM.Weights):
    """tensors() over the numpy oracle's lazily generated bf16 weights (tiny presets)."""
    s = w.s

    def get(key):
        if key == "embed":
            sc = float(NUM.np.float32(s.emb_std) * NUM.SQRT3)
            return torch.from_numpy(NUM.init_uniform(s.vocab * s.hidden, w.seed, NUM.TID_EMBED, sc, 0.0)
                                    .reshape(s.vocab, s.hidden))
        if key == "lm_head":
            return torch.from_numpy(w.lm_head())
        if key == "final_norm":
            return torch.from_numpy(w.final_norm())
        l, name = key
        return torch.from_numpy(NUM.np.ascontiguousarray(w.layer(l)[name]))
    return get


def torch_tensors(w):
    """tensors() over tests/torch_ref.TorchWeights (device-generated bf16, upcast)."""
    def get(key):
        if key == "embed":
            return w.embed().float()
        if key == "lm_head":
            return w.lm_head().float()
        if key == "final_norm":
            return w.final_norm().float()
        l, name = key
        return w.layer(l)[name].float()
    return get


@torch.no_grad()
def hf_logits(m, tokens, device="cpu"):
    """Logits of every position of one prompt, [T, vocab] fp32."""
    ids = torch.as_tensor(NUM.np.asarray(tokens), dtype=torch.long, device=device)[None]
    return m(input_ids=ids, use_cache=False).logits[0].float()
