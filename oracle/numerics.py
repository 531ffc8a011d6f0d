"""TEST INFRASTRUCTURE ONLY — CPU fp32 restatement of the decoder the B200 engine runs.

The reference (/root/reference) has no model arithmetic at all (SURVEY.md section 8(c):
its GPU work is three linear cost formulas, proj/src/costmodel.cpp:9-15). Its paper ran
vLLM 0.6.1.post2, which is not vendored. This module restates the
published LLaMA-3 / Qwen2 decoder (RMSNorm, rotate-half RoPE, GQA causal attention,
SiLU-gated MLP, Qwen2 QKV bias, greedy argmax) in numpy fp32 over the exact bf16 weights
the engine initialises on device, and the exact prompt tokens it synthesises.

Pinned against a published implementation: tests/test_numerics_oracle.py loads the same
weights into Hugging Face LlamaForCausalLM / Qwen2ForCausalLM (tests/hf_ref.py) and
requires max |d logit| <= 1e-4 in fp32 on the tiny presets (measured ~1e-5), plus split
prefill == monolithic prefill and incremental decode == full-sequence forward.

Bit-exact restatements (checked by the GPU tests, tests/test_kernels_gpu.py):
  * splitmix64 weight init      csrc/kernels/elementwise.cu init_uniform_kernel
  * prompt-token hash           csrc/kernels/elementwise.cu prompt_tokens_kernel
  * RoPE tables (fp64 -> fp32)  csrc/kernels/elementwise.cu rope_table_kernel
Storage precision mirrors the engine (bf16 for normalised activations, q, k, v,
attention output and SiLU product; fp32 residual stream and accumulation), so the
remaining GPU/CPU difference is summation order only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
C_SEED = np.uint64(0x9E3779B97F4A7C15)
C_TID = np.uint64(0xD1B54A32D192ED03)


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def init_uniform(n: int, seed: int, tid: int, scale: float, offset: float, start: int = 0) -> np.ndarray:
    """Restates ck_init_uniform: bf16(offset + scale * (u24 - 2^23) / 2^23)."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * C_SEED + np.uint64(tid) * C_TID
        idx = np.arange(start, start + n, dtype=np.uint64)
        h = mix64(base + idx)
    u = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    step = np.float32(np.float32(scale) * np.float32(1.0 / 8388608.0))
    v = u.astype(np.float32) * step + np.float32(offset)
    return bf16_round(v.astype(np.float32))


def prompt_tokens(seed: int, req_id: int, n: int, vocab: int) -> np.ndarray:
    """Restates ck_prompt_tokens for positions 0..n-1 of request `req_id`."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * C_SEED + np.uint64(req_id & 0xFFFFFFFF) * C_TID
        h = mix64(base + np.arange(n, dtype=np.uint64))
    return (h % np.uint64(vocab)).astype(np.int64)


@dataclass
class Spec:
    """Mirror of csrc/gpu/model.cpp ModelSpec::preset."""
    name: str
    hidden: int
    layers: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float
    rms_eps: float
    qkv_bias: bool
    w_std: float = 0.02
    emb_std: float = 0.5
    lm_std: float = 0.05
    seed: int = 1234
    head_dim: int = 128

    @property
    def qkv_n(self):
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim


PRESETS = {
    "llama3-8b": Spec("llama3-8b", 4096, 32, 32, 8, 14336, 128256, 500000.0, 1e-5, False),
    "qwen2-7b": Spec("qwen2-7b", 3584, 28, 28, 4, 18944, 152064, 1000000.0, 1e-6, True),
    "tiny": Spec("tiny", 256, 2, 2, 1, 1024, 4096, 10000.0, 1e-5, False, lm_std=0.25),
    "tiny-qwen": Spec("tiny-qwen", 512, 2, 4, 2, 1024, 4096, 1000000.0, 1e-6, True, lm_std=0.25),
}

SQRT3 = np.float32(1.7320508075688772)
TID_EMBED, TID_LM, TID_FNORM = 1, 2, 3
W_QKV, W_O, W_GU, W_D, N_ATTN, N_FFN, B_QKV = range(7)


def layer_tid(l, which):
    return 16 + 16 * l + which


class Weights:
    """Lazily materialised bf16 weights (as fp32 arrays) of a preset."""

    def __init__(self, spec: Spec, seed: int | None = None):
        self.s = spec
        self.seed = spec.seed if seed is None else seed
        self._cache = {}

    def _mat(self, key, tid, rows, cols, std=None, scale=None, offset=0.0):
        if key not in self._cache:
            sc = float(np.float32(std) * SQRT3) if std is not None else scale
            self._cache[key] = init_uniform(rows * cols, self.seed, tid, sc, offset).reshape(rows, cols)
        return self._cache[key]

    def embed_rows(self, toks):
        s = self.s
        sc = float(np.float32(s.emb_std) * SQRT3)
        out = np.empty((len(toks), s.hidden), np.float32)
        for i, t in enumerate(toks):
            out[i] = init_uniform(s.hidden, self.seed, TID_EMBED, sc, 0.0, start=int(t) * s.hidden)
        return out

    def lm_head(self):
        s = self.s
        return self._mat("lm", TID_LM, s.vocab, s.hidden, std=s.lm_std)

    def final_norm(self):
        return self._mat("fn", TID_FNORM, 1, self.s.hidden, scale=0.1, offset=1.0)[0]

    def layer(self, l):
        s, H = self.s, self.s.hidden
        d = {
            "wqkv": self._mat(("qkv", l), layer_tid(l, W_QKV), s.qkv_n, H, std=s.w_std),
            "wo": self._mat(("o", l), layer_tid(l, W_O), H, s.n_heads * s.head_dim, std=s.w_std),
            "wgu": self._mat(("gu", l), layer_tid(l, W_GU), 2 * s.ffn, H, std=s.w_std),
            "wd": self._mat(("d", l), layer_tid(l, W_D), H, s.ffn, std=s.w_std),
            "an": self._mat(("an", l), layer_tid(l, N_ATTN), 1, H, scale=0.1, offset=1.0)[0],
            "fn": self._mat(("fn", l), layer_tid(l, N_FFN), 1, H, scale=0.1, offset=1.0)[0],
        }
        d["bqkv"] = (self._mat(("b", l), layer_tid(l, B_QKV), 1, s.qkv_n, scale=0.1)[0] if s.qkv_bias else None)
        return d


def rope_tables(max_pos: int, theta: float):
    f = np.arange(64, dtype=np.float64)
    inv = np.power(theta, -(2.0 * f) / 128.0)
    a = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(a).astype(np.float32), np.sin(a).astype(np.float32)


def rmsnorm(x, g, eps):
    ms = np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True, dtype=np.float32)
    return (x * (1.0 / np.sqrt(ms + np.float32(eps))).astype(np.float32)) * g


def rope(x, cos, sin):
    """x [..., 128] at positions with tables cos/sin [..., 64]; rotate-half pairs (i, i+64)."""
    a, b = x[..., :64], x[..., 64:]
    return np.concatenate([a * cos - b * sin, b * cos + a * sin], axis=-1)


class Decoder:
    """One request's forward over a growing KV cache (dense per request: paging is
    address arithmetic and does not change the math)."""

    def __init__(self, w: Weights, mirror_bf16: bool = True, max_pos: int = 16384):
        self.w = w
        self.s = w.s
        self.mirror = mirror_bf16
        self.cos, self.sin = rope_tables(max_pos, self.s.rope_theta)
        self.k = [np.zeros((0, self.s.n_kv_heads, 128), np.float32) for _ in range(self.s.layers)]
        self.v = [np.zeros((0, self.s.n_kv_heads, 128), np.float32) for _ in range(self.s.layers)]

    def _b(self, x):
        return bf16_round(x) if self.mirror else x.astype(np.float32)

    def forward(self, toks, pos0: int):
        """Rows toks[i] at positions pos0+i; appends their K/V; returns final hidden
        (normalised, pre-LM-head) of every row."""
        s = self.s
        n = len(toks)
        pos = np.arange(pos0, pos0 + n)
        x = self.w.embed_rows(toks)
        G = s.n_heads // s.n_kv_heads
        cs, sn = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        for l in range(s.layers):
            L = self.w.layer(l)
            h = self._b(rmsnorm(x, L["an"], s.rms_eps))
            qkv = h @ L["wqkv"].T
            if L["bqkv"] is not None:
                qkv = qkv + L["bqkv"]
            q = qkv[:, : s.n_heads * 128].reshape(n, s.n_heads, 128)
            k = qkv[:, s.n_heads * 128:(s.n_heads + s.n_kv_heads) * 128].reshape(n, s.n_kv_heads, 128)
            v = qkv[:, (s.n_heads + s.n_kv_heads) * 128:].reshape(n, s.n_kv_heads, 128)
            q = self._b(rope(q, cs, sn))
            k = self._b(rope(k, cs, sn))
            v = self._b(v)
            self.k[l] = np.concatenate([self.k[l], k], 0)
            self.v[l] = np.concatenate([self.v[l], v], 0)
            K, V = self.k[l], self.v[l]
            T = K.shape[0]
            out = np.empty((n, s.n_heads, 128), np.float32)
            scale = np.float32(1.0 / math.sqrt(128.0))
            mask = np.arange(T)[None, :] > pos[:, None]
            for hq in range(s.n_heads):
                kv = hq // G
                sc = (q[:, hq, :] @ K[:, kv, :].T) * scale
                sc = np.where(mask, -np.inf, sc)
                sc = sc - sc.max(axis=1, keepdims=True)
                p = np.exp(sc)
                p = p / p.sum(axis=1, keepdims=True)
                out[:, hq, :] = p @ V[:, kv, :]
            attn = self._b(out.reshape(n, -1))
            x = x + attn @ L["wo"].T
            h = self._b(rmsnorm(x, L["fn"], s.rms_eps))
            gu = h @ L["wgu"].T
            g, u = gu[:, 0::2], gu[:, 1::2]
            act = self._b(g / (1.0 + np.exp(-g)) * u)
            x = x + act @ L["wd"].T
        return self._b(rmsnorm(x, self.w.final_norm(), s.rms_eps))

    def logits(self, hidden):
        return hidden @ self.w.lm_head().T


def teacher_forced_logits(w: Weights, prompt: np.ndarray, tokens: np.ndarray, split: int | None = None,
                          mirror_bf16: bool = True) -> np.ndarray:
    """Logits [len(tokens), vocab] each generated token is sampled from: the prompt as a
    PPI prefix of `split` tokens plus the rest (the Cronus split), then the given tokens fed
    back one at a time (teacher forcing)."""
    dec = Decoder(w, mirror_bf16=mirror_bf16)
    if split and 0 < split < len(prompt):
        dec.forward(prompt[:split], 0)
        h = dec.forward(prompt[split:], split)[-1:]
    else:
        h = dec.forward(prompt, 0)[-1:]
    out = []
    for i, tok in enumerate(tokens):
        out.append(dec.logits(h)[0])
        if i + 1 < len(tokens):
            h = dec.forward(np.array([int(tok)]), len(prompt) + i)
    return np.stack(out)


def greedy_check(spec_name: str, prompt: np.ndarray, gpu_tokens: np.ndarray, tol: float, weights=None,
                 split: int | None = None):
    """Teacher-forced check of one request's generated tokens.

    Feeds the prompt (optionally as a partial prefill of `split` tokens plus the rest,
    the Cronus PPI/CPI split) and then the GPU's own tokens; at every step asserts
      * the GPU token's oracle logit is within `tol` of the oracle max, and
      * when the oracle's top-1/top-2 margin exceeds `tol`, the tokens are equal.
    Returns (n_steps, n_exact, min_margin).
    """
    w = weights or Weights(PRESETS[spec_name])
    dec = Decoder(w)
    if split and 0 < split < len(prompt):
        dec.forward(prompt[:split], 0)
        hid = dec.forward(prompt[split:], split)
    else:
        hid = dec.forward(prompt, 0)
    h = hid[-1:]
    exact = 0
    min_margin = np.inf
    for i, tok in enumerate(gpu_tokens):
        lg = dec.logits(h)[0]
        order = np.argsort(-lg, kind="stable")
        top, second = lg[order[0]], lg[order[1]]
        margin = float(top - second)
        min_margin = min(min_margin, margin)
        assert lg[tok] >= top - tol, f"step {i}: gpu token {tok} logit {lg[tok]:.4f} < max {top:.4f} - {tol}"
        if margin > tol:
            assert tok == order[0], f"step {i}: gpu {tok} != oracle {order[0]} (margin {margin:.4f})"
        exact += int(tok == order[0])
        if i + 1 < len(gpu_tokens):
            h = dec.forward(np.array([tok]), len(prompt) + i)
    return len(gpu_tokens), exact, min_margin
