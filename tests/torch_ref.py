"""Plain PyTorch fp32 reference decoder on the GPU, for the LLaMA3-8B / Qwen2-7B shapes the
bench serves (test infrastructure; the numpy oracle oracle/numerics.py is the same math for the
tiny presets, where numpy is fast enough).

Weights are regenerated with the engine's own deterministic init kernel (ck_init_uniform,
bit-exact with oracle/numerics.init_uniform — tests/test_kernels_gpu.py) so they equal the
engine's bit for bit; the forward mirrors oracle/numerics.Decoder step by step (fp32 math,
bf16 rounding where the engine stores bf16: normed activations, q/k/v, attention output,
SiLU output, final hidden).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from oracle import numerics as NUM


class TorchWeights:
    def __init__(self, spec: NUM.Spec, L, device="cuda"):
        self.s, self.L, self.dev = spec, L, device
        self._cache = {}

    def _gen(self, n, tid, scale, offset=0.0):
        out = torch.empty(n, dtype=torch.bfloat16, device=self.dev)
        st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        rc = self.L.ck_init_uniform(ctypes.c_void_p(out.data_ptr()), n, self.s.seed, tid, scale, offset, st)
        assert rc == 0
        return out

    def _mat(self, key, tid, rows, cols, std=None, scale=None, offset=0.0):
        if key not in self._cache:
            sc = float(np.float32(std) * NUM.SQRT3) if std is not None else scale
            self._cache[key] = self._gen(rows * cols, tid, sc, offset).view(rows, cols)
        return self._cache[key]

    def embed(self):
        s = self.s
        return self._mat("emb", NUM.TID_EMBED, s.vocab, s.hidden, std=s.emb_std)

    def lm_head(self):
        s = self.s
        return self._mat("lm", NUM.TID_LM, s.vocab, s.hidden, std=s.lm_std)

    def final_norm(self):
        return self._mat("fn", NUM.TID_FNORM, 1, self.s.hidden, scale=0.1, offset=1.0)[0]

    def layer(self, l):
        s, H, lt = self.s, self.s.hidden, NUM.layer_tid
        d = {
            "wqkv": self._mat(("qkv", l), lt(l, NUM.W_QKV), s.qkv_n, H, std=s.w_std),
            "wo": self._mat(("o", l), lt(l, NUM.W_O), H, s.n_heads * 128, std=s.w_std),
            "wgu": self._mat(("gu", l), lt(l, NUM.W_GU), 2 * s.ffn, H, std=s.w_std),
            "wd": self._mat(("d", l), lt(l, NUM.W_D), H, s.ffn, std=s.w_std),
            "an": self._mat(("an", l), lt(l, NUM.N_ATTN), 1, H, scale=0.1, offset=1.0)[0],
            "fn": self._mat(("fn", l), lt(l, NUM.N_FFN), 1, H, scale=0.1, offset=1.0)[0],
        }
        d["bqkv"] = self._mat(("b", l), lt(l, NUM.B_QKV), 1, s.qkv_n, scale=0.1)[0] if s.qkv_bias else None
        return d


def _b(x):
    return x.to(torch.bfloat16).float()


def _rms(x, g, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps) * g.float()


def _rope(x, cs, sn):
    a, b = x[..., :64], x[..., 64:]
    return torch.cat([a * cs - b * sn, b * cs + a * sn], -1)


class TorchDecoder:
    """One request over a growing dense KV cache (oracle/numerics.Decoder on torch)."""

    def __init__(self, w: TorchWeights, max_pos: int = 16384, mirror_bf16: bool = True):
        self.w, self.s = w, w.s
        self._b = _b if mirror_bf16 else (lambda x: x)  # bf16 storage points of the engine, or fp32
        c, s = NUM.rope_tables(max_pos, self.s.rope_theta)
        self.cos, self.sin = torch.from_numpy(c).to(w.dev), torch.from_numpy(s).to(w.dev)
        self.k = [None] * self.s.layers
        self.v = [None] * self.s.layers

    @torch.no_grad()
    def forward(self, toks, pos0: int):
        s = self.s
        n = len(toks)
        pos = torch.arange(pos0, pos0 + n, device=self.w.dev)
        x = self.w.embed()[torch.as_tensor(np.asarray(toks), device=self.w.dev).long()].float()
        G = s.n_heads // s.n_kv_heads
        cs, sn = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        for l in range(s.layers):
            L = self.w.layer(l)
            h = self._b(_rms(x, L["an"], s.rms_eps))
            qkv = h @ L["wqkv"].float().t()
            if L["bqkv"] is not None:
                qkv = qkv + L["bqkv"].float()
            q = qkv[:, : s.n_heads * 128].view(n, s.n_heads, 128)
            k = qkv[:, s.n_heads * 128:(s.n_heads + s.n_kv_heads) * 128].view(n, s.n_kv_heads, 128)
            v = qkv[:, (s.n_heads + s.n_kv_heads) * 128:].view(n, s.n_kv_heads, 128)
            q, k, v = self._b(_rope(q, cs, sn)), self._b(_rope(k, cs, sn)), self._b(v)
            self.k[l] = k if self.k[l] is None else torch.cat([self.k[l], k])
            self.v[l] = v if self.v[l] is None else torch.cat([self.v[l], v])
            K = self.k[l].repeat_interleave(G, 1)  # [T, nq, 128]
            V = self.v[l].repeat_interleave(G, 1)
            T = K.shape[0]
            sc = torch.einsum("nhd,thd->hnt", q, K) / math.sqrt(128.0)
            mask = torch.arange(T, device=self.w.dev)[None, :] > pos[:, None]
            sc = sc.masked_fill(mask[None], float("-inf"))
            out = torch.einsum("hnt,thd->nhd", torch.softmax(sc, -1), V)
            x = x + self._b(out.reshape(n, -1)) @ L["wo"].float().t()
            h = self._b(_rms(x, L["fn"], s.rms_eps))
            gu = h @ L["wgu"].float().t()
            g, u = gu[:, 0::2], gu[:, 1::2]
            x = x + self._b(g * torch.sigmoid(g) * u) @ L["wd"].float().t()
        return self._b(_rms(x, self.w.final_norm(), s.rms_eps))

    @torch.no_grad()
    def logits(self, hidden):
        return hidden @ self.w.lm_head().float().t()


@torch.no_grad()
def teacher_forced_logits(w: TorchWeights, prompt, tokens, split=None, mirror_bf16=True):
    """[len(tokens), vocab] reference logits each generated token is sampled from (prompt as
    a PPI prefix of `split` tokens + the rest, then the tokens fed back one at a time)."""
    dec = TorchDecoder(w, max_pos=max(16384, len(prompt) + len(tokens) + 1), mirror_bf16=mirror_bf16)
    cuts = sorted({0, len(prompt), *(range(0, len(prompt), 2048)), *([split] if split and 0 < split < len(prompt) else [])})
    for a, b in zip(cuts[:-1], cuts[1:]):
        hid = dec.forward(prompt[a:b], a)
    h = hid[-1:]
    out = []
    for i, tok in enumerate(tokens):
        out.append(dec.logits(h)[0])
        if i + 1 < len(tokens):
            h = dec.forward(np.array([int(tok)]), len(prompt) + i)
    return torch.stack(out)


def greedy_check(w: TorchWeights, prompt, gpu_tokens, tol, split=None):
    """Teacher-forced check (oracle/numerics.greedy_check on torch): every GPU token's
    reference logit is within `tol` of the max, and equals the reference argmax whenever
    the top-1/top-2 margin exceeds `tol`. Returns (steps, exact, min_margin, max_deficit),
    deficit = reference max - reference logit of the GPU token."""
    dec = TorchDecoder(w, max_pos=max(16384, len(prompt) + len(gpu_tokens) + 1))
    # prefill in pieces (bounded score tensors for long prompts), breaking at the split too
    cuts = sorted({0, len(prompt), *(range(0, len(prompt), 2048)), *([split] if split and 0 < split < len(prompt) else [])})
    for a, b in zip(cuts[:-1], cuts[1:]):
        hid = dec.forward(prompt[a:b], a)
    h = hid[-1:]
    exact, min_margin, max_deficit = 0, float("inf"), 0.0
    for i, tok in enumerate(gpu_tokens):
        lg = dec.logits(h)[0]
        top2 = torch.topk(lg, 2)
        top, second, arg = float(top2.values[0]), float(top2.values[1]), int(top2.indices[0])
        margin = top - second
        min_margin = min(min_margin, margin)
        assert float(lg[int(tok)]) >= top - tol, f"step {i}: gpu token {tok} logit {float(lg[int(tok)]):.4f} < max {top:.4f} - {tol}"
        if margin > tol:
            assert int(tok) == arg, f"step {i}: gpu {tok} != reference {arg} (margin {margin:.4f})"
        exact += int(int(tok) == arg)
        max_deficit = max(max_deficit, top - float(lg[int(tok)]))
        if i + 1 < len(gpu_tokens):
            h = dec.forward(np.array([int(tok)]), len(prompt) + i)
    return len(gpu_tokens), exact, min_margin, max_deficit
