"""sm_100a kernels of the C-ABI layer (include/cronus_ck.h) against references.

* init / prompt hash / RoPE table: bit-exact (or 1-ulp) against oracle/numerics.py.
* RMSNorm, QKV+RoPE+KV-append, decode and prefill paged attention, SiLU-mul,
  argmax, KV handoff copy: against plain torch fp32 references of the same op.
Tolerances are stated per test (bf16 storage => ~2^-8 relative).
"""
import ctypes
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import numerics as NUM  # noqa: E402


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2509_17357_b200._lib import lib
    return lib()


def p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ok(rc):
    assert rc == 0, f"kernel rc={rc}"
    torch.cuda.synchronize()


def test_init_uniform_bit_exact(L):
    for tid, scale, off, n in [(1, 0.866, 0.0, 100003), (37, 0.1, 1.0, 4096), (2**40 + 5, 0.0346, 0.0, 77777)]:
        out = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        ok(L.ck_init_uniform(p(out), n, 1234, tid, scale, off, stream()))
        want = NUM.init_uniform(n, 1234, tid, scale, off)
        got = out.float().cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_prompt_tokens_bit_exact(L):
    for rid, n, vocab in [(0, 300, 4096), (12345, 1000, 128256), (7, 17, 152064)]:
        req = torch.full((n,), rid, dtype=torch.int32, device="cuda")
        pos = torch.arange(n, dtype=torch.int32, device="cuda")
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        ok(L.ck_prompt_tokens(p(out), p(req), p(pos), n, 99, vocab, stream()))
        assert np.array_equal(out.cpu().numpy(), NUM.prompt_tokens(99, rid, n, vocab))


def test_rope_table(L):
    P = 5000
    c = torch.empty(P * 64, device="cuda")
    s = torch.empty(P * 64, device="cuda")
    ok(L.ck_rope_table(p(c), p(s), P, 500000.0, stream()))
    wc, ws = NUM.rope_tables(P, 500000.0)
    assert np.abs(c.cpu().numpy().reshape(P, 64) - wc).max() <= 1e-7
    assert np.abs(s.cpu().numpy().reshape(P, 64) - ws).max() <= 1e-7


def test_rmsnorm(L):
    for H, R in [(256, 7), (4096, 33), (3584, 5)]:
        x = torch.randn(R + 3, H, device="cuda") * 3
        g = (1 + 0.1 * torch.randn(H, device="cuda")).bfloat16()
        rows = torch.tensor([2, 0] + list(range(3, R + 1)), dtype=torch.int32, device="cuda")
        out = torch.empty(R, H, dtype=torch.bfloat16, device="cuda")
        zero = torch.randn(R + 1, 512, device="cuda")
        ok(L.ck_rmsnorm(p(x), p(g), p(out), p(rows), R, H, 1e-5, p(zero), 512, stream()))
        xs = x[rows.long()]
        ref = xs * torch.rsqrt(xs.pow(2).mean(-1, keepdim=True) + 1e-5) * g.float()
        assert torch.allclose(out.float(), ref, rtol=8e-3, atol=8e-3)
        assert zero[:R].abs().sum() == 0 and zero[R].abs().sum() > 0


def make_pool(n_blocks, layers, nkv, fill=float("nan")):
    # unwritten slots hold NaN: a kernel that lets masked keys/values leak fails loudly
    return torch.full((n_blocks, layers, 2, nkv, 16, 128), fill, dtype=torch.bfloat16, device="cuda")


def rope_ref(x, pos, theta):
    f = torch.arange(64, dtype=torch.float64, device=x.device)
    inv = theta ** (-(2.0 * f) / 128.0)
    a = pos.double()[:, None] * inv[None, :]
    c, s = a.cos().float()[:, None, :], a.sin().float()[:, None, :]
    x1, x2 = x[..., :64], x[..., 64:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)


@pytest.mark.parametrize("nq,nkv,bias", [(2, 1, False), (32, 8, False), (28, 4, True)])
def test_qkv_rope_append(L, nq, nkv, bias):
    layers, layer, theta = 3, 1, 500000.0
    M = 37
    width = (nq + 2 * nkv) * 128
    qkv = torch.randn(M, width, device="cuda")
    b = (0.1 * torch.randn(width, device="cuda")).bfloat16() if bias else None
    pos = torch.randint(0, 900, (M,), dtype=torch.int32, device="cuda")
    nb = 64
    pool = make_pool(nb, layers, nkv, fill=0.0)
    # each row its own sequence: table = a random permutation slice
    perm = torch.randperm(nb, device="cuda").int()
    bt = perm.repeat(M)  # flat table long enough for pos/16 < 64
    row_bt = (torch.arange(M, device="cuda", dtype=torch.int32) * nb)
    c = torch.empty(2048 * 64, device="cuda"); s = torch.empty(2048 * 64, device="cuda")
    ok(L.ck_rope_table(p(c), p(s), 2048, theta, stream()))
    qout = torch.empty(M, nq * 128, dtype=torch.bfloat16, device="cuda")
    # use distinct positions to avoid two rows writing the same slot
    pos = torch.randperm(1000, device="cuda")[:M].int()
    qkv_in = qkv.clone()
    ok(L.ck_qkv_rope_append(p(qkv), p(b), p(qout), p(pool), p(bt), p(row_bt), p(pos), p(c), p(s), M, nq, nkv, layer,
                            layers, 1, stream()))
    assert qkv.abs().sum() == 0  # zero_after
    x = qkv_in + (b.float() if bias else 0)
    q = rope_ref(x[:, :nq * 128].view(M, nq, 128), pos, theta)
    k = rope_ref(x[:, nq * 128:(nq + nkv) * 128].view(M, nkv, 128), pos, theta)
    v = x[:, (nq + nkv) * 128:].view(M, nkv, 128)
    assert torch.allclose(qout.float().view(M, nq, 128), q, rtol=1e-2, atol=2e-2)
    for m in range(M):
        pp = int(pos[m])
        blk = int(perm[pp // 16])
        assert torch.allclose(pool[blk, layer, 0, :, pp % 16].float(), k[m], rtol=1e-2, atol=2e-2)
        assert torch.allclose(pool[blk, layer, 1, :, pp % 16].float(), v[m], rtol=1e-2, atol=2e-2)


def fill_sequences(pool, layer, lens, nkv, gen):
    """Random K/V for each sequence in freshly allocated blocks; returns tables."""
    nb_total = pool.shape[0]
    perm = torch.randperm(nb_total, device="cuda", generator=gen)
    tables, k_all, v_all, used = [], [], [], 0
    for ln in lens:
        nb = (ln + 15) // 16
        t = perm[used:used + nb].int()
        used += nb
        k = torch.randn(ln, nkv, 128, device="cuda", generator=gen).bfloat16()
        v = torch.randn(ln, nkv, 128, device="cuda", generator=gen).bfloat16()
        for j in range(ln):
            pool[int(t[j // 16]), layer, 0, :, j % 16] = k[j]
            pool[int(t[j // 16]), layer, 1, :, j % 16] = v[j]
        tables.append(t)
        k_all.append(k)
        v_all.append(v)
    return tables, k_all, v_all


def attn_ref(q, k, v, qpos, scale):
    """q [n, nq, 128], k/v [T, nkv, 128]; causal by absolute position."""
    nq, nkv = q.shape[1], k.shape[1]
    G = nq // nkv
    kk = k.float().repeat_interleave(G, 1)
    vv = v.float().repeat_interleave(G, 1)
    s = torch.einsum("nhd,thd->hnt", q.float(), kk) * scale
    T = k.shape[0]
    mask = torch.arange(T, device=q.device)[None, :] > qpos[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    return torch.einsum("hnt,thd->nhd", s.softmax(-1), vv)


def decode_work(lens, bps, reverse=False):
    """Work list of ck_attn_decode_tma: parts of <= bps blocks per sequence, work[i] =
    seq << 16 | nparts << 8 | part, parts of a sequence contiguous; reverse=True lists the
    sequences last-first (the engine's planner orders them heaviest first), so item order
    and sequence order differ."""
    work, item0 = [], [0] * len(lens)
    order = range(len(lens) - 1, -1, -1) if reverse else range(len(lens))
    for s_i in order:
        nblk = (lens[s_i] + 15) // 16
        parts = (nblk + bps - 1) // bps
        assert parts < 256
        item0[s_i] = len(work)
        work += [(s_i << 16) | (parts << 8) | sp for sp in range(parts)]
    return work, item0


@pytest.mark.parametrize("nq,nkv", [(2, 1), (32, 8), (28, 4), (4, 2)])
def test_attn_decode(L, nq, nkv):
    gen = torch.Generator(device="cuda").manual_seed(nq)
    layers, layer = 2, 1
    lens = [1, 15, 16, 17, 100, 333, 1024, 2049]
    # TMA reads whole blocks and masks, so stale slots hold large finite garbage
    pool = make_pool(sum((l + 15) // 16 for l in lens) + 3, layers, nkv, fill=3e4)
    tables, ks, vs = fill_sequences(pool, layer, lens, nkv, gen)
    S = len(lens)
    rows = torch.arange(S, dtype=torch.int32, device="cuda") * 2 + 1  # non-trivial row mapping
    M = 2 * S + 1
    q = torch.randn(M, nq * 128, device="cuda", generator=gen).bfloat16()
    bt = torch.cat(tables)
    offs = np.concatenate([[0], np.cumsum([len(t) for t in tables])[:-1]]).astype(np.int32)
    # (blocks per part, cluster CTAs per part)
    cases = [(64, 1), (3, 1), (64, 2), (5, 4), (64, 8), (1000, 16)]
    for bps, cluster in cases:
        work, item0 = decode_work(lens, bps, reverse=cluster % 2 == 0)
        # keep every argument tensor alive across the call (the caching allocator
        # would otherwise hand the same block to the next temporary)
        t_len, t_off, t_item0, t_work = (torch.tensor(a, dtype=torch.int32, device="cuda")
                                         for a in (lens, offs, item0, work))
        ws = torch.empty(len(work) * nq * 130, device="cuda")
        tickets = torch.zeros(S * nkv, dtype=torch.int32, device="cuda")
        out = torch.zeros(M, nq * 128, dtype=torch.bfloat16, device="cuda")
        scale = 1 / math.sqrt(128)
        ok(L.ck_attn_decode_tma(p(q), p(pool), pool.shape[0], p(bt), p(rows), p(t_len), p(t_off), p(t_item0),
                                p(t_work), len(work), S, cluster, p(ws), p(tickets), p(out), nq, nkv, layer,
                                layers, scale, None, stream()))
        assert tickets.abs().sum() == 0  # self-resetting
        for s_i, ln in enumerate(lens):
            r = int(rows[s_i])
            ref = attn_ref(q[r].view(1, nq, 128), ks[s_i], vs[s_i], torch.tensor([ln - 1], device="cuda"), scale)
            got = out[r].float().view(1, nq, 128)
            assert torch.allclose(got, ref, rtol=2e-2, atol=2e-2), (bps, cluster, ln, (got - ref).abs().max().item())


@pytest.mark.parametrize("nq,nkv", [(2, 1), (32, 8), (28, 4), (4, 2), (32, 4)])
@pytest.mark.parametrize("pos0,qlen", [(0, 1), (0, 77), (0, 256), (300, 64), (1000, 212), (48, 512), (2000, 700),
                                       (1024, 448), (130, 33)])
def test_attn_prefill(L, nq, nkv, pos0, qlen):
    gen = torch.Generator(device="cuda").manual_seed(pos0 + qlen + nq)
    layers, layer = 2, 0
    T = pos0 + qlen
    # whole blocks are read (masked): stale slots must be finite -> large finite garbage
    pool = make_pool((T + 15) // 16 + 5, layers, nkv, fill=3e4)
    tables, ks, vs = fill_sequences(pool, layer, [T], nkv, gen)
    row0 = 3
    q = torch.randn(row0 + qlen + 2, nq * 128, device="cuda", generator=gen).bfloat16()
    out = torch.zeros_like(q)
    scale = 1 / math.sqrt(128)
    qpos = torch.arange(pos0, T, device="cuda")
    ref = attn_ref(q[row0:row0 + qlen].view(qlen, nq, 128), ks[0], vs[0], qpos, scale)
    # no workspace (never split); a full B200 (148 CTAs: splits when the units do not fill
    # it); a small partition (37) and a tiny one (5) that force deep key splits
    for max_ctas in (0, 148, 37, 5):
        out.zero_()
        ws = torch.empty(max(1, L.ck_attn_prefill_ws_floats(max_ctas)), device="cuda")
        tickets = torch.zeros(max(1, max_ctas), dtype=torch.int32, device="cuda")
        ok(L.ck_attn_prefill_pp(p(q), q.shape[0], p(pool), pool.shape[0], p(tables[0]), row0, qlen, pos0, p(out), nq,
                                nkv, layer, layers, scale, p(ws) if max_ctas else None, p(tickets), max_ctas,
                                stream()))
        got = out[row0:row0 + qlen].float().view(qlen, nq, 128)
        assert torch.allclose(got, ref, rtol=3e-2, atol=3e-2), (max_ctas, (got - ref).abs().max().item())
        assert out[:row0].abs().sum() == 0 and out[row0 + qlen:].abs().sum() == 0
        assert tickets.abs().sum() == 0  # self-resetting


def test_silu_mul_and_argmax(L):
    M, F = 9, 1024
    gu = torch.randn(M, 2 * F, device="cuda") * 3
    act = torch.empty(M, F, dtype=torch.bfloat16, device="cuda")
    gu_in = gu.clone()
    ok(L.ck_silu_mul(p(gu), p(act), M, F, 1, stream()))
    assert gu.abs().sum() == 0
    g, u = gu_in[:, 0::2], gu_in[:, 1::2]
    assert torch.allclose(act.float(), torch.nn.functional.silu(g) * u, rtol=1e-2, atol=1e-2)

    R, V = 5, 128256
    logits = torch.randn(R, V, device="cuda")
    logits[1, 77] = 100.0
    logits[1, 99] = 100.0  # tie: lowest index wins
    rid = torch.tensor([4, 0, 2, 1, 3], dtype=torch.int32, device="cuda")
    out_idx = torch.tensor([10, 11, 12, 13, 14], dtype=torch.int64, device="cuda")
    last = torch.full((5,), -1, dtype=torch.int32, device="cuda")
    out_tok = torch.full((20,), -1, dtype=torch.int32, device="cuda")
    ws = torch.empty(64 * R, device="cuda")
    tickets = torch.zeros(R, dtype=torch.int32, device="cuda")
    keep = logits.clone()
    sink = torch.zeros(20, V, device="cuda")  # logits test hook: rows land at out_idx
    ok(L.ck_argmax_emit(p(logits), R, V, p(rid), p(out_idx), p(last), p(out_tok), p(ws), p(tickets), 1, p(sink),
                        stream()))
    assert logits.abs().sum() == 0  # zero_after: cleared for the next red.add LM head
    logits = keep
    assert torch.equal(sink[10:15], keep) and sink[:10].abs().sum() == 0
    assert tickets.abs().sum() == 0
    want = logits.argmax(-1).int()
    assert int(want[1]) == 77
    assert torch.equal(out_tok[10:15], want)
    assert torch.equal(last[rid.long()], want)


def test_kv_copy(L):
    bb = 2 * 1024 * 1024 + 16 * 7
    src = torch.randint(0, 255, (10 * bb,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros(12 * bb, dtype=torch.uint8, device="cuda")
    sid = torch.tensor([3, 0, 9, 4], dtype=torch.int32, device="cuda")
    did = torch.tensor([11, 2, 0, 5], dtype=torch.int32, device="cuda")
    ok(L.ck_kv_copy(p(src), p(sid), p(dst), p(did), 4, bb, stream()))
    for s, d in zip(sid.tolist(), did.tolist()):
        assert torch.equal(dst[d * bb:(d + 1) * bb], src[s * bb:(s + 1) * bb])
    assert dst[bb:2 * bb].sum() == 0


class DecodeRope(ctypes.Structure):
    _fields_ = [("qkv", ctypes.c_void_p), ("cos_tab", ctypes.c_void_p), ("sin_tab", ctypes.c_void_p)]


@pytest.mark.parametrize("nq,nkv", [(32, 8), (28, 4)])
def test_attn_decode_fused_rope(L, nq, nkv):
    """ck_attn_decode_tma with a ck_decode_rope: RoPE(q), RoPE(k) / v of the decode token
    from the fp32 qkv rows, the token's K/V written to its pool slot, attention over the
    whole context == ck_qkv_rope_append followed by the unfused kernel."""
    gen = torch.Generator(device="cuda").manual_seed(nq + 1)
    layers, layer, theta = 2, 1, 500000.0
    lens = [1, 16, 17, 300, 1025, 2048]
    S = len(lens)
    pool = make_pool(sum((n + 15) // 16 for n in lens) + 2, layers, nkv, fill=0.0)
    tables, ks, vs = fill_sequences(pool, layer, [n - 1 for n in lens], nkv, gen) if False else (None, None, None)
    # context of len-1 tokens per sequence, the last slot left for the decode token
    perm = torch.randperm(pool.shape[0], device="cuda", generator=gen).int()
    tables, used = [], 0
    for n in lens:
        nb = (n + 15) // 16
        tables.append(perm[used:used + nb])
        used += nb
        for j in range(n - 1):
            pool[int(tables[-1][j // 16]), layer, :, :, j % 16] = torch.randn(2, nkv, 128, device="cuda",
                                                                             generator=gen).bfloat16()
    width = (nq + 2 * nkv) * 128
    rows = torch.arange(S, dtype=torch.int32, device="cuda")
    qkv = torch.randn(S, width, device="cuda", generator=gen)
    c = torch.empty(4096 * 64, device="cuda"); s_ = torch.empty(4096 * 64, device="cuda")
    ok(L.ck_rope_table(p(c), p(s_), 4096, theta, stream()))
    bt = torch.cat(tables)
    offs = torch.tensor(np.concatenate([[0], np.cumsum([len(t) for t in tables])[:-1]]), dtype=torch.int32,
                        device="cuda")
    t_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    pos = t_len - 1
    scale = 1 / math.sqrt(128)
    for cluster in (1, 4):
        work, item0 = decode_work([1] * S, 1)
        t_item0 = torch.tensor(item0, dtype=torch.int32, device="cuda")
        t_work = torch.tensor(work, dtype=torch.int32, device="cuda")
        ws = torch.empty(len(work) * nq * 130, device="cuda")
        tickets = torch.zeros(S * nkv, dtype=torch.int32, device="cuda")
        # reference: rope kernel (writes q and the token's K/V) + unfused attention
        pool_ref = pool.clone()
        q = torch.empty(S, nq * 128, dtype=torch.bfloat16, device="cuda")
        row_bt = offs.clone()
        ok(L.ck_qkv_rope_append(p(qkv.clone()), None, p(q), p(pool_ref), p(bt), p(row_bt), p(pos), p(c), p(s_), S,
                                nq, nkv, layer, layers, 0, stream()))
        out_ref = torch.zeros(S, nq * 128, dtype=torch.bfloat16, device="cuda")
        ok(L.ck_attn_decode_tma(p(q), p(pool_ref), pool.shape[0], p(bt), p(rows), p(t_len), p(offs), p(t_item0),
                                p(t_work), len(work), S, cluster, p(ws), p(tickets), p(out_ref), nq, nkv, layer,
                                layers, scale, None, stream()))
        # fused
        pool_f = pool.clone()
        out = torch.zeros_like(out_ref)
        rope = DecodeRope(qkv.data_ptr(), c.data_ptr(), s_.data_ptr())
        ok(L.ck_attn_decode_tma(None, p(pool_f), pool.shape[0], p(bt), p(rows), p(t_len), p(offs), p(t_item0),
                                p(t_work), len(work), S, cluster, p(ws), p(tickets), p(out), nq, nkv, layer,
                                layers, scale, ctypes.byref(rope), stream()))
        assert torch.allclose(out.float(), out_ref.float(), rtol=2e-2, atol=2e-2), \
            (cluster, (out.float() - out_ref.float()).abs().max().item())
        assert torch.equal(pool_f, pool_ref)  # the token's K/V slot written identically


def fill_sequences_fast(pool, layer, lens, nkv, gen):
    """fill_sequences with one indexed store per sequence (long contexts)."""
    perm = torch.randperm(pool.shape[0], device="cuda", generator=gen)
    tables, k_all, v_all, used = [], [], [], 0
    for ln in lens:
        nb = (ln + 15) // 16
        t = perm[used:used + nb].int()
        used += nb
        k = torch.randn(ln, nkv, 128, device="cuda", generator=gen).bfloat16()
        v = torch.randn(ln, nkv, 128, device="cuda", generator=gen).bfloat16()
        j = torch.arange(ln, device="cuda")
        blk, slot = t[j // 16].long(), j % 16
        pool[blk, layer, 0, :, slot] = k
        pool[blk, layer, 1, :, slot] = v
        tables.append(t)
        k_all.append(k)
        v_all.append(v)
    return tables, k_all, v_all


@pytest.mark.parametrize("nq,nkv", [(32, 8), (28, 4)])
def test_attn_long_context(L, nq, nkv):
    """SURVEY.md §8 K5/K6 maxima: decode over 16k and ~49k-token contexts (the 4x long
    trace's largest request), both kernels, and chunked prefill at a 16k prefix."""
    gen = torch.Generator(device="cuda").manual_seed(7 * nq)
    layers, layer = 2, 1
    lens = [16384, 49157, 3]
    pool = make_pool(sum((l + 15) // 16 for l in lens) + 2, layers, nkv, fill=3e4)
    tables, ks, vs = fill_sequences_fast(pool, layer, lens, nkv, gen)
    S = len(lens)
    rows = torch.arange(S, dtype=torch.int32, device="cuda")
    q = torch.randn(S, nq * 128, device="cuda", generator=gen).bfloat16()
    bt = torch.cat(tables)
    offs = np.concatenate([[0], np.cumsum([len(t) for t in tables])[:-1]]).astype(np.int32)
    scale = 1 / math.sqrt(128)
    refs = [attn_ref(q[s].view(1, nq, 128), ks[s], vs[s], torch.tensor([ln - 1], device="cuda"), scale)
            for s, ln in enumerate(lens)]
    for bps, cluster in [(128, 8), (400, 16), (64, 1)]:
        work, item0 = decode_work(lens, bps, reverse=cluster == 8)
        t_len, t_off, t_item0, t_work = (torch.tensor(a, dtype=torch.int32, device="cuda")
                                         for a in (lens, offs, item0, work))
        ws = torch.empty(len(work) * nq * 130, device="cuda")
        tickets = torch.zeros(S * nkv, dtype=torch.int32, device="cuda")
        out = torch.zeros(S, nq * 128, dtype=torch.bfloat16, device="cuda")
        ok(L.ck_attn_decode_tma(p(q), p(pool), pool.shape[0], p(bt), p(rows), p(t_len), p(t_off), p(t_item0),
                                p(t_work), len(work), S, cluster, p(ws), p(tickets), p(out), nq, nkv, layer,
                                layers, scale, None, stream()))
        assert tickets.abs().sum() == 0
        for s_i in range(S):
            got = out[s_i].float().view(1, nq, 128)
            assert torch.allclose(got, refs[s_i], rtol=2e-2, atol=2e-2), (bps, cluster, lens[s_i], (got - refs[s_i]).abs().max().item())
    # chunked prefill of 512 tokens over a 16k prefix (the first sequence's KV)
    pos0, qlen = 16384 - 512, 512
    q2 = torch.randn(qlen, nq * 128, device="cuda", generator=gen).bfloat16()
    out2 = torch.zeros_like(q2)
    ref2 = attn_ref(q2.view(qlen, nq, 128), ks[0], vs[0], torch.arange(pos0, pos0 + qlen, device="cuda"), scale)
    for max_ctas in (0, 108):  # unsplit, and split into balanced key pieces
        ws2 = torch.empty(max(1, L.ck_attn_prefill_ws_floats(max_ctas)), device="cuda")
        tk2 = torch.zeros(max(1, max_ctas), dtype=torch.int32, device="cuda")
        out2.zero_()
        ok(L.ck_attn_prefill_pp(p(q2), q2.shape[0], p(pool), pool.shape[0], p(tables[0]), 0, qlen, pos0, p(out2), nq,
                                nkv, layer, layers, scale, p(ws2) if max_ctas else None, p(tk2), max_ctas, stream()))
        assert torch.allclose(out2.float().view(qlen, nq, 128), ref2, rtol=3e-2, atol=3e-2), \
            (max_ctas, (out2.float().view(qlen, nq, 128) - ref2).abs().max().item())
