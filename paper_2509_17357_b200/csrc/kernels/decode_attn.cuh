// Decode (single query token) paged attention for one (split item, kv head), executed by
// a group of 4 warps (128 threads). Shared by the standalone split-KV kernel
// (attention.cu) and the persistent decode forward (mega_decode.cu).
//
// Per warp: every 4th 16-token block of the split streams through a cp.async ring
// (STAGES deep, 128-B XOR-swizzled rows: conflict-free ldmatrix) and is consumed by
//   S[16 x 16] = Qpad[16 x 128] K^T   (G query heads padded to 16 MMA rows, mma.sync)
//   O[16 x 128] += P[16 x 16] V       online softmax in registers.
// The 4 warps merge in smem; split partials merge in the last group to finish
// (atomic ticket per (sequence, kv head), self-resetting).
#pragma once

#include "common.cuh"

namespace ck {

constexpr int kDHD = 128;                   // head dim
constexpr int kDBlk = 16;                   // tokens per KV block
constexpr int kDTile = kDBlk * kDHD;        // elements of one (block, layer, K|V, head) tile
constexpr int kDTileBytes = kDTile * 2;     // 4 KiB

__device__ __forceinline__ size_t kv_tile_off(int block, int layer, int kv, int head, int n_layers, int nkv) {
    return ((static_cast<size_t>(block) * n_layers + layer) * 2 + kv) * static_cast<size_t>(nkv) * kDTile +
           static_cast<size_t>(head) * kDTile;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t swz(int row, int chunk) {  // byte offset in a [16][128] bf16 tile
    return static_cast<uint32_t>(row * 256 + ((chunk ^ (row & 7)) << 4));
}
// Named barrier over the 4-warp group (id != 0 so other warps of the CTA are free).
__device__ __forceinline__ void group_bar(int id) { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }

struct DecodeAttnArgs {
    const __nv_bfloat16* q;
    const __nv_bfloat16* pool;
    const int* bt;
    const int* seq_row;
    const int* seq_len;
    const int* seq_bt;
    const int* seq_item0;
    const int* work;
    int blocks_per_split;
    float* ws;
    int* tickets;
    __nv_bfloat16* out;
    int nq, nkv, layer, n_layers;
    float qk_scale_log2;
    // Fused RoPE + KV append of the decode token (TMA kernel only; null = off): q, k, v
    // are read from the fp32 QKV accumulator [rows][(nq + 2 nkv) * 128] instead of `q`,
    // the token's K/V is written to its pool slot and patched into the staged block.
    const float* qkv;
    const float* cos_tab;
    const float* sin_tab;
};

// [16 tok][256 B] rows (cp.async ring): 16-B chunk c of row r at c ^ (r & 7).
struct SwzRow256 {
    __device__ __forceinline__ uint32_t operator()(int row, int chunk) const { return swz(row, chunk); }
};
// The layout two 64-dim TMA SWIZZLE_128B boxes land in: [2 halves][16 tok][128 B],
// 16-B chunk c of a 128-B line at c ^ (row & 7).
struct SwzTma128 {
    __device__ __forceinline__ uint32_t operator()(int row, int chunk) const {
        return static_cast<uint32_t>((chunk >> 3) * 2048 + row * 128 + (((chunk & 7) ^ (row & 7)) << 4));
    }
};

// One 16-token K/V block against the warp's padded query tile:
//   S[16 x 16] = Qpad K^T, online softmax (base 2), O[16 x 128] += P V.
// tok0 = first token of the block; keys >= len are masked.
template <typename SW>
__device__ __forceinline__ void dec_block(const uint8_t* K, const uint8_t* V, const uint32_t (&qf)[8][4],
                                          float (&o)[16][4], float& m_run, float& l_run, int tok0, int len, float qk,
                                          int lane) {
    const SW sw{};
    const int tq = lane & 3;
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        uint32_t b[4];
        const int r = (lane & 7) + ((lane >> 4) << 3), ch = 2 * kk + ((lane >> 3) & 1);
        ldsm_x4(b, K + sw(r, ch));
        mma16816(s0, qf[kk], b[0], b[1]);
        mma16816(s1, qf[kk], b[2], b[3]);
    }
    float sc[4];
    sc[0] = tok0 + 2 * tq < len ? s0[0] * qk : -INFINITY;
    sc[1] = tok0 + 2 * tq + 1 < len ? s0[1] * qk : -INFINITY;
    sc[2] = tok0 + 8 + 2 * tq < len ? s1[0] * qk : -INFINITY;
    sc[3] = tok0 + 9 + 2 * tq < len ? s1[1] * qk : -INFINITY;
    float mx = fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m_run, mx);  // finite: token 0 of every block is valid
    const float corr = exp2f(m_run - mn);
    float p[4], rs = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        p[e] = exp2f(sc[e] - mn);
        rs += p[e];
    }
    rs += __shfl_xor_sync(0xffffffffu, rs, 1);
    rs += __shfl_xor_sync(0xffffffffu, rs, 2);
    l_run = l_run * corr + rs;
    m_run = mn;
    uint32_t pf[4];
    pf[0] = pack_bf16x2(p[0], p[1]);
    pf[1] = 0u;  // padded rows 8..15
    pf[2] = pack_bf16x2(p[2], p[3]);
    pf[3] = 0u;
#pragma unroll
    for (int nd = 0; nd < 16; ++nd) {
        o[nd][0] *= corr;
        o[nd][1] *= corr;
    }
#pragma unroll
    for (int nd = 0; nd < 16; nd += 2) {
        uint32_t b[4];
        const int r = (lane & 7) + (((lane >> 3) & 1) << 3), ch = nd + (lane >> 4);
        ldsm_x4_t(b, V + sw(r, ch));
        mma16816(o[nd], pf, b[0], b[1]);
        mma16816(o[nd + 1], pf, b[2], b[3]);
    }
}

// Per-head result of one work item before normalisation: res[h * kDRes + 0] = running
// max M (log2 units), [1] = sum L, [2 + d] = unnormalised accumulator A[d].
constexpr int kDRes = kDHD + 2;
constexpr int kDResOff = 4 * 16 * kDHD * 4;  // res lives after the warp-merge scratch in the ring

// Merge the group's 4 warps (ring reused as [4][16][128] fp32 scratch) into res.
template <int G>
__device__ void dec_merge_warps(uint8_t* ring_all, float* small, const float (&o)[16][4], float m_run, float l_run,
                                int t, int bar_id, float* res) {
    float(*wm)[16] = reinterpret_cast<float(*)[16]>(small);
    float(*wl)[16] = reinterpret_cast<float(*)[16]>(small + 64);
    const int warp = t >> 5, lane = t & 31;
    const int g = lane >> 2, tq = lane & 3;
    group_bar(bar_id);
    float* wo = reinterpret_cast<float*>(ring_all);
    if (tq == 0) {
        wm[warp][g] = m_run;
        wl[warp][g] = l_run;
    }
#pragma unroll
    for (int nd = 0; nd < 16; ++nd) {
        wo[(warp * 16 + g) * kDHD + nd * 8 + 2 * tq] = o[nd][0];
        wo[(warp * 16 + g) * kDHD + nd * 8 + 2 * tq + 1] = o[nd][1];
    }
    group_bar(bar_id);
    for (int i = t; i < G * kDHD; i += 128) {
        const int h = i / kDHD, d = i % kDHD;
        float M = -INFINITY;
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) M = fmaxf(M, wm[w2][h]);
        float Ls = 0.f, A = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) {
            const float f = wm[w2][h] == -INFINITY ? 0.f : exp2f(wm[w2][h] - M);
            Ls += wl[w2][h] * f;
            A += wo[(w2 * 16 + h) * kDHD + d] * f;
        }
        res[h * kDRes + 2 + d] = A;
        if (d == 0) {
            res[h * kDRes] = M;
            res[h * kDRes + 1] = Ls;
        }
    }
    group_bar(bar_id);
}

// Store one work item's merged result: the output row when the sequence has a single
// item, else its partial; the last item of each (sequence, kv head) to finish merges
// all partials (self-resetting ticket).
template <int G>
__device__ void dec_store(const DecodeAttnArgs& a, int item, int kvh, const float* res, float* small, int t,
                          int bar_id) {
    int* s_last = reinterpret_cast<int*>(small + 128);
    const int s = a.work[item] >> 16;
    const int nsplit = a.seq_item0[s + 1] - a.seq_item0[s];
    const int row = a.seq_row[s];
    const int nq = a.nq;
    const bool single = nsplit == 1;
    for (int i = t; i < G * kDHD; i += 128) {
        const int h = i / kDHD, d = i % kDHD;
        const float M = res[h * kDRes], Ls = res[h * kDRes + 1], A = res[h * kDRes + 2 + d];
        if (single) {
            a.out[static_cast<size_t>(row) * nq * kDHD + (kvh * G + h) * kDHD + d] = f2bf(Ls > 0.f ? A / Ls : 0.f);
        } else {
            float* part = a.ws + (static_cast<size_t>(item) * nq + kvh * G + h) * kDRes;
            part[2 + d] = A;
            if (d == 0) {
                part[0] = M;
                part[1] = Ls;
            }
        }
    }
    if (single) {
        group_bar(bar_id);  // scratch / small reused by the group's next item
        return;
    }
    __threadfence();
    group_bar(bar_id);
    if (t == 0) {
        const int prev = atomicAdd(&a.tickets[s * a.nkv + kvh], 1);
        *s_last = prev == nsplit - 1;
        if (*s_last) a.tickets[s * a.nkv + kvh] = 0;  // self-resetting
    }
    group_bar(bar_id);
    if (*s_last) {
        __threadfence();
        const int i0 = a.seq_item0[s], i1 = a.seq_item0[s + 1];
        for (int i = t; i < G * kDHD; i += 128) {
            const int h = i / kDHD, d = i % kDHD;
            const int hq = kvh * G + h;
            float M = -INFINITY;
            for (int it = i0; it < i1; ++it) M = fmaxf(M, __ldcg(a.ws + (static_cast<size_t>(it) * nq + hq) * kDRes));
            float Ls = 0.f, A = 0.f;
            for (int it = i0; it < i1; ++it) {
                const float* part = a.ws + (static_cast<size_t>(it) * nq + hq) * kDRes;
                const float pm = __ldcg(part);
                const float f = pm == -INFINITY ? 0.f : exp2f(pm - M);
                Ls += __ldcg(part + 1) * f;
                A += __ldcg(part + 2 + d) * f;
            }
            a.out[static_cast<size_t>(row) * nq * kDHD + hq * kDHD + d] = f2bf(Ls > 0.f ? A / Ls : 0.f);
        }
    }
    group_bar(bar_id);
}

template <int G>
__device__ void dec_merge(const DecodeAttnArgs& a, int item, int kvh, uint8_t* ring_all, float* small,
                          const float (&o)[16][4], float m_run, float l_run, int t, int bar_id) {
    float* res = reinterpret_cast<float*>(ring_all + kDResOff);
    dec_merge_warps<G>(ring_all, small, o, m_run, l_run, t, bar_id, res);
    dec_store<G>(a, item, kvh, res, small, t, bar_id);
}

// smem: sQ 4 KiB (1 KiB aligned), ring = 4 * STAGES * 8 KiB (also reused as the 32 KiB
// warp-merge scratch), small = 2 * 64 floats + 1 int. t = thread index in the group.
template <int G, int STAGES>
__device__ void decode_attn_item(const DecodeAttnArgs& a, int item, int kvh, uint8_t* sQ, uint8_t* ring_all,
                                 float* small, int t, int bar_id) {
    static_assert(4 * STAGES * 2 * kDTileBytes >= kDResOff + 8 * kDRes * 4, "merge scratch must fit in the ring");

    const int wk = a.work[item];
    const int s = wk >> 16, split = wk & 0xffff;
    const int len = a.seq_len[s];
    const int nblk = (len + kDBlk - 1) / kDBlk;
    const int b0 = split * a.blocks_per_split, b1 = min(nblk, b0 + a.blocks_per_split);
    const int warp = t >> 5, lane = t & 31;
    const int* table = a.bt + a.seq_bt[s];
    const int row = a.seq_row[s];
    const int nq = a.nq;

    {  // Q (G rows, zero padded to 16)
        const __nv_bfloat16* qrow = a.q + static_cast<size_t>(row) * nq * kDHD + static_cast<size_t>(kvh) * G * kDHD;
        for (int c = t; c < 16 * 16; c += 128) {
            const int r = c >> 4, ch = c & 15;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (r < G) v = *reinterpret_cast<const uint4*>(qrow + r * kDHD + ch * 8);
            *reinterpret_cast<uint4*>(sQ + swz(r, ch)) = v;
        }
    }
    uint8_t* ring = ring_all + static_cast<size_t>(warp) * STAGES * 2 * kDTileBytes;
    const int first = b0 + warp;
    const int mine = first < b1 ? (b1 - first + 3) / 4 : 0;
    auto load = [&](int i) {
        const int b = first + 4 * i;
        const int blk = table[b];
        const __nv_bfloat16* kt = a.pool + kv_tile_off(blk, a.layer, 0, kvh, a.n_layers, a.nkv);
        const __nv_bfloat16* vt = kt + static_cast<size_t>(a.nkv) * kDTile;
        uint8_t* dK = ring + (i % STAGES) * 2 * kDTileBytes;
        uint8_t* dV = dK + kDTileBytes;
        const int valid = min(kDBlk, len - b * kDBlk);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = lane + 32 * j;
            const int r = c >> 4, ch = c & 15;
            const bool ok = r < valid;  // slots past the sequence end may hold stale data: zero-fill
            cp_async16(dK + swz(r, ch), kt + r * kDHD + ch * 8, ok);
            cp_async16(dV + swz(r, ch), vt + r * kDHD + ch * 8, ok);
        }
    };
#pragma unroll
    for (int i = 0; i < STAGES - 1; ++i) {
        if (i < mine) load(i);
        cp_commit();
    }
    group_bar(bar_id);  // sQ visible
    uint32_t qf[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int r = lane & 15, ch = 2 * kk + (lane >> 4);
        ldsm_x4(qf[kk], sQ + swz(r, ch));
    }
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;

    for (int i = 0; i < mine; ++i) {
        cp_wait<STAGES - 2>();
        __syncwarp();
        const uint8_t* K = ring + (i % STAGES) * 2 * kDTileBytes;
        dec_block<SwzRow256>(K, K + kDTileBytes, qf, o, m_run, l_run, (first + 4 * i) * kDBlk, len, a.qk_scale_log2,
                             lane);
        __syncwarp();
        const int nxt = i + STAGES - 1;
        if (nxt < mine) load(nxt);
        cp_commit();
    }
    cp_wait<0>();

    dec_merge<G>(a, item, kvh, ring_all, small, o, m_run, l_run, t, bar_id);
}

}  // namespace ck
