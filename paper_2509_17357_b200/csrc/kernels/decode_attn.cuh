// Building blocks of the decode (single query token) paged attention (attention.cu):
// per-block math on mma.sync, the 4-warp smem merge and the ticketed global merge of a
// sequence's parts.
//
// Per warp, 16-token K/V blocks (128-B XOR-swizzled rows: conflict-free ldmatrix) are
// consumed by
//   S[16 x 16] = Qpad[16 x 128] K^T   (G query heads padded to 16 MMA rows, mma.sync)
//   O[16 x 128] += P[16 x 16] V       online softmax in registers.
// The 4 warps merge in smem; part partials merge in the last group to finish
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
    const int nsplit = (a.work[item] >> 8) & 0xff;
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
        const int i0 = a.seq_item0[s], i1 = i0 + nsplit;
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

}  // namespace ck
