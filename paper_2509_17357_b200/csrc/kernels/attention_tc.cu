// Causal prefill / chunk attention on the 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// One CTA = 128 query rows of one head. Per 128-key tile j of the paged KV:
//   S_j  = Q K_j^T              tcgen05.mma M=128 (queries) N=128 (keys) K=128 (dims) -> TMEM
//   P_j  = exp2(S_j * scale - m) softmax warps: TMEM -> registers (one query row per
//                               thread: row max / sum need no shuffles) -> bf16 P in smem
//   O   += P_j V_j              tcgen05.mma M=128 N=128 (dims) K=128 (keys), V consumed
//                               MN-major straight from its TMA tile -> TMEM accumulator
// O is rescaled lazily (only when a row max grows by more than 2^8), so the common
// case never touches the accumulator between MMAs.
//
// Shared-memory operands are in the canonical 128-byte-swizzled layouts TMA produces
// (Swizzle<3,4,3>): K-major for Q, K and P (rows of 64 bf16), MN-major for V (64-dim
// rows per key, 8-key atoms at SBO = 1 KiB, the second 64-dim half at LBO = 16 KiB).
// K/V tiles are gathered from the paged pool with one 16-row TMA box per 16-token
// block and 64-dim half (pool viewed as a [rows][128] bf16 matrix).
//
// Warp roles (192 threads): warp 0 TMA producer, warp 1 MMA issuer (+ TMEM owner),
// warps 2..5 softmax / correction / epilogue (TMEM lane quarter = warp % 4).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <cstdio>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "cronus_ck.h"

namespace {

using namespace ck;

constexpr int kQ = 128;       // query rows per CTA
constexpr int kKT = 128;      // keys per tile
constexpr int kHalf = 16384;  // one 128-row x 64-col bf16 swizzled region
constexpr int kTileBytes = 2 * kHalf;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units


__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t addr) {
    // MN-major, 128B swizzle: LBO = 16 KiB between the two 64-element MN halves,
    // SBO = 1 KiB between 8-row (K) groups.
    return (static_cast<uint64_t>((addr >> 4) & 0x3FFFu)) | (static_cast<uint64_t>(kHalf >> 4) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
           (static_cast<uint64_t>(2) << 61);
}

__host__ __device__ constexpr uint32_t idesc_attn(bool b_mn_major) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | (static_cast<uint32_t>(128 >> 3) << 17) |
           (static_cast<uint32_t>(128 >> 4) << 24);
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
        "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
// 2^x on the FMA pipe: Cody-Waite split x = i + f, f in [0, 1), cubic fit of 2^f (max
// relative error 2.6e-4, far below the bf16 rounding P gets next); x < -127 -> ~0.
__device__ __forceinline__ float exp2_poly(float x) {
    x = fmaxf(x, -127.f);
    const float xi = floorf(x);
    const float f = x - xi;
    const float pf = fmaf(fmaf(fmaf(0.07558665f, f, 0.22877255f), f, 0.69511601f), f, 1.0f);
    return __int_as_float(__float_as_int(pf) + (static_cast<int>(xi) << 23));
}
// MUFU.EX2 alone (exp2f adds range fix-ups: 3 more instructions per element)
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ============================================================ ping-pong kernel
// Two 128-row query tiles per CTA, one softmax warpgroup each, sharing the K/V rings. P never
// leaves the tensor memory: each softmax warpgroup writes its bf16 P over the first 64 columns
// of its own S tile (tcgen05.st) and the PV MMA takes A straight from TMEM. The MMA warp
// interleaves
//   PV_0(j), S_0(j+1), PV_1(j), S_1(j+1)
// so while one warpgroup exponentiates, the tensor pipe works for the other. tcgen05 MMAs
// execute in issue order, so S_i(j+1) (same TMEM as P_i(j)) follows PV_i(j), and "S_i(j) done"
// implies "PV_i(j-1) done": the O rescale needs no extra barrier.
// TMEM: S_0 | S_1 | O_0 | O_1 (128 columns each). smem: Q_0, Q_1, K[2], V[2] = 192 KB.
//
// GQA packing: a 128-row tile holds HT query heads x TT = 128/HT tokens of ONE kv head
// (head-major: rows [g*TT, (g+1)*TT) are head g), so a CTA's two tiles cover 2*TT tokens of
// HT heads and every K/V tile it loads serves all of them; HT = 4 for LLaMA (G = 4), 1 for
// Qwen2 (G = 7). A unit = (kv head, head subgroup, token block of 2*TT tokens).
//
// Balanced key split: when the units do not fill the partition (a 448-token chunk is 56 units
// for 108 SMs), each unit's key tiles are cut into pieces of at most steps_cap tiles (the
// smallest cap whose piece count fits one wave, chosen on the host). A piece's unnormalised O
// (fp32, coalesced [tile][dim/4][row] float4 layout) and per-row (max, sum) go to ws; the last
// piece of a unit to finish (self-resetting ticket) folds the others into its own TMEM
// accumulator and writes the bf16 rows. Units run heaviest first (token blocks descending).
//
// PDL: K/V tiles wholly below pos0 were written by earlier passes (a pass starts with a
// stream-ordered metadata copy), so the producer requests up to two of them before
// griddepcontrol.wait; Q and the chunk's own keys only after it.
constexpr int kPPOffQ = 0;
constexpr int kPPOffK = kPPOffQ + 2 * kTileBytes;
constexpr int kPPOffV = kPPOffK + 2 * kTileBytes;
constexpr int kPPOffTab = kPPOffV + 2 * kTileBytes;  // the piece's block ids (first kPPTabMax)
constexpr int kPPTabMax = 2048;                      // 256 key tiles = 32k keys
constexpr int kPPOffBar = kPPOffTab + kPPTabMax * 4;
constexpr int kPPSmemBytes = kPPOffBar + 256 + 1024;
constexpr int kPPThreads = 320;  // producer, MMA, 2 x 4 softmax warps
constexpr int kPfWsO = 2 * 32 * 128 * 4;  // floats of one piece's partial O: [tile][dim/4][row] float4
constexpr int kPfWsFloats = kPfWsO + 2 * 128 * 2;  // + (max, sum) per tile row

struct PfParams {
    int q_row0, q_len, pos0;
    int nq, nkv, layer, n_layers;
    float scale_log2;
    __nv_bfloat16* out;
    const int* table;
    int n_tb;       // token blocks of 2*TT tokens
    int steps_cap;  // key tiles per piece at most
    float* ws;      // piece partials [grid][kPfWsFloats]
    int* tickets;   // [grid], zero, self-resetting
};

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]: A (M=128 rows in lanes, K packed 2 x bf16 per column).
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Key tiles of token block tb (its second tile's last valid token).
template <int HT>
__host__ __device__ __forceinline__ int pf_steps(int q_len, int pos0, int tb) {
    constexpr int TT = 128 / HT;
    const int end = (tb + 1) * 2 * TT < q_len ? (tb + 1) * 2 * TT : q_len;
    return (pos0 + end + kKT - 1) / kKT;
}

template <int HT>
__global__ void __launch_bounds__(kPPThreads, 1)
    attn_prefill_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                           PfParams p) {
    constexpr int TT = 128 / HT;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kPPOffBar);
    uint64_t* q_full = bar + 0;    // [2] per query tile
    uint64_t* k_full = bar + 2;    // [2] per stage
    uint64_t* k_empty = bar + 4;   // [2]
    uint64_t* v_full = bar + 6;    // [2]
    uint64_t* v_empty = bar + 8;   // [2]
    uint64_t* s_full = bar + 10;   // [2] per query tile
    uint64_t* p_full = bar + 12;   // [2] per query tile (4 warp arrivals)
    uint64_t* o_done = bar + 14;   // [2] per query tile
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);
    int* s_last = reinterpret_cast<int*>(bar + 17);

    const int warp = warp_id(), lane = lane_id();
    // ---- which piece of which unit (metadata only: safe before griddepcontrol.wait)
    const int G = p.nq / p.nkv, NS = G / HT, per_tb = p.nkv * NS;
    int b = blockIdx.x, tb = p.n_tb - 1, pieces = 1, n_steps = 1;
    for (; tb >= 0; --tb) {  // heaviest token blocks first
        n_steps = pf_steps<HT>(p.q_len, p.pos0, tb);
        pieces = (n_steps + p.steps_cap - 1) / p.steps_cap;
        if (b < per_tb * pieces) break;
        b -= per_tb * pieces;
    }
    const int unit = b / pieces, piece = b % pieces;
    const int kvh = unit / NS, h_base = kvh * G + (unit % NS) * HT;
    const int bsz = (n_steps + pieces - 1) / pieces;
    const int j0 = piece * bsz, j1 = min(n_steps, j0 + bsz), jmax = j1 - j0;
    const int first_cta = blockIdx.x - piece;
    int t_base[2], cnt[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        t_base[i] = tb * 2 * TT + i * TT;
        const int n_i = (p.pos0 + min(p.q_len, t_base[i] + TT) + kKT - 1) / kKT;
        cnt[i] = t_base[i] < p.q_len ? max(0, min(j1, n_i) - j0) : 0;
    }
    const int n_qt = t_base[1] < p.q_len ? 2 : 1;

    if (warp == 1) {
        tmem_alloc(tmem_slot, 512);
        tmem_relinquish();
    } else if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmQ);
        tma_prefetch_desc(&tmKV);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&q_full[i], 1);
            mbar_init(&k_full[i], 1);
            mbar_init(&k_empty[i], 1);
            mbar_init(&v_full[i], 1);
            mbar_init(&v_empty[i], 1);
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 4);
            mbar_init(&o_done[i], 1);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_launch();

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        // The piece's block ids are staged in smem by the whole warp (coalesced, one round
        // trip; metadata, so before griddepcontrol.wait): a TMA issue loop that reads the
        // table from global pays one dependent L2 round trip per 16-token block.
        const int n_tab = (p.pos0 + min(p.q_len, (tb + 1) * 2 * TT) + 15) / 16;
        int* tab = reinterpret_cast<int*>(sm + kPPOffTab);
        const int t0 = j0 * (kKT / 16), n_stage = min(jmax * (kKT / 16), kPPTabMax);
        for (int x = lane; x < n_stage; x += 32) {
            const int ti = t0 + x;
            tab[x] = p.table[ti < n_tab ? ti : 0];  // past the end: any finite block (masked)
        }
        __syncwarp();
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();
            auto load_kv = [&](int jj) {
                const int s = jj & 1;
                int rows[kKT / 16];
#pragma unroll
                for (int bb = 0; bb < kKT / 16; ++bb) {
                    const int x = jj * (kKT / 16) + bb, ti = t0 + x;
                    const int id = x < kPPTabMax ? tab[x] : p.table[ti < n_tab ? ti : 0];
                    rows[bb] = ((id * p.n_layers + p.layer) * 2 + 0) * p.nkv * 16 + kvh * 16;
                }
                mbar_wait(&k_empty[s], ((jj >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&k_full[s], kTileBytes);
                uint8_t* K = sm + kPPOffK + s * kTileBytes;
#pragma unroll
                for (int bb = 0; bb < kKT / 16; ++bb) {
                    tma_load_2d_hint(K + bb * 2048, &tmKV, &k_full[s], 0, rows[bb], keep);
                    tma_load_2d_hint(K + kHalf + bb * 2048, &tmKV, &k_full[s], 64, rows[bb], keep);
                }
                mbar_wait(&v_empty[s], ((jj >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&v_full[s], kTileBytes);
                uint8_t* V = sm + kPPOffV + s * kTileBytes;
#pragma unroll
                for (int bb = 0; bb < kKT / 16; ++bb) {
                    tma_load_2d_hint(V + bb * 2048, &tmKV, &v_full[s], 0, rows[bb] + p.nkv * 16, keep);
                    tma_load_2d_hint(V + kHalf + bb * 2048, &tmKV, &v_full[s], 64, rows[bb] + p.nkv * 16, keep);
                }
            };
            int jj = 0;
            while (jj < 2 && jj < jmax && (j0 + jj + 1) * kKT <= p.pos0) load_kv(jj++);  // prefix: pre-wait
            pdl_wait();
            for (int i = 0; i < n_qt; ++i) {
                mbar_arrive_expect_tx(&q_full[i], kTileBytes);
                uint8_t* Q = sm + kPPOffQ + i * kTileBytes;
                const int qrow = p.q_row0 + t_base[i];
#pragma unroll
                for (int g = 0; g < HT; ++g) {
                    tma_load_2d(Q + g * TT * 128, &tmQ, &q_full[i], (h_base + g) * 128, qrow);
                    tma_load_2d(Q + kHalf + g * TT * 128, &tmQ, &q_full[i], (h_base + g) * 128 + 64, qrow);
                }
            }
            for (; jj < jmax; ++jj) load_kv(jj);
        } else {
            pdl_wait();
        }
    } else if (warp == 1) {
        pdl_wait();
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t id_s = idesc_attn(false), id_o = idesc_attn(true);
            for (int i = 0; i < n_qt; ++i) mbar_wait(&q_full[i], 0);
            auto issue_s = [&](int i, int jj) {  // S_i(j) = Q_i K(j)^T -> TMEM cols [128 i, +128)
                const uint32_t q0 = smem_u32(sm + kPPOffQ + i * kTileBytes);
                const uint32_t k0 = smem_u32(sm + kPPOffK + (jj & 1) * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                    tc_mma_bf16(tmem + i * 128, sdesc_sw128(q0 + off), sdesc_sw128(k0 + off), id_s, kk > 0);
                }
                tc_commit(&s_full[i]);
            };
            auto issue_pv = [&](int i, int jj) {  // O_i += P_i(j) V(j), P from TMEM (packed bf16 pairs)
                mbar_wait(&p_full[i], jj & 1);
                tc_fence_after();
                const uint32_t v0 = smem_u32(sm + kPPOffV + (jj & 1) * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    tc_mma_ts(tmem + 256 + i * 128, tmem + i * 128 + kk * 8, sdesc_mn_sw128(v0 + kk * 2048), id_o,
                              (jj > 0 || kk > 0) ? 1u : 0u);
                if (jj == cnt[i] - 1) tc_commit(&o_done[i]);
            };
            auto k_ready = [&](int jj) {
                mbar_wait(&k_full[jj & 1], (jj >> 1) & 1);
                tc_fence_after();
            };
            if (jmax > 0) {
                k_ready(0);
                for (int i = 0; i < 2; ++i)
                    if (cnt[i] > 0) issue_s(i, 0);
                tc_commit(&k_empty[0]);
            }
            for (int jj = 0; jj < jmax; ++jj) {
                const bool next = jj + 1 < jmax;
                mbar_wait(&v_full[jj & 1], (jj >> 1) & 1);
                tc_fence_after();
                if (next) k_ready(jj + 1);
                for (int i = 0; i < 2; ++i) {
                    if (jj < cnt[i]) issue_pv(i, jj);
                    if (jj + 1 < cnt[i]) issue_s(i, jj + 1);
                }
                tc_commit(&v_empty[jj & 1]);
                if (next) tc_commit(&k_empty[(jj + 1) & 1]);
            }
        }
    } else {
        pdl_wait();
        // ------------------------------------------------------------ softmax warpgroups
        const int i = (warp - 2) >> 2;  // query tile of this warpgroup
        const int cnt_i = i ? cnt[1] : cnt[0], tb_i = i ? t_base[1] : t_base[0];  // (no local-memory indexing)
        const int qw = warp & 3;
        const int row = qw * 32 + lane;
        const int tok = tb_i + row % TT;
        const int head = h_base + row / TT;
        const int qpos = p.pos0 + tok;
        const int warp_q0 = p.pos0 + tb_i + (qw * 32) % TT;
        const uint32_t lane_base = static_cast<uint32_t>(qw * 32) << 16;
        const uint32_t s_col = tmem + lane_base + i * 128, o_col = tmem + lane_base + 256 + i * 128;
        float m_ref = -INFINITY, l_sum = 0.f;
        for (int jj = 0; jj < cnt_i; ++jj) {
            mbar_wait(&s_full[i], jj & 1);
            tc_fence_after();
            uint32_t sv[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(s_col + c * 32, sv[c]);
            tmem_ld_wait();
            const int key0 = (j0 + jj) * kKT;
            // row max over 128 columns as 8 independent chains (one warp per SM sub-partition
            // per warpgroup: a single 128-long fmax chain would cost ~512 cycles of latency)
            float pmx[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) pmx[e] = -INFINITY;
            if (key0 + kKT - 1 <= warp_q0) {
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) pmx[e & 7] = fmaxf(pmx[e & 7], __uint_as_float(sv[c][e]));
            } else {
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        if (key0 + c * 32 + e > qpos) sv[c][e] = __float_as_uint(-INFINITY);
                        pmx[e & 7] = fmaxf(pmx[e & 7], __uint_as_float(sv[c][e]));
                    }
            }
            float mx = fmaxf(fmaxf(fmaxf(pmx[0], pmx[1]), fmaxf(pmx[2], pmx[3])),
                             fmaxf(fmaxf(pmx[4], pmx[5]), fmaxf(pmx[6], pmx[7])));
            mx *= p.scale_log2;
            const bool need = __any_sync(0xffffffffu, mx > m_ref + kRescaleThreshold || m_ref == -INFINITY);
            if (need) {
                const float m_new = fmaxf(m_ref, mx);
                const float corr = m_ref == -INFINITY ? 0.f : exp2f(m_ref - m_new);
                l_sum *= corr;
                m_ref = m_new;
                if (jj > 0) {  // PV_i(j-1) retired before S_i(j) (in-order tensor pipe)
#pragma unroll 1
                    for (int c = 0; c < 8; ++c) {  // 16 columns at a time: S stays in registers
                        uint32_t o[16];
                        tmem_ld16(o_col + c * 16, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
                        tmem_st16(o_col + c * 16, o);
                    }
                }
            }
            // P = exp2(S * scale - m) -> bf16 pairs over S's first 64 columns; the row sum as 8
            // independent chains (see the max above)
            float rsp[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) rsp[e] = 0.f;
            // a row whose keys in this piece are all masked keeps m = -inf: P = 0, not NaN
            const float m_use = m_ref == -INFINITY ? 0.f : m_ref;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t pk[16];
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const bool poly = g == 3;
                    float pv[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float x = fmaf(__uint_as_float(sv[c][g * 8 + e]), p.scale_log2, -m_use);
                        pv[e] = poly ? exp2_poly(x) : ex2_approx(x);
                        rsp[e] += pv[e];
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) pk[g * 4 + e] = pack_bf16x2(pv[2 * e], pv[2 * e + 1]);
                }
                tmem_st16(s_col + c * 16, pk);
            }
            tmem_st_wait();
            l_sum += ((rsp[0] + rsp[1]) + (rsp[2] + rsp[3])) + ((rsp[4] + rsp[5]) + (rsp[6] + rsp[7]));
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[i]);
        }
        if (cnt_i > 0) {
            mbar_wait(&o_done[i], 0);
            tc_fence_after();
        }
        __nv_bfloat16* dst = p.out + static_cast<size_t>(p.q_row0 + tok) * p.nq * 128 + head * 128;
        const bool store = i < n_qt && tok < p.q_len;
        if (pieces == 1) {
            // ---- epilogue: O / l -> bf16 rows
            const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
            if (cnt_i > 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[32];
                    tmem_ld32(o_col + c * 32, o);
                    tmem_ld_wait();
                    if (store) {
#pragma unroll
                        for (int e = 0; e < 32; e += 8) {
                            uint4 w;
                            w.x = pack_bf16x2(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv);
                            w.y = pack_bf16x2(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
                            w.z = pack_bf16x2(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv);
                            w.w = pack_bf16x2(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv);
                            *reinterpret_cast<uint4*>(dst + c * 32 + e) = w;
                        }
                    }
                }
            }
        } else {
            // ---- split unit: publish this piece's partial, the last piece merges
            float* ws = p.ws + static_cast<size_t>(blockIdx.x) * kPfWsFloats;
            float4* wo = reinterpret_cast<float4*>(ws) + i * 32 * 128;
            if (cnt_i > 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[32];
                    tmem_ld32(o_col + c * 32, o);
                    tmem_ld_wait();
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4)
                        __stcg(wo + (c * 8 + q4) * 128 + row,
                               make_float4(__uint_as_float(o[4 * q4]), __uint_as_float(o[4 * q4 + 1]),
                                           __uint_as_float(o[4 * q4 + 2]), __uint_as_float(o[4 * q4 + 3])));
                }
            }
            __stcg(reinterpret_cast<float2*>(ws + kPfWsO) + i * 128 + row,
                   make_float2(cnt_i > 0 ? m_ref : -INFINITY, cnt_i > 0 ? l_sum : 0.f));
            __threadfence();
            softmax_bar();
            if (threadIdx.x == 64) {
                const int prev = atomicAdd(&p.tickets[first_cta], 1);
                *s_last = prev == pieces - 1;
                if (prev == pieces - 1) p.tickets[first_cta] = 0;  // self-resetting
            }
            softmax_bar();
            if (*s_last && i < n_qt) {  // warp-uniform: tcgen05.ld below is warp-collective
                __threadfence();
                const float m_own = cnt_i > 0 ? m_ref : -INFINITY;
                float M = m_own;
                for (int q = 0; q < pieces; ++q) {
                    if (q == piece) continue;
                    const float* wq = p.ws + static_cast<size_t>(first_cta + q) * kPfWsFloats + kPfWsO;
                    M = fmaxf(M, __ldcg(wq + 2 * (i * 128 + row)));
                }
                const float f_own = m_own == -INFINITY ? 0.f : exp2f(m_own - M);
                float L = f_own * l_sum;
                auto weight = [&](int q, float* l_q) {  // exp2(m_q - M) of piece q (0 for an empty one)
                    const float2 ml = __ldcg(reinterpret_cast<const float2*>(
                                                 p.ws + static_cast<size_t>(first_cta + q) * kPfWsFloats + kPfWsO) +
                                             i * 128 + row);
                    *l_q = ml.y;
                    return ml.x == -INFINITY ? 0.f : exp2f(ml.x - M);
                };
                for (int q = 0; q < pieces; ++q) {
                    if (q == piece) continue;
                    float lq;
                    const float f = weight(q, &lq);
                    L += f * lq;
                }
                const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll 1
                for (int c = 0; c < 4; ++c) {
                    float acc[32];
                    if (cnt_i > 0) {
                        uint32_t o[32];
                        tmem_ld32(o_col + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) acc[e] = __uint_as_float(o[e]) * f_own;
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e) acc[e] = 0.f;
                    }
                    for (int q = 0; q < pieces; ++q) {
                        float lq;
                        const float f = q == piece ? 0.f : weight(q, &lq);
                        if (f == 0.f) continue;
                        const float4* oq = reinterpret_cast<const float4*>(p.ws + static_cast<size_t>(first_cta + q) *
                                                                                      kPfWsFloats) +
                                           i * 32 * 128;
#pragma unroll
                        for (int q4 = 0; q4 < 8; ++q4) {
                            const float4 v = __ldcg(oq + (c * 8 + q4) * 128 + row);
                            acc[4 * q4] += f * v.x;
                            acc[4 * q4 + 1] += f * v.y;
                            acc[4 * q4 + 2] += f * v.z;
                            acc[4 * q4 + 3] += f * v.w;
                        }
                    }
#pragma unroll
                    for (int e = 0; e < 32; e += 8) {
                        if (!store) break;
                        uint4 w;
                        w.x = pack_bf16x2(acc[e] * inv, acc[e + 1] * inv);
                        w.y = pack_bf16x2(acc[e + 2] * inv, acc[e + 3] * inv);
                        w.z = pack_bf16x2(acc[e + 4] * inv, acc[e + 5] * inv);
                        w.w = pack_bf16x2(acc[e + 6] * inv, acc[e + 7] * inv);
                        *reinterpret_cast<uint4*>(dst + c * 32 + e) = w;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace

namespace ck {
// ------------------------------------------------------------------ host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_map_2d(const void* ptr, unsigned long long rows, unsigned long long cols, unsigned box_rows, CUtensorMap* m) {
    static std::mutex mu;
    static std::unordered_map<std::string, CUtensorMap> cache;
    char key[96];
    std::snprintf(key, sizeof key, "%p/%llu/%llu/%u", ptr, rows, cols, box_rows);
    {
        std::lock_guard<std::mutex> g(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *m = it->second;
            return 0;
        }
    }
    static EncodeFn enc = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        return reinterpret_cast<EncodeFn>(f);
    }();
    if (!enc) return static_cast<int>(cudaErrorNotSupported);
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {64, box_rows};
    cuuint32_t es[2] = {1, 1};
    if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return static_cast<int>(cudaErrorInvalidValue);
    std::lock_guard<std::mutex> g(mu);
    if (cache.size() > 4096) cache.clear();
    cache.emplace(key, *m);
    return 0;
}

}  // namespace ck

namespace {
// Host plan of a prefill launch: token blocks, key tiles per piece, grid. Splits only when the
// units do not fill `max_ctas` (and a workspace exists): then the smallest cap whose pieces fit
// one wave, with at most 16 pieces per unit (the merge's register budget).
template <int HT>
int pf_plan(int q_len, int pos0, int nq, int nkv, int max_ctas, bool can_split, int* n_tb_out, int* cap_out) {
    constexpr int TT = 128 / HT;
    const int n_tb = (q_len + 2 * TT - 1) / (2 * TT);
    const int per_tb = nkv * (nq / nkv / HT);
    const int n_max = pf_steps<HT>(q_len, pos0, n_tb - 1);
    auto grid_for = [&](int cap) {
        long long g = 0;
        for (int tb = 0; tb < n_tb; ++tb) g += static_cast<long long>(per_tb) * ((pf_steps<HT>(q_len, pos0, tb) + cap - 1) / cap);
        return g;
    };
    int cap = n_max;
    if (can_split && static_cast<long long>(per_tb) * n_tb < max_ctas) {
        long long total = 0;
        for (int tb = 0; tb < n_tb; ++tb) total += static_cast<long long>(per_tb) * pf_steps<HT>(q_len, pos0, tb);
        int c = static_cast<int>(std::max<long long>(std::max(1, (n_max + 15) / 16), (total + max_ctas - 1) / max_ctas));
        while (c < n_max && grid_for(c) > max_ctas) ++c;
        cap = std::min(c, n_max);
    }
    *n_tb_out = n_tb;
    *cap_out = cap;
    return static_cast<int>(grid_for(cap));
}

template <int HT>
int launch_prefill(const void* q, int q_rows_total, const CUtensorMap& mkv, const int* bt, int q_row0, int q_len,
                   int pos0, void* out, int nq, int nkv, int layer, int n_layers, float scale, float* ws, int* tickets,
                   int max_ctas, cudaStream_t st) {
    constexpr int TT = 128 / HT;
    CUtensorMap mq;
    int rc = make_map_2d(q, static_cast<unsigned long long>(q_rows_total), static_cast<unsigned long long>(nq) * 128,
                         TT, &mq);
    if (rc) return rc;
    static unsigned mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(mask & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(attn_prefill_pp_kernel<HT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kPPSmemBytes);
        if (e != cudaSuccess) return static_cast<int>(e);
        mask |= 1u << dev;
    }
    PfParams prm;
    prm.q_row0 = q_row0;
    prm.q_len = q_len;
    prm.pos0 = pos0;
    prm.nq = nq;
    prm.nkv = nkv;
    prm.layer = layer;
    prm.n_layers = n_layers;
    prm.scale_log2 = scale * kLog2e;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.table = bt;
    prm.ws = ws;
    prm.tickets = tickets;
    const int grid = pf_plan<HT>(q_len, pos0, nq, nkv, max_ctas, ws != nullptr && tickets != nullptr && max_ctas > 0,
                                 &prm.n_tb, &prm.steps_cap);
    if (ws && grid > max_ctas && prm.steps_cap < pf_steps<HT>(q_len, pos0, prm.n_tb - 1))
        return static_cast<int>(cudaErrorInvalidValue);  // split pieces beyond the workspace
    return launch_pdl(attn_prefill_pp_kernel<HT>, dim3(grid), dim3(kPPThreads), kPPSmemBytes, st, mq, mkv, prm);
}
}  // namespace

extern "C" int ck_attn_prefill_pp(const void* q, int q_rows_total, const void* kv_pool, long long pool_blocks,
                                  const int* bt, int q_row0, int q_len, int pos0, void* out, int nq, int nkv, int layer,
                                  int n_layers, float scale, float* ws, int* tickets, int max_ctas, void* stream) {
    if (q_len <= 0) return 0;
    if (nq % nkv) return static_cast<int>(cudaErrorInvalidValue);
    CUtensorMap mkv;
    const unsigned long long pool_rows = static_cast<unsigned long long>(pool_blocks) * n_layers * 2 * nkv * 16;
    const int rc = make_map_2d(kv_pool, pool_rows, 128, 16, &mkv);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int G = nq / nkv;
    if (G % 4 == 0)
        return launch_prefill<4>(q, q_rows_total, mkv, bt, q_row0, q_len, pos0, out, nq, nkv, layer, n_layers, scale,
                                 ws, tickets, max_ctas, st);
    if (G % 2 == 0)
        return launch_prefill<2>(q, q_rows_total, mkv, bt, q_row0, q_len, pos0, out, nq, nkv, layer, n_layers, scale,
                                 ws, tickets, max_ctas, st);
    return launch_prefill<1>(q, q_rows_total, mkv, bt, q_row0, q_len, pos0, out, nq, nkv, layer, n_layers, scale, ws,
                             tickets, max_ctas, st);
}

extern "C" long long ck_attn_prefill_ws_floats(int max_ctas) { return static_cast<long long>(max_ctas) * kPfWsFloats; }
