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

struct AttnParams {
    int q_row0, q_len, pos0;
    int nq, nkv, layer, n_layers;
    int row_stride_blk;  // pool rows per block = n_layers * 2 * nkv * 16
    float scale_log2;
    __nv_bfloat16* out;
    const int* table;
};

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

// ============================================================ ping-pong variant (default)
// Two 128-row query tiles of one head per CTA (rows [r0, r0+128) and [r0+128, r0+256)),
// one softmax warpgroup each, sharing the K/V rings. P never leaves the tensor memory:
// each softmax warpgroup writes its bf16 P over the first 64 columns of its own S tile
// (tcgen05.st) and the PV MMA takes A straight from TMEM. The MMA warp interleaves
//   PV_0(j), S_0(j+1), PV_1(j), S_1(j+1)
// so while one warpgroup exponentiates, the tensor pipe works for the other. tcgen05
// MMAs execute in issue order, so S_i(j+1) (same TMEM as P_i(j)) follows PV_i(j), and
// "S_i(j) done" implies "PV_i(j-1) done": the O rescale needs no extra barrier.
// TMEM: S_0 | S_1 | O_0 | O_1 (128 columns each). smem: Q_0, Q_1, K[2], V[2] = 192 KB.
constexpr int kPPOffQ = 0;
constexpr int kPPOffK = kPPOffQ + 2 * kTileBytes;
constexpr int kPPOffV = kPPOffK + 2 * kTileBytes;
constexpr int kPPOffBar = kPPOffV + 2 * kTileBytes;
constexpr int kPPSmemBytes = kPPOffBar + 256 + 1024;
constexpr int kPPThreads = 320;  // producer, MMA, 2 x 4 softmax warps

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

__global__ void __launch_bounds__(kPPThreads, 1)
    attn_prefill_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                           AttnParams p) {
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

    const int warp = warp_id(), lane = lane_id();
    const int ct = gridDim.x - 1 - blockIdx.x, h = blockIdx.y;  // heaviest tiles first
    const int kvh = h / (p.nq / p.nkv);
    const int r0 = ct * 2 * kQ;
    const int n_qt = r0 + kQ < p.q_len ? 2 : 1;
    int n_kt[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) n_kt[i] = (p.pos0 + min(p.q_len, r0 + (i + 1) * kQ) + kKT - 1) / kKT;
    const int n_kt_max = n_kt[n_qt - 1];

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
    pdl_wait();

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            const uint64_t keep = policy_evict_last();
            for (int i = 0; i < n_qt; ++i) {
                mbar_arrive_expect_tx(&q_full[i], kTileBytes);
                const int qrow = p.q_row0 + r0 + i * kQ;
                tma_load_2d(sm + kPPOffQ + i * kTileBytes, &tmQ, &q_full[i], h * 128, qrow);
                tma_load_2d(sm + kPPOffQ + i * kTileBytes + kHalf, &tmQ, &q_full[i], h * 128 + 64, qrow);
            }
            const int n_tab = (p.pos0 + min(p.q_len, r0 + n_qt * kQ) + 15) / 16;
            auto row_of = [&](int j, int b) {
                const int tb = j * (kKT / 16) + b;
                const int blk = p.table[tb < n_tab ? tb : 0];  // past the end: any finite block (masked)
                return ((blk * p.n_layers + p.layer) * 2 + 0) * p.nkv * 16 + kvh * 16;
            };
            for (int j = 0; j < n_kt_max; ++j) {
                const int s = j & 1;
                mbar_wait(&k_empty[s], ((j >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&k_full[s], kTileBytes);
                uint8_t* K = sm + kPPOffK + s * kTileBytes;
                for (int b = 0; b < kKT / 16; ++b) {
                    const int rk = row_of(j, b);
                    tma_load_2d_hint(K + b * 2048, &tmKV, &k_full[s], 0, rk, keep);
                    tma_load_2d_hint(K + kHalf + b * 2048, &tmKV, &k_full[s], 64, rk, keep);
                }
                mbar_wait(&v_empty[s], ((j >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&v_full[s], kTileBytes);
                uint8_t* V = sm + kPPOffV + s * kTileBytes;
                for (int b = 0; b < kKT / 16; ++b) {
                    const int rv = row_of(j, b) + p.nkv * 16;
                    tma_load_2d_hint(V + b * 2048, &tmKV, &v_full[s], 0, rv, keep);
                    tma_load_2d_hint(V + kHalf + b * 2048, &tmKV, &v_full[s], 64, rv, keep);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            constexpr uint32_t id_s = idesc_attn(false), id_o = idesc_attn(true);
            for (int i = 0; i < n_qt; ++i) mbar_wait(&q_full[i], 0);
            auto issue_s = [&](int i, int j) {  // S_i(j) = Q_i K(j)^T -> TMEM cols [128 i, +128)
                const uint32_t q0 = smem_u32(sm + kPPOffQ + i * kTileBytes);
                const uint32_t k0 = smem_u32(sm + kPPOffK + (j & 1) * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kHalf + (kk & 3) * 32;
                    tc_mma_bf16(tmem + i * 128, sdesc_sw128(q0 + off), sdesc_sw128(k0 + off), id_s, kk > 0);
                }
                tc_commit(&s_full[i]);
            };
            auto issue_pv = [&](int i, int j) {  // O_i += P_i(j) V(j), P from TMEM (packed bf16 pairs)
                mbar_wait(&p_full[i], j & 1);
                tc_fence_after();
                const uint32_t v0 = smem_u32(sm + kPPOffV + (j & 1) * kTileBytes);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk)
                    tc_mma_ts(tmem + 256 + i * 128, tmem + i * 128 + kk * 8, sdesc_mn_sw128(v0 + kk * 2048), id_o,
                              (j > 0 || kk > 0) ? 1u : 0u);
                if (j == n_kt[i] - 1) tc_commit(&o_done[i]);
            };
            auto k_ready = [&](int j) {
                mbar_wait(&k_full[j & 1], (j >> 1) & 1);
                tc_fence_after();
            };
            k_ready(0);
            for (int i = 0; i < n_qt; ++i)
                if (n_kt[i] > 0) issue_s(i, 0);
            tc_commit(&k_empty[0]);
            for (int j = 0; j < n_kt_max; ++j) {
                const bool next = j + 1 < n_kt_max;
                mbar_wait(&v_full[j & 1], (j >> 1) & 1);
                tc_fence_after();
                if (next) k_ready(j + 1);
                for (int i = 0; i < n_qt; ++i) {
                    if (j < n_kt[i]) issue_pv(i, j);
                    if (j + 1 < n_kt[i]) issue_s(i, j + 1);
                }
                tc_commit(&v_empty[j & 1]);
                if (next) tc_commit(&k_empty[(j + 1) & 1]);
            }
        }
    } else {
        // ------------------------------------------------------------ softmax warpgroups
        const int i = (warp - 2) >> 2;  // query tile of this warpgroup
        if (i < n_qt) {
            const int qw = warp & 3;
            const int row = qw * 32 + lane;
            const int qbase = r0 + i * kQ;
            const int qpos = p.pos0 + qbase + row;
            const int warp_q0 = p.pos0 + qbase + qw * 32;
            const uint32_t lane_base = static_cast<uint32_t>(qw * 32) << 16;
            const uint32_t s_col = tmem + lane_base + i * 128, o_col = tmem + lane_base + 256 + i * 128;
            float m_ref = -INFINITY, l_sum = 0.f;
            for (int j = 0; j < n_kt[i]; ++j) {
                mbar_wait(&s_full[i], j & 1);
                tc_fence_after();
                uint32_t sv[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(s_col + c * 32, sv[c]);
                tmem_ld_wait();
                const int key0 = j * kKT;
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
                    if (j > 0) {  // PV_i(j-1) retired before S_i(j) (in-order tensor pipe)
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
                // P = exp2(S * scale - m) -> bf16 pairs over S's first 64 columns; the row sum
                // as 8 independent chains (see the max above)
                float rsp[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) rsp[e] = 0.f;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pk[16];
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const bool poly = g == 3;
                        float pv[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float x = fmaf(__uint_as_float(sv[c][g * 8 + e]), p.scale_log2, -m_ref);
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
            // ---- epilogue: O / l -> bf16 rows
            mbar_wait(&o_done[i], 0);
            tc_fence_after();
            const int grow = qbase + row;
            const float inv = l_sum > 0.f ? 1.f / l_sum : 0.f;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t o[32];
                tmem_ld32(o_col + c * 32, o);
                tmem_ld_wait();
                if (grow < p.q_len) {
                    __nv_bfloat16* dst = p.out + static_cast<size_t>(p.q_row0 + grow) * p.nq * 128 + h * 128 + c * 32;
#pragma unroll
                    for (int e = 0; e < 32; e += 8) {
                        uint4 w;
                        w.x = pack_bf16x2(__uint_as_float(o[e]) * inv, __uint_as_float(o[e + 1]) * inv);
                        w.y = pack_bf16x2(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
                        w.z = pack_bf16x2(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv);
                        w.w = pack_bf16x2(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv);
                        *reinterpret_cast<uint4*>(dst + e) = w;
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

extern "C" int ck_attn_prefill_pp(const void* q, int q_rows_total, const void* kv_pool, long long pool_blocks,
                                  const int* bt, int q_row0, int q_len, int pos0, void* out, int nq, int nkv, int layer,
                                  int n_layers, float scale, void* stream) {
    if (q_len <= 0) return 0;
    CUtensorMap mq, mkv;
    int rc = make_map_2d(q, static_cast<unsigned long long>(q_rows_total), static_cast<unsigned long long>(nq) * 128,
                         kQ, &mq);
    if (rc) return rc;
    const unsigned long long pool_rows = static_cast<unsigned long long>(pool_blocks) * n_layers * 2 * nkv * 16;
    rc = make_map_2d(kv_pool, pool_rows, 128, 16, &mkv);
    if (rc) return rc;
    static unsigned mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(mask & (1u << dev))) {
        cudaError_t e =
            cudaFuncSetAttribute(attn_prefill_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPPSmemBytes);
        if (e != cudaSuccess) return static_cast<int>(e);
        mask |= 1u << dev;
    }
    AttnParams prm;
    prm.q_row0 = q_row0;
    prm.q_len = q_len;
    prm.pos0 = pos0;
    prm.nq = nq;
    prm.nkv = nkv;
    prm.layer = layer;
    prm.n_layers = n_layers;
    prm.row_stride_blk = n_layers * 2 * nkv * 16;
    prm.scale_log2 = scale * kLog2e;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.table = bt;
    const dim3 grid((q_len + 2 * kQ - 1) / (2 * kQ), nq);
    return launch_pdl(attn_prefill_pp_kernel, grid, dim3(kPPThreads), kPPSmemBytes, static_cast<cudaStream_t>(stream),
                      mq, mkv, prm);
}
