// Dense projection GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   out[m, n] (op)= sum_k X[m, k] * W[n, k]          X: activations [M, K] bf16
//                                                    W: weights     [N, K] bf16
// Every LLaMA/Qwen2 projection (QKV, O, gate_up, down, LM head) is this shape.
//
// Design (B200-first, "swap AB"): the weight matrix is the MMA's M operand
// (128 weight rows per tile, UMMA_M = 128) and the token batch is the MMA's N
// operand (BN = 32..256 tokens). This one kernel therefore covers
//   * decode-only CPI iterations (M = n_decode ~ 10..128 tokens): a 128 x BN tile
//     per 64-deep K step is weight-streaming bound; split-K spreads the weight
//     stream over all 148 SMs and the fp32 partials meet in L2 via red.add;
//   * chunked / PPI prefill (M = 512 .. 8192 tokens): 128 x 256 tiles, tensor bound.
//
// Warp roles (192 threads, one CTA per SM, persistent over work units):
//   warp 0      TMA producer (one elected lane): W tile 128x64 + X tile BNx64 per stage
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma (K = 16 each) per stage
//   warps 2..5  epilogue: tcgen05.ld TMEM -> registers -> global (bf16 / fp32 / red.add)
// Pipelines: STAGES-deep smem ring (full/empty mbarriers) and a double-buffered
// TMEM accumulator (tmem_full/tmem_empty) so the epilogue of unit i overlaps the
// MMAs of unit i+1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <unordered_map>

#include "common.cuh"
#include "cronus_ck.h"

namespace {

using namespace ck;

constexpr int kThreads = 192;
constexpr int kTileN = 128;  // weight rows per tile (UMMA M)
constexpr int kTileK = 64;   // K per stage: one 128-byte swizzle row of bf16

struct GemmParams {
    void* out;
    const __nv_bfloat16* bias;  // [N] or null, added once (by the unit that starts at k = 0)
    int M, N, K, ldo;
    int m_tiles, splits, kb_total, kb_per_split, units;
    int epi;
    // stream-K (red.add epilogue only): CTA c owns global K-block iterations
    // [c * iters / grid, (c + 1) * iters / grid) of the (tile, k-block) space, so every
    // CTA streams the same number of weight bytes regardless of tile count.
    int stream_k;
    long long iters;
    // hybrid (SiLU epilogue): the first dp_tiles tiles are whole-tile units (tile
    // blockIdx.x + i * grid, silu(gate) * up straight from TMEM into fuse.act); the
    // remaining tiles' K-blocks — a last wave that would leave most SMs idle — are cut
    // into kb_piece-long stream-K pieces, CTA c taking piece c, red.added into the fp32
    // accumulator `out` [M, N] and finalized by the tile's last piece (ticket).
    int hybrid;
    int dp_tiles;
    int kb_piece;
    long long tail_iters;
    ck_gemm_fuse fuse;
    unsigned long long* probe;  // dev (CRONUS_GEMM_PROBE=1): per-CTA timeline stamps, else null
    int stages;                 // ring depth actually used (<= Cfg<BN, PAIR>::kStages)
    int pair;                   // CTAs per work unit: 1, or 2 (a cta_group::2 pair on one TPC)
};

// The unit iteration works in "unit CTAs": a CTA, or a CTA pair when p.pair == 2 (both CTAs
// of the pair walk the identical unit sequence).
__device__ __forceinline__ int unit_cta(const GemmParams& p) { return static_cast<int>(blockIdx.x) / p.pair; }
__device__ __forceinline__ int unit_grid(const GemmParams& p) { return static_cast<int>(gridDim.x) / p.pair; }

__device__ __forceinline__ void probe_stamp(const GemmParams& p, int slot) {
    if (p.probe != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
        p.probe[blockIdx.x * 6 + slot] = t;
    }
}

// ------------------------------------------------------------------ fused tile finalize
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// CK_FUSE_RMSNORM finalize of tile (nt, mt) of a residual red.add GEMM: clear this tile's
// slice of the next accumulator, then the m-tile's last finished tile normalizes its rows
// (x = out, fp32, complete once every tile of the m-tile passed its ticket). Same
// arithmetic as rmsnorm_kernel (elementwise.cu); only the fp32 sum order differs.
constexpr int kNormMaxVec = 8;  // float4 per thread per row: N <= 8 * 4 * 128 = 4096
__device__ void finalize_norm(const GemmParams& p, int nt, int mt, int BN, int t) {
    const ck_gemm_fuse& f = p.fuse;
    const int m0 = mt * BN, m1 = min(p.M, m0 + BN);
    const int n_tiles = p.N / kTileN;
    if (f.zero != nullptr) {
        const int z4 = f.zero_cols / 4, per = (z4 + n_tiles - 1) / n_tiles;
        const int c0 = nt * per, c1 = min(z4, c0 + per);
        for (int m = m0; m < m1; ++m) {
            float4* z = reinterpret_cast<float4*>(f.zero + static_cast<size_t>(m) * f.zero_cols);
            for (int c = c0 + t; c < c1; c += 128) z[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __shared__ int s_norm;
    __shared__ float s_red[2][4];
    if (t == 0) {
        const int d = atomicAdd(&f.row_tickets[mt], 1);
        s_norm = d == n_tiles - 1;
        if (d == n_tiles - 1) f.row_tickets[mt] = 0;
    }
    epi_bar();
    if (!s_norm) return;
    __threadfence();
    const float* x = static_cast<const float*>(p.out);
    const int n4 = p.N / 4, lane = t & 31, w = t >> 5;
    const uint2* g = reinterpret_cast<const uint2*>(f.gamma);
    for (int m = m0; m < m1; m += 2) {
        float4 v[2][kNormMaxVec];
        float ss[2] = {0.f, 0.f};
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(m + r) * p.ldo);
#pragma unroll
            for (int j = 0; j < kNormMaxVec; ++j) {
                const int i = t + j * 128;
                v[r][j] = (m + r < m1 && i < n4) ? __ldcg(xr + i) : make_float4(0.f, 0.f, 0.f, 0.f);
                ss[r] += v[r][j].x * v[r][j].x + v[r][j].y * v[r][j].y + v[r][j].z * v[r][j].z + v[r][j].w * v[r][j].w;
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ss[r] += __shfl_xor_sync(0xffffffffu, ss[r], o);
            if (lane == 0) s_red[r][w] = ss[r];
        }
        epi_bar();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (m + r >= m1) break;
            const float tot = s_red[r][0] + s_red[r][1] + s_red[r][2] + s_red[r][3];
            const float inv = rsqrtf(tot / static_cast<float>(p.N) + f.eps);
            uint2* o = reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(f.norm_out) + static_cast<size_t>(m + r) * p.N);
#pragma unroll
            for (int j = 0; j < kNormMaxVec; ++j) {
                const int i = t + j * 128;
                if (i < n4) {
                    const uint2 gg = g[i];
                    const float2 g0 = unpack_bf16x2(gg.x), g1 = unpack_bf16x2(gg.y);
                    o[i] = make_uint2(pack_bf16x2(v[r][j].x * inv * g0.x, v[r][j].y * inv * g0.y),
                                      pack_bf16x2(v[r][j].z * inv * g1.x, v[r][j].w * inv * g1.y));
                }
            }
        }
        epi_bar();  // s_red is rewritten by the next row pair
    }
}

// Runs on the 128 epilogue threads (t = 0..127) of the CTA that completed tile (nt, mt).
__device__ void finalize_tile(const GemmParams& p, int nt, int mt, int BN, int t) {
    const ck_gemm_fuse& f = p.fuse;
    float* acc = static_cast<float*>(p.out);
    const int m0 = mt * BN, m1 = min(p.M, m0 + BN);
    const int n0 = nt * kTileN;
    if (f.kind == CK_FUSE_RMSNORM) {
        finalize_norm(p, nt, mt, BN, t);
    } else if (f.kind == CK_FUSE_QKV_ROPE) {
        const int h = nt;  // a 128-column tile is exactly one head
        const int nrot = f.nq + f.nkv;
        const size_t hs = 16 * 128;
        __nv_bfloat16* pool = static_cast<__nv_bfloat16*>(f.kv_pool);
        for (int m = m0; m < m1; ++m) {
            float* row = acc + static_cast<size_t>(m) * p.ldo + n0;
            const int pos = f.row_pos[m];
            if (h < nrot) {
                if (t < 64) {
                    const float a = __ldcg(row + t), b = __ldcg(row + t + 64);
                    if (f.zero_after) {
                        row[t] = 0.f;
                        row[t + 64] = 0.f;
                    }
                    const float c = f.cos_tab[static_cast<size_t>(pos) * 64 + t];
                    const float sn = f.sin_tab[static_cast<size_t>(pos) * 64 + t];
                    __nv_bfloat16* dst;
                    if (h < f.nq) {
                        dst = static_cast<__nv_bfloat16*>(f.q_out) + static_cast<size_t>(m) * f.nq * 128 + h * 128;
                    } else {
                        const int blk = f.bt[f.row_bt[m] + (pos >> 4)];
                        dst = pool + ((static_cast<size_t>(blk) * f.n_layers + f.layer) * 2 * f.nkv + (h - f.nq)) * hs +
                              (pos & 15) * 128;
                    }
                    dst[t] = f2bf(a * c - b * sn);
                    dst[t + 64] = f2bf(b * c + a * sn);
                }
            } else {
                const float v = __ldcg(row + t);
                if (f.zero_after) row[t] = 0.f;
                const int blk = f.bt[f.row_bt[m] + (pos >> 4)];
                pool[((static_cast<size_t>(blk) * f.n_layers + f.layer) * 2 * f.nkv + f.nkv + (h - nrot)) * hs +
                     (pos & 15) * 128 + t] = f2bf(v);
            }
        }
    } else {  // CK_FUSE_SILU: 64 (gate, up) pairs = 32 float4 per row; 16 rows in flight per thread
        const int cg = t & 31;
        __nv_bfloat16* act = static_cast<__nv_bfloat16*>(f.act);
        const int F = p.N / 2;
        constexpr int U = 16;
        for (int base = m0 + (t >> 5); base < m1; base += 4 * U) {
            float4 v[U];
#pragma unroll
            for (int i = 0; i < U; ++i) {
                const int m = base + 4 * i;
                if (m < m1) v[i] = __ldcg(reinterpret_cast<const float4*>(acc + static_cast<size_t>(m) * p.ldo + n0) + cg);
            }
#pragma unroll
            for (int i = 0; i < U; ++i) {
                const int m = base + 4 * i;
                if (m < m1) {
                    if (f.zero_after)
                        reinterpret_cast<float4*>(acc + static_cast<size_t>(m) * p.ldo + n0)[cg] =
                            make_float4(0.f, 0.f, 0.f, 0.f);
                    const float a = __fdividef(v[i].x, 1.f + __expf(-v[i].x)) * v[i].y;
                    const float b = __fdividef(v[i].z, 1.f + __expf(-v[i].z)) * v[i].w;
                    reinterpret_cast<__nv_bfloat162*>(act + static_cast<size_t>(m) * F + n0 / 2)[cg] =
                        __floats2bfloat162_rn(a, b);
                }
            }
        }
    }
}

template <int BN, int PAIR = 1>
struct Cfg {
    static constexpr int kABytes = kTileN * kTileK * 2;
    static constexpr int kBBytes = (BN / PAIR) * kTileK * 2;  // a pair's CTAs hold half the token tile each
    static constexpr int kStageBytes = kABytes + kBBytes;
    // As many stages as fit in ~220 KB: the weight stream is latency bound (Little's
    // law: bytes in flight per SM / loaded HBM latency), so small token tiles get a
    // deeper ring (BN=32: 11 x 20 KB).
    static constexpr int kStages = (220 * 1024) / kStageBytes > 12 ? 12 : (220 * 1024) / kStageBytes;
    static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*align slack*/ + 256 /*barriers*/;
};

__device__ __forceinline__ void decode_unit(const GemmParams& p, int u, int& nt, int& mt, int& kb0, int& kb1) {
    const int per_n = p.m_tiles * p.splits;
    nt = u / per_n;
    const int r = u - nt * per_n;
    mt = r / p.splits;
    const int s = r - mt * p.splits;
    kb0 = s * p.kb_per_split;
    kb1 = min(p.kb_total, kb0 + p.kb_per_split);
}

// Work iteration shared by the producer, MMA and epilogue roles (all three walk the
// identical unit sequence). `pos` starts at first_unit().
__device__ __forceinline__ long long tail_lo(const GemmParams& p) {
    return static_cast<long long>(p.dp_tiles) * p.kb_total + static_cast<long long>(unit_cta(p)) * p.kb_piece;
}
__device__ __forceinline__ long long first_unit(const GemmParams& p) {
    const int c = unit_cta(p);
    if (p.hybrid) return c < p.dp_tiles ? static_cast<long long>(c) * p.kb_total : tail_lo(p);
    return p.stream_k ? (static_cast<long long>(c) * p.iters) / unit_grid(p) : c;
}
// `tail`: the unit is a partial-K piece of a hybrid launch (goes through the accumulator).
__device__ __forceinline__ bool next_unit(const GemmParams& p, long long& pos, int& nt, int& mt, int& kb0, int& kb1,
                                          bool* tail = nullptr) {
    if (p.hybrid) {
        const long long dp_end = static_cast<long long>(p.dp_tiles) * p.kb_total;
        int tile;
        if (pos < dp_end) {
            tile = static_cast<int>(pos / p.kb_total);
            kb0 = 0;
            kb1 = p.kb_total;
            pos += static_cast<long long>(unit_grid(p)) * p.kb_total;
            if (pos >= dp_end) pos = tail_lo(p);
            if (tail) *tail = false;
        } else {
            const long long hi = min(dp_end + p.tail_iters, tail_lo(p) + p.kb_piece);
            if (pos >= hi) return false;
            tile = static_cast<int>(pos / p.kb_total);
            kb0 = static_cast<int>(pos - static_cast<long long>(tile) * p.kb_total);
            kb1 = static_cast<int>(min(static_cast<long long>(p.kb_total), kb0 + (hi - pos)));
            pos += kb1 - kb0;
            if (tail) *tail = true;
        }
        nt = tile / p.m_tiles;
        mt = tile - nt * p.m_tiles;
        return true;
    }
    if (tail) *tail = false;
    if (p.stream_k) {
        const long long end = (static_cast<long long>(unit_cta(p) + 1) * p.iters) / unit_grid(p);
        if (pos >= end) return false;
        const int tile = static_cast<int>(pos / p.kb_total);
        kb0 = static_cast<int>(pos - static_cast<long long>(tile) * p.kb_total);
        kb1 = static_cast<int>(min(static_cast<long long>(p.kb_total), kb0 + (end - pos)));
        nt = tile / p.m_tiles;
        mt = tile - nt * p.m_tiles;
        pos += kb1 - kb0;
        return true;
    }
    if (pos >= p.units) return false;
    decode_unit(p, static_cast<int>(pos), nt, mt, kb0, kb1);
    pos += unit_grid(p);
    return true;
}

// ------------------------------------------------------------------ CTA pair (cta_group::2)
// PAIR == 2: two CTAs of a cluster on one TPC share a 256-weight-row x BN-token tile. Each
// loads its own 128 weight rows and HALF of the token tile (the A / B halves of a
// cta_group::2 MMA), the leader (rank 0) issues M = 256 MMAs that write each CTA's 128 rows x
// BN accumulator into that CTA's TMEM, and every stage moves 16 + BN/2 x 128 B per CTA instead of
// 16 + BN x 128 B: 1.5x less shared-memory fill per FLOP and a 6-deep ring at BN = 256 (4 alone).
__device__ __forceinline__ uint32_t cluster_rank_u32() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of `local` (this CTA's shared::cta address) in CTA `rank`
__device__ __forceinline__ uint32_t mapa_rank(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's smem, completion counted on the pair leader's barrier (cluster address)
__device__ __forceinline__ void tma_load_2d_pair_warp(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0,
                                                      int c1, uint64_t policy) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1, {%3, %4}], [%2], %5;\n"
        "}\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void tc_mma_bf16_pair_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                      uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p, e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive on the barrier at this offset in both CTAs of the pair once the MMAs retire
__device__ __forceinline__ void tc_commit_pair_warp(uint64_t* bar) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
template <int PAIR>
__device__ __forceinline__ void tmem_alloc_g(uint32_t* dst_smem, uint32_t ncols) {
    if constexpr (PAIR == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                     "r"(ncols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
        tmem_alloc(dst_smem, ncols);
        tmem_relinquish();
    }
}
template <int PAIR>
__device__ __forceinline__ void tmem_dealloc_g(uint32_t taddr, uint32_t ncols) {
    if constexpr (PAIR == 2)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
    else
        tmem_dealloc(taddr, ncols);
}

template <int BN, int PAIR>
__global__ void __launch_bounds__(kThreads, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, GemmParams p) {
    using C = Cfg<BN, PAIR>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    const int S = p.stages;
    uint8_t* sB = smem + S * C::kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = warp_id();
    const int lane = lane_id();
    const uint32_t rank = PAIR == 2 ? cluster_rank_u32() : 0u;  // 0 = the pair's MMA leader

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch_desc(&tmW);
            tma_prefetch_desc(&tmX);
        }
        tmem_alloc_g<PAIR>(tmem_slot, C::kTmemCols);
    } else if (warp == 1 && lane == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4 * PAIR);  // one arrive per epilogue warp (of both CTAs: the leader's)
        }
        fence_mbar_init();
    }
    tc_fence_before();
    if constexpr (PAIR == 2)
        cluster_sync_all();  // both CTAs' barriers initialised before any peer TMA / commit reaches them
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) probe_stamp(p, 0);
    // Everything above overlaps the previous kernel under PDL. Only the activations X
    // and the output depend on it: the producer streams the first stages' WEIGHT tiles
    // before griddepcontrol.wait, the epilogue waits before its first store, and the
    // MMA warp only consumes shared memory.
    pdl_launch();

    if (warp == 0) {
        // ------------------------------------------------------------ producer (whole warp,
        // convergent; one elected lane issues: see tc_mma_bf16_warp)
        {
            const uint64_t keep = policy_evict_last();    // activations: reused by every weight tile
            const uint64_t stream = policy_evict_first();  // weights: streamed once per launch
            // TMA of one stage's weight / activation half; a pair's loads complete on the
            // leader's full barrier (cluster address), the leader expects both CTAs' bytes
            auto full_addr = [&](int st) {
                return PAIR == 2 ? mapa_rank(smem_u32(&full[st]), 0) : smem_u32(&full[st]);
            };
            auto load_w = [&](int st, int kb, int nt, uint64_t pol) {
                const int row = (nt * PAIR + static_cast<int>(rank)) * kTileN;
                if constexpr (PAIR == 2)
                    tma_load_2d_pair_warp(sA + st * C::kABytes, &tmW, full_addr(st), kb * kTileK, row, pol);
                else
                    tma_load_2d_hint_warp(sA + st * C::kABytes, &tmW, &full[st], kb * kTileK, row, pol);
            };
            auto load_x = [&](int st, int kb, int mt, uint64_t pol) {
                const int row = mt * BN + static_cast<int>(rank) * (BN / PAIR);
                if constexpr (PAIR == 2)
                    tma_load_2d_pair_warp(sB + st * C::kBBytes, &tmX, full_addr(st), kb * kTileK, row, pol);
                else
                    tma_load_2d_hint_warp(sB + st * C::kBBytes, &tmX, &full[st], kb * kTileK, row, pol);
            };
            // (1) weight prefetch: the first kStages k-blocks of this CTA's work (their
            //     slots are free at kernel start), before the dependency wait
            int pre_nt[C::kStages], pre_mt[C::kStages], pre_kb[C::kStages];
            int n_pre = 0;
            {
                long long pos = first_unit(p);
                int nt, mt, kb0, kb1;
                while (n_pre < S && next_unit(p, pos, nt, mt, kb0, kb1))
                    for (int kb = kb0; kb < kb1 && n_pre < S; ++kb) {
                        if (rank == 0) mbar_expect_tx_warp(&full[n_pre], C::kStageBytes * PAIR);
                        load_w(n_pre, kb, nt, stream);
                        pre_nt[n_pre] = nt, pre_mt[n_pre] = mt, pre_kb[n_pre] = kb;
                        ++n_pre;
                    }
            }
            pdl_wait();
            if (lane == 0) probe_stamp(p, 1);
            // (2) the activation tiles of the prefetched stages
            for (int i = 0; i < n_pre; ++i)
                load_x(i, pre_kb[i], pre_mt[i], keep);
            (void)pre_nt;
            // (3) steady state
            int stage = 0;
            uint32_t phase = 0;
            int issued = 0;
            long long pos = first_unit(p);
            int nt, mt, kb0, kb1;
            while (next_unit(p, pos, nt, mt, kb0, kb1)) {
                for (int kb = kb0; kb < kb1; ++kb, ++issued) {
                    if (issued >= n_pre) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (rank == 0) mbar_expect_tx_warp(&full[stage], C::kStageBytes * PAIR);
                        load_w(stage, kb, nt, stream);
                        load_x(stage, kb, mt, keep);
                    }
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (whole warp;
        // the pair's leader only)
        if (rank == 0) {
            const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);  // provably warp-uniform
            constexpr uint32_t idesc = idesc_bf16_f32(kTileN * PAIR, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            long long pos = first_unit(p);
            int nt, mt, kb0, kb1;
            while (next_unit(p, pos, nt, mt, kb0, kb1)) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tbase + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    if (lane == 0 && p.probe != nullptr && p.probe[blockIdx.x * 6 + 2] == 0) probe_stamp(p, 2);
                    const uint32_t a0 = smem_u32(sA + stage * C::kABytes);
                    const uint32_t b0 = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < kTileK / 16; ++k)
                        if constexpr (PAIR == 2)
                            tc_mma_bf16_pair_warp(d_tmem, sdesc_sw128(a0 + k * 32), sdesc_sw128(b0 + k * 32), idesc,
                                                  (kb > kb0 || k > 0) ? 1u : 0u);
                        else
                            tc_mma_bf16_warp(d_tmem, sdesc_sw128(a0 + k * 32), sdesc_sw128(b0 + k * 32), idesc,
                                             (kb > kb0 || k > 0) ? 1u : 0u);
                    if constexpr (PAIR == 2)
                        tc_commit_pair_warp(&empty[stage]);  // both CTAs' slots free once these MMAs retire
                    else
                        tc_commit_warp(&empty[stage]);  // smem slot free once these MMAs retire
                    if (++stage == S) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if constexpr (PAIR == 2)
                    tc_commit_pair_warp(&tfull[acc]);  // both CTAs' accumulators ready
                else
                    tc_commit_warp(&tfull[acc]);  // accumulator ready for the epilogue
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
            if (lane == 0) probe_stamp(p, 3);
        }
    } else {
        // ------------------------------------------------------------ epilogue
        pdl_wait();  // `out` (residual / zeroed accumulator) is produced upstream
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        long long pos = first_unit(p);
        int nt, mt, kb0, kb1;
        bool tail = false;
        while (next_unit(p, pos, nt, mt, kb0, kb1, &tail)) {
            nt = nt * PAIR + static_cast<int>(rank);  // this CTA's 128 weight rows of the (pair) tile
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int n = nt * kTileN + row;
            const int m_base = mt * BN;
            float bias = 0.f;
            if (p.bias != nullptr && kb0 == 0) bias = bf2f(p.bias[n]);
            // hybrid: whole tiles -> SiLU into fuse.act; partial pieces -> red.add into out
            const int epi = p.hybrid && tail ? CK_EPI_RED_F32 : p.epi;
#pragma unroll 1
            for (int c = 0; c < BN; c += 16) {
                if (m_base + c >= p.M) break;  // warp-uniform
                uint32_t v[16];
                tmem_ld16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c, v);
                tmem_ld_wait();
                const int mlim = min(16, p.M - (m_base + c));
                if (epi == CK_EPI_BF16) {
                    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(m_base + c) * p.ldo + n;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < mlim) o[static_cast<size_t>(j) * p.ldo] = f2bf(__uint_as_float(v[j]) + bias);
                } else if (epi == CK_EPI_SILU_BF16) {
                    // adjacent lanes hold the (gate, up) rows of one activation column
                    const int lda = p.hybrid ? p.N / 2 : p.ldo;
                    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(p.hybrid ? p.fuse.act : p.out) +
                                       static_cast<size_t>(m_base + c) * lda + (n >> 1);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const float g = __uint_as_float(v[j]);
                        const float u = __shfl_xor_sync(0xffffffffu, g, 1);
                        if (!(lane & 1) && j < mlim)
                            o[static_cast<size_t>(j) * lda] = f2bf(__fdividef(g, 1.f + __expf(-g)) * u);
                    }
                } else if (epi == CK_EPI_F32) {
                    float* o = static_cast<float*>(p.out) + static_cast<size_t>(m_base + c) * p.ldo + n;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < mlim) o[static_cast<size_t>(j) * p.ldo] = __uint_as_float(v[j]) + bias;
                } else {
                    // 4x4 register transposes inside each quad of lanes: lane 4g+t ends up
                    // holding rows n0+4g..+3 of column 4b+t, so one 16-byte vector
                    // reduction replaces four scalar atomics.
                    float a[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) a[j] = __uint_as_float(v[j]) + bias;
                    const int t = lane & 3;
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        float* r = a + 4 * b;
                        float x0 = __shfl_xor_sync(0xffffffffu, (t & 1) ? r[0] : r[1], 1);
                        float x1 = __shfl_xor_sync(0xffffffffu, (t & 1) ? r[2] : r[3], 1);
                        if (t & 1) {
                            r[0] = x0;
                            r[2] = x1;
                        } else {
                            r[1] = x0;
                            r[3] = x1;
                        }
                        x0 = __shfl_xor_sync(0xffffffffu, (t & 2) ? r[0] : r[2], 2);
                        x1 = __shfl_xor_sync(0xffffffffu, (t & 2) ? r[1] : r[3], 2);
                        if (t & 2) {
                            r[0] = x0;
                            r[1] = x1;
                        } else {
                            r[2] = x0;
                            r[3] = x1;
                        }
                    }
                    const int n4 = nt * kTileN + q * 32 + (lane & ~3);
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int j = 4 * b + t;
                        if (j < mlim)
                            red_add_v4_f32(static_cast<float*>(p.out) + static_cast<size_t>(m_base + c + j) * p.ldo + n4,
                                           a[4 * b], a[4 * b + 1], a[4 * b + 2], a[4 * b + 3]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if constexpr (PAIR == 2)  // the leader's MMA reuses the pair's accumulator
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(
                                     mapa_rank(smem_u32(&tempty[acc]), 0))
                                 : "memory");
                else
                    mbar_arrive(&tempty[acc]);
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
            if (p.fuse.kind != CK_FUSE_NONE && (!p.hybrid || tail)) {
                // tile ticket: K-blocks finished so far; the CTA that completes the tile
                // finalizes it (its own partial is made visible first)
                __threadfence();
                epi_bar();
                const int t = (warp - 2) * 32 + lane;  // 0..127
                int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
                if (t == 0) {
                    const int tile = nt * p.m_tiles + mt;
                    const int done = atomicAdd(&p.fuse.tickets[tile], kb1 - kb0) + (kb1 - kb0);
                    *s_last = done == p.kb_total;
                    if (done == p.kb_total) p.fuse.tickets[tile] = 0;
                }
                epi_bar();
                if (*s_last) {
                    __threadfence();
                    finalize_tile(p, nt, mt, BN, t);
                }
                epi_bar();
            }
        }
        if (warp == 2 && lane == 0) probe_stamp(p, 4);
    }

    tc_fence_before();
    if constexpr (PAIR == 2)
        cluster_sync_all();  // the peer's epilogue has drained; no MMA writes either TMEM any more
    else
        __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_g<PAIR>(tmem_base, C::kTmemCols);
    }
}

// ------------------------------------------------------------------ host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
}

struct MapKey {
    const void* ptr;
    long long rows, cols;
    int box_rows;
    bool operator==(const MapKey& o) const {
        return ptr == o.ptr && rows == o.rows && cols == o.cols && box_rows == o.box_rows;
    }
};
struct MapKeyHash {
    size_t operator()(const MapKey& k) const {
        return std::hash<const void*>()(k.ptr) ^ (std::hash<long long>()(k.rows) * 31) ^
               (std::hash<long long>()(k.cols) * 131) ^ static_cast<size_t>(k.box_rows) * 7919;
    }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// Row-major [rows, cols] bf16 matrix, tile box = 64 columns x box_rows rows, 128B swizzle.
int tensor_map(const void* ptr, long long rows, long long cols, int box_rows, CUtensorMap* out) {
    const MapKey key{ptr, rows, cols, box_rows};
    {
        std::lock_guard<std::mutex> g(g_map_mu);
        auto it = g_maps.find(key);
        if (it != g_maps.end()) {
            *out = it->second;
            return 0;
        }
    }
    EncodeFn enc = encode_fn();
    if (!enc) return static_cast<int>(cudaErrorNotSupported);
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kTileK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return static_cast<int>(cudaErrorInvalidValue);
    std::lock_guard<std::mutex> g(g_map_mu);
    if (g_maps.size() > 65536) g_maps.clear();
    g_maps.emplace(key, *out);
    return 0;
}

int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

template <int BN, int PAIR = 1>
int launch(const CUtensorMap& mw, const CUtensorMap& mx, GemmParams p, int max_ctas, cudaStream_t s) {
    using C = Cfg<BN, PAIR>;
    static unsigned attr_set_mask = 0;  // per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set_mask & (1u << dev))) {
        cudaError_t e =
            cudaFuncSetAttribute(gemm_tc_kernel<BN, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return static_cast<int>(e);
        attr_set_mask |= 1u << dev;
    }
    static const int ring_kb = [] {
        const char* e = std::getenv("CRONUS_GEMM_RING_KB");
        return e ? std::atoi(e) : -1;
    }();
    p.stages = C::kStages;
    p.pair = PAIR;
    const int kb = ring_kb >= 0 ? ring_kb : (BN <= 32 ? 100 : 0);
    if (p.stream_k && kb > 0) p.stages = std::clamp(kb * 1024 / C::kStageBytes, 2, C::kStages);
    const int smem = p.stages * C::kStageBytes + 1024 + 256;
    const long long work = p.stream_k ? p.iters : p.hybrid ? (1ll << 40) : p.units;
    // Weight-streaming stream-K grids of small token tiles (BN <= 32, 100 KB rings) run 2 CTAs
    // per SM: ~200 KB of weights in flight per SM instead of ~100 (Little's law against the
    // loaded HBM latency). Measured on the 108-SM CPI partition (tools/scripts/r2_stream2.sh,
    // 1400-key contexts): 3 / 16 / 24 / 32 / 48-decoder passes 3.94 / 4.16 / 4.87 / 4.67 /
    // 6.18 -> 3.58 / 3.86 / 4.56 / 4.33 / 5.57 ms (all 148 SMs: 2-5 %); BN = 128 keeps the full
    // ring with 1 CTA per SM (81 decoders: 6.34 ms vs 6.44 with 2 x 100 KB). BN = 64 would gain
    // too (48 decoders), but its 100-KB ring hung the bench's CUPTI-traced serve (an unexplained
    // interaction with the profiler; plain serves were fine), so it keeps the full ring.
    // CRONUS_GEMM_SK_PER_SM (1 or 2) forces it for every weight-streaming tile size.
    static const int sk_per_sm = [] {
        const char* e = std::getenv("CRONUS_GEMM_SK_PER_SM");
        const int v = e ? std::atoi(e) : 0;
        return v >= 1 && v <= 2 ? v : 0;
    }();
    const int per_sm = !p.stream_k || BN > 128 ? 1 : sk_per_sm ? sk_per_sm : (BN <= 32 && kb == 100 ? 2 : 1);
    const int grid =
        PAIR * static_cast<int>(std::min<long long>(work, per_sm * (max_ctas > 0 ? max_ctas : num_sms()) / PAIR));
    if constexpr (PAIR == 2) {
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_enabled() ? 2 : 1;
        return static_cast<int>(cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, 2>, mw, mx, p));
    } else {
    static const bool probe = [] {
        const char* e = std::getenv("CRONUS_GEMM_PROBE");
        return e && e[0] == '1';
    }();
    if (!probe) return launch_pdl(gemm_tc_kernel<BN, 1>, dim3(grid), dim3(kThreads), smem, s, mw, mx, p);
    // dev: per-CTA timeline (entry, after dependency wait, first stage ready, last MMA
    // issued, epilogue done), printed relative to the earliest CTA entry
    static unsigned long long* buf = nullptr;
    if (!buf) cudaMalloc(&buf, 1024 * 6 * sizeof(unsigned long long));
    cudaMemsetAsync(buf, 0, grid * 6 * sizeof(unsigned long long), s);
    p.probe = buf;
    const int rc = launch_pdl(gemm_tc_kernel<BN, 1>, dim3(grid), dim3(kThreads), smem, s, mw, mx, p);
    std::vector<unsigned long long> h(grid * 6);
    cudaMemcpyAsync(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, h[c * 6]);
    std::fprintf(stderr, "[gemm probe] M=%d N=%d K=%d BN=%d grid=%d sk=%d:", p.M, p.N, p.K, BN, grid, p.stream_k);
    const char* names[5] = {"entry", "dep_ok", "first_full", "last_mma", "epi_done"};
    for (int k = 0; k < 5; ++k) {
        std::vector<double> v;
        for (int c = 0; c < grid; ++c)
            if (h[c * 6 + k]) v.push_back((h[c * 6 + k] - t0) * 1e-3);
        std::sort(v.begin(), v.end());
        if (!v.empty())
            std::fprintf(stderr, " %s=%.1f/%.1f/%.1f", names[k], v.front(), v[v.size() / 2], v.back());
    }
    std::fprintf(stderr, " us\n");
    return rc;
    }
}

}  // namespace

namespace {
int gemm_impl(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int ldo, int epi,
              int splits, int max_ctas, const ck_gemm_fuse* fuse, void* stream);
}

extern "C" int ck_gemm(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int ldo,
                       int epi, int splits, int max_ctas, void* stream) {
    return gemm_impl(W, X, out, bias, M, N, K, ldo, epi, splits, max_ctas, nullptr, stream);
}

extern "C" int ck_gemm_fused(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int epi,
                             int splits, int max_ctas, const ck_gemm_fuse* fuse, void* stream) {
    if (fuse && fuse->kind != CK_FUSE_NONE && (epi == CK_EPI_BF16 || !fuse->tickets))
        return static_cast<int>(cudaErrorInvalidValue);  // finalize reads the fp32 tile back
    if (fuse && fuse->kind == CK_FUSE_RMSNORM &&
        (epi != CK_EPI_RED_F32 || splits > 0 || !fuse->row_tickets || !fuse->gamma || !fuse->norm_out ||
         N > 4096 || (fuse->zero && fuse->zero_cols % 4)))
        return static_cast<int>(cudaErrorInvalidValue);  // residual stream-K GEMM, rows of <= 4096
    return gemm_impl(W, X, out, bias, M, N, K, 0, epi, splits, max_ctas, fuse, stream);
}

namespace {
// CRONUS_GEMM_PAIR=0: tensor-regime GEMMs on single CTAs (the round-1 kernel) instead of CTA pairs
bool gemm_pair() {
    static const bool on = [] {
        const char* e = std::getenv("CRONUS_GEMM_PAIR");
        return !(e && e[0] == '0');
    }();
    return on;
}

int gemm_impl(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int ldo, int epi,
              int splits, int max_ctas, const ck_gemm_fuse* fuse, void* stream) {
    if (M <= 0) return 0;
    if (N % kTileN != 0 || K % kTileK != 0 || N <= 0 || K <= 0) return static_cast<int>(cudaErrorInvalidValue);
    if ((reinterpret_cast<uintptr_t>(W) | reinterpret_cast<uintptr_t>(X)) & 15) return static_cast<int>(cudaErrorMisalignedAddress);
    if (epi < CK_EPI_BF16 || epi > CK_EPI_SILU_BF16) return static_cast<int>(cudaErrorInvalidValue);
    // SiLU epilogue: splits 1 = whole tiles into `out`; splits 0 with a CK_FUSE_SILU fuse =
    // hybrid (whole tiles into fuse->act, a sparse last wave as stream-K pieces through the
    // zeroed fp32 accumulator `out` [M, N] + ticketed finalize)
    const bool silu_hybrid = epi == CK_EPI_SILU_BF16 && splits <= 0 && fuse && fuse->kind == CK_FUSE_SILU;
    if (epi == CK_EPI_SILU_BF16 && ((splits != 1 && !silu_hybrid) || bias != nullptr))
        return static_cast<int>(cudaErrorInvalidValue);
    const int BN = M <= 16 ? 16 : M <= 32 ? 32 : M <= 64 ? 64 : M <= 128 ? 128 : 256;
    // tensor regime: CTA pairs (cta_group::2, 256 weight rows per tile) unless disabled
    const int PAIR = BN == 256 && N % (2 * kTileN) == 0 && gemm_pair() && !(fuse && fuse->kind == CK_FUSE_RMSNORM) ? 2 : 1;
    GemmParams p{};
    p.out = out;
    p.bias = static_cast<const __nv_bfloat16*>(bias);
    p.M = M;
    p.N = N;
    p.K = K;
    p.ldo = ldo > 0 ? ldo : (epi == CK_EPI_SILU_BF16 ? N / 2 : N);
    p.epi = epi;
    p.fuse = fuse ? *fuse : ck_gemm_fuse{};
    p.m_tiles = (M + BN - 1) / BN;
    p.kb_total = K / kTileK;
    const int tiles = (N / (kTileN * PAIR)) * p.m_tiles;  // (pair) tiles
    p.stream_k = 0;
    p.iters = static_cast<long long>(tiles) * p.kb_total;
    if (splits <= 0 && epi == CK_EPI_RED_F32) {
        // Partial sums meet through red.add, so balance K-block iterations exactly
        // across the persistent grid (stream-K) instead of quantizing to whole tiles.
        p.stream_k = 1;
        splits = 1;
    } else if (splits <= 0) {
        splits = 1;
    }
    if (splits > 1 && epi != CK_EPI_RED_F32) return static_cast<int>(cudaErrorInvalidValue);
    splits = std::min(splits, p.kb_total);
    p.kb_per_split = (p.kb_total + splits - 1) / splits;
    p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;  // no empty splits
    p.units = tiles * p.splits;
    if (silu_hybrid) {
        const int ctas = (max_ctas > 0 ? max_ctas : num_sms()) / PAIR;  // unit CTAs (pairs)
        const int tail = tiles % ctas;
        p.dp_tiles = tiles - tail;
        if (tail == 0 || p.dp_tiles == 0 || tail * 2 >= ctas) {  // last wave >= half full: keep it
            // whole tiles fill the waves well enough: plain SiLU epilogue into act
            p.out = fuse->act;
            p.ldo = N / 2;
            p.fuse = ck_gemm_fuse{};
        } else {
            p.hybrid = 1;
            p.ldo = N;  // the fp32 accumulator the tail pieces meet in
            p.tail_iters = static_cast<long long>(tail) * p.kb_total;
            // pieces of >= 16 K-blocks (fewer partial tiles to reduce), at most one per CTA
            p.kb_piece = static_cast<int>(std::max<long long>(16, (p.tail_iters + ctas - 1) / ctas));
        }
    }

    CUtensorMap mw, mx;
    int rc = tensor_map(W, N, K, kTileN, &mw);
    if (rc) return rc;
    rc = tensor_map(X, M, K, BN / PAIR, &mx);
    if (rc) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (PAIR == 2) return launch<256, 2>(mw, mx, p, max_ctas, s);
    switch (BN) {
        case 16: return launch<16>(mw, mx, p, max_ctas, s);
        case 32: return launch<32>(mw, mx, p, max_ctas, s);
        case 64: return launch<64>(mw, mx, p, max_ctas, s);
        case 128: return launch<128>(mw, mx, p, max_ctas, s);
        default: return launch<256>(mw, mx, p, max_ctas, s);
    }
}
}  // namespace
