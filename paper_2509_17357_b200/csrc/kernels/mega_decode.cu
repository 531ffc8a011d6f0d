// Persistent decode forward: one launch runs a whole decode-only CPI iteration
// (embedding -> L x [norm, QKV, RoPE+append, attention, O, norm, gate_up, SiLU, down]
// -> final norm -> LM head -> greedy argmax) for M <= 64 decode rows.
//
// Why: at small M every projection is a weight stream (15 GB per forward for
// LLaMA3-8B). As ~290 separate kernels each stream pays a launch/ramp/drain
// (~3-7 us) and HBM idles across every boundary. Here the weight stream never stops:
// the TMA producer walks the 4L+1 GEMMs' weight tiles back to back through one smem
// ring — prefetching the next GEMM's weights while the other warps run the
// norm / RoPE / attention phases — and only the activation tiles wait for the grid
// barrier that publishes them.
//
// Roles (192 threads, one CTA per SM of the CPI partition, co-resident):
//   warp 0      TMA producer (weights first, activations once their phase barrier passed)
//   warp 1      tcgen05 MMA issuer (accumulators double-buffered in TMEM)
//   warps 2..5  "general" warps: GEMM epilogue (red.add.v4 into fp32 accumulators) in GEMM
//               phases, and every non-GEMM phase, separated by grid barriers
// Grid barrier = monotonic counter (zeroed by the host before launch) + acquire spin.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "cronus_ck.h"
#include "decode_attn.cuh"

namespace {

using namespace ck;

constexpr int kThreads = 192;
constexpr int kTileN = 128, kTileK = 64;
constexpr int kAttnStages = 4;
constexpr int kAttnBytes = kDTileBytes /*Q*/ + 4 * kAttnStages * 2 * kDTileBytes;  // 132 KiB, aliases the ring
constexpr int kSmemBudget = 227 * 1024;

struct MegaParams {
    int M, H, NQKV, NQ, F, V, nq, nkv, L, G;  // G = grid size (CTAs)
    float eps, qk_scale_log2;
    // activations / accumulators
    float* x;
    __nv_bfloat16* h;
    float* qkv;
    __nv_bfloat16* q;
    __nv_bfloat16* attn;
    float* gu;
    __nv_bfloat16* act;
    __nv_bfloat16* hs;
    float* logits;
    // weights
    const CUtensorMap* tm_w;  // [4L + 1]: per layer qkv, o, gu, d; then lm_head
    const CUtensorMap* tm_x;  // [4]: h (K=H), attn (K=NQ), act (K=F), hs (K=H), rows = M
    const __nv_bfloat16* const* wptr;  // [4L + 1] raw weight pointers (L2 prefetch)
    int l2pf_kb;                       // per-CTA L2 prefetch of the next GEMM's weights (KiB)
    const __nv_bfloat16* embed;
    const __nv_bfloat16* const* attn_norm;  // [L]
    const __nv_bfloat16* const* ffn_norm;   // [L]
    const __nv_bfloat16* const* bqkv;       // [L] (entries may be null)
    const __nv_bfloat16* final_norm;
    const float* cos_tab;
    const float* sin_tab;
    // per-pass metadata (decode rows only: row r is decode sequence r)
    const int* row_rid;
    const int* row_pos;
    const int* bt;
    const int* d_row;
    const int* d_len;
    const int* d_bt;
    const int* d_item0;
    const int* d_work;
    int n_work, blocks_per_split;
    float* attn_ws;
    int* attn_tickets;
    __nv_bfloat16* pool;
    // sampling
    const long long* s_out;
    int* last_tok;
    int* out_tok;
    float* arg_ws;
    int* arg_tickets;
    unsigned* gbar;
    int pf_tiles;                // L2 prefetch lookahead of the weight stream (tiles per CTA)
    unsigned long long* trace;   // optional: CTA 0's barrier completion times (globaltimer)
};

template <int BN>
struct MegaCfg {
    static constexpr int kABytes = kTileN * kTileK * 2;
    static constexpr int kBBytes = BN * kTileK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    // the attention phase borrows the ring (the producer keeps it empty from the QKV
    // GEMM's end until the attention barrier; the O weights wait in L2 meanwhile)
    static constexpr int kStages = (kSmemBudget - 2048) / kStageBytes;
    static_assert(kStages * kStageBytes >= kAttnBytes, "attention scratch must fit in the ring");
    static constexpr int kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 1024;
};

// ---------------------------------------------------------------- GEMM sequence
struct GemmInfo {
    const CUtensorMap* w;
    const CUtensorMap* x;
    float* out;
    const __nv_bfloat16* bias;
    int N, K, stream_k;
    unsigned x_ready;  // barrier count (x G) after which the activation rows are published
};

__device__ __forceinline__ GemmInfo gemm_info(const MegaParams& p, int g) {
    GemmInfo gi;
    const int L = p.L;
    if (g < 4 * L) {
        const int l = g >> 2, kind = g & 3;
        const unsigned base = 1 + 9u * l;
        gi.w = p.tm_w + g;
        gi.stream_k = 1;
        gi.bias = nullptr;
        if (kind == 0) {
            gi.x = p.tm_x + 0, gi.out = p.qkv, gi.N = p.NQKV, gi.K = p.H, gi.x_ready = base + 1, gi.bias = p.bqkv[l];
        } else if (kind == 1) {
            gi.x = p.tm_x + 1, gi.out = p.x, gi.N = p.H, gi.K = p.NQ, gi.x_ready = base + 4;
        } else if (kind == 2) {
            gi.x = p.tm_x + 0, gi.out = p.gu, gi.N = 2 * p.F, gi.K = p.H, gi.x_ready = base + 6;
        } else {
            gi.x = p.tm_x + 2, gi.out = p.x, gi.N = p.H, gi.K = p.F, gi.x_ready = base + 8;
        }
    } else {  // LM head: plain fp32 tile stores
        gi.w = p.tm_w + 4 * L, gi.x = p.tm_x + 3, gi.out = p.logits, gi.N = p.V, gi.K = p.H, gi.stream_k = 0;
        gi.bias = nullptr;
        gi.x_ready = 1 + 9u * L + 1;
    }
    return gi;
}

// Units of GEMM g owned by this CTA: stream-K ranges (stream_k) or whole tiles.
struct UnitIt {
    long long pos, end;
    int kb_total, tiles;
    bool sk;
};
__device__ __forceinline__ UnitIt units_begin(const GemmInfo& gi, int G) {
    UnitIt u;
    u.kb_total = gi.K / kTileK;
    u.tiles = gi.N / kTileN;  // single m tile (M <= BN)
    u.sk = gi.stream_k;
    if (u.sk) {
        const long long iters = static_cast<long long>(u.tiles) * u.kb_total;
        u.pos = (static_cast<long long>(blockIdx.x) * iters) / G;
        u.end = (static_cast<long long>(blockIdx.x + 1) * iters) / G;
    } else {
        u.pos = blockIdx.x;
        u.end = u.tiles;
    }
    return u;
}
__device__ __forceinline__ bool units_next(UnitIt& u, int G, int& nt, int& kb0, int& kb1) {
    if (u.sk) {
        if (u.pos >= u.end) return false;
        nt = static_cast<int>(u.pos / u.kb_total);
        kb0 = static_cast<int>(u.pos - static_cast<long long>(nt) * u.kb_total);
        kb1 = static_cast<int>(min(static_cast<long long>(u.kb_total), kb0 + (u.end - u.pos)));
        u.pos += kb1 - kb0;
        return true;
    }
    if (u.pos >= u.end) return false;
    nt = static_cast<int>(u.pos);
    kb0 = 0;
    kb1 = u.kb_total;
    u.pos += G;
    return true;
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* m, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(m), "r"(c0), "r"(c1) : "memory");
}

// Walks the weight tiles of the whole GEMM sequence in the producer's load order.
struct TileCursor {
    int g, n_gemm, nt, kb, kb1;
    bool valid;
    GemmInfo gi;
    UnitIt it;
    __device__ __forceinline__ void start(const MegaParams& p, int n) {
        g = -1, n_gemm = n, valid = true;
        next_unit(p);
    }
    __device__ __forceinline__ void next_unit(const MegaParams& p);
    __device__ __forceinline__ void advance(const MegaParams& p) {
        if (++kb >= kb1) next_unit(p);
    }
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void TileCursor::next_unit(const MegaParams& p) {
    while (true) {
        if (g >= 0 && units_next(it, p.G, nt, kb, kb1)) return;
        if (++g >= n_gemm) {
            valid = false;
            return;
        }
        gi = gemm_info(p, g);
        it = units_begin(gi, p.G);
    }
}

__device__ __forceinline__ void wait_count(const unsigned* ctr, unsigned target) {
    uint32_t spins = 0;
    while (ld_acquire(ctr) < target) {
        if (++spins == (1u << 28)) {
            printf("[cronus watchdog] mega grid barrier stuck: block %d waits %u\n", blockIdx.x, target);
            __trap();
        }
    }
}

// ---------------------------------------------------------------- general phases
constexpr int kGenBar = 2;  // named barrier id for the 4 general warps

__device__ __forceinline__ void grid_barrier(const MegaParams& p, unsigned& k, int t) {
    __threadfence();
    group_bar(kGenBar);
    ++k;
    if (t == 0) {
        atomicAdd(p.gbar, 1u);
        wait_count(p.gbar, k * p.G);
        if (p.trace != nullptr && blockIdx.x == 0) p.trace[k] = globaltimer();
    }
    group_bar(kGenBar);
}

__device__ void phase_embed(const MegaParams& p, int t) {
    for (int r = blockIdx.x; r < p.M; r += p.G) {
        const int tok = p.last_tok[p.row_rid[r]];
        const uint4* src = reinterpret_cast<const uint4*>(p.embed + static_cast<size_t>(tok) * p.H);
        float4* dst = reinterpret_cast<float4*>(p.x + static_cast<size_t>(r) * p.H);
        for (int i = t; i < p.H / 8; i += 128) {
            const uint4 v = src[i];
            const float2 a = unpack_bf16x2(v.x), b = unpack_bf16x2(v.y), c = unpack_bf16x2(v.z), d = unpack_bf16x2(v.w);
            dst[2 * i] = make_float4(a.x, a.y, b.x, b.y);
            dst[2 * i + 1] = make_float4(c.x, c.y, d.x, d.y);
        }
    }
}

__device__ void phase_norm(const MegaParams& p, const __nv_bfloat16* gamma, __nv_bfloat16* out, int t, float* red) {
    for (int r = blockIdx.x; r < p.M; r += p.G) {
        const float4* xr = reinterpret_cast<const float4*>(p.x + static_cast<size_t>(r) * p.H);
        float ss = 0.f;
        for (int i = t; i < p.H / 4; i += 128) {
            const float4 v = __ldcg(xr + i);
            ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
        }
        ss = warp_sum(ss);
        if ((t & 31) == 0) red[t >> 5] = ss;
        group_bar(kGenBar);
        const float tot = red[0] + red[1] + red[2] + red[3];
        group_bar(kGenBar);
        const float inv = rsqrtf(tot / static_cast<float>(p.H) + p.eps);
        const uint2* g = reinterpret_cast<const uint2*>(gamma);
        uint2* o = reinterpret_cast<uint2*>(out + static_cast<size_t>(r) * p.H);
        for (int i = t; i < p.H / 4; i += 128) {
            const float4 v = __ldcg(xr + i);
            const uint2 gg = g[i];
            const float2 g0 = unpack_bf16x2(gg.x), g1 = unpack_bf16x2(gg.y);
            o[i] = make_uint2(pack_bf16x2(v.x * inv * g0.x, v.y * inv * g0.y), pack_bf16x2(v.z * inv * g1.x, v.w * inv * g1.y));
        }
    }
}

// RoPE + KV append for (row, head) items, one warp each; clears the qkv rows read.
__device__ void phase_rope(const MegaParams& p, int l, int t) {
    const int nh = p.nq + 2 * p.nkv;
    const int warp = t >> 5, lane = t & 31;
    const size_t hs = 16 * 128;
    for (int it = blockIdx.x * 4 + warp; it < p.M * nh; it += p.G * 4) {
        const int m = it / nh, h = it % nh;
        float* row = p.qkv + static_cast<size_t>(m) * p.NQKV + h * 128;
        const int pos = p.row_pos[m];
        if (h < p.nq + p.nkv) {
            __nv_bfloat16* dst;
            if (h < p.nq) {
                dst = p.q + static_cast<size_t>(m) * p.NQ + h * 128;
            } else {
                const int blk = p.bt[p.d_bt[m] + (pos >> 4)];
                dst = p.pool + ((static_cast<size_t>(blk) * p.L + l) * 2 * p.nkv + (h - p.nq)) * hs + (pos & 15) * 128;
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int i = lane + 32 * k;
                const float a = __ldcg(row + i), b = __ldcg(row + i + 64);
                row[i] = 0.f;
                row[i + 64] = 0.f;
                const float c = p.cos_tab[static_cast<size_t>(pos) * 64 + i], s = p.sin_tab[static_cast<size_t>(pos) * 64 + i];
                dst[i] = f2bf(a * c - b * s);
                dst[i + 64] = f2bf(b * c + a * s);
            }
        } else {
            const int blk = p.bt[p.d_bt[m] + (pos >> 4)];
            __nv_bfloat16* dst = p.pool + ((static_cast<size_t>(blk) * p.L + l) * 2 * p.nkv + p.nkv + (h - p.nq - p.nkv)) * hs +
                                 (pos & 15) * 128;
            const float4 v = __ldcg(reinterpret_cast<const float4*>(row) + lane);
            reinterpret_cast<float4*>(row)[lane] = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<uint2*>(dst + 4 * lane) = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
        }
    }
}

__device__ void phase_silu(const MegaParams& p, int t) {
    const long long n4 = static_cast<long long>(p.M) * p.F / 4;
    for (long long i = static_cast<long long>(blockIdx.x) * 128 + t; i < n4; i += static_cast<long long>(p.G) * 128) {
        float4* g = reinterpret_cast<float4*>(p.gu) + 2 * i;
        const float4 a = __ldcg(g), b = __ldcg(g + 1);
        g[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        g[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        const float s0 = a.x / (1.f + __expf(-a.x)) * a.y, s1 = a.z / (1.f + __expf(-a.z)) * a.w;
        const float s2 = b.x / (1.f + __expf(-b.x)) * b.y, s3 = b.z / (1.f + __expf(-b.z)) * b.w;
        reinterpret_cast<uint2*>(p.act)[i] = make_uint2(pack_bf16x2(s0, s1), pack_bf16x2(s2, s3));
    }
}

template <int G>
__device__ void phase_attn(const MegaParams& p, int l, uint8_t* attn_smem, float* small, int t) {
    const DecodeAttnArgs a{p.q,       p.pool,           p.bt,      p.d_row,        p.d_len, p.d_bt,
                           p.d_item0, p.d_work,         p.blocks_per_split, p.attn_ws, p.attn_tickets,
                           p.attn,    p.nq,             p.nkv,     l,              p.L,     p.qk_scale_log2};
    const int items = p.n_work * p.nkv;
    for (int it = blockIdx.x; it < items; it += p.G)
        decode_attn_item<G, kAttnStages>(a, it / p.nkv, it % p.nkv, attn_smem, attn_smem + kDTileBytes, small, t, kGenBar);
}

// Greedy sampling: (row, slice) items, one warp each; the last warp of a row emits.
constexpr int kArgSlices = 32;
__device__ void phase_argmax(const MegaParams& p, int t) {
    const int warp = t >> 5, lane = t & 31;
    const int n4 = p.V / 4;
    for (int it = blockIdx.x * 4 + warp; it < p.M * kArgSlices; it += p.G * 4) {
        const int r = it / kArgSlices, c = it % kArgSlices;
        const int lo = static_cast<int>(static_cast<long long>(c) * n4 / kArgSlices);
        const int hi = static_cast<int>(static_cast<long long>(c + 1) * n4 / kArgSlices);
        const float4* row = reinterpret_cast<const float4*>(p.logits + static_cast<size_t>(r) * p.V);
        float best = -INFINITY;
        int bi = 0x7fffffff;
        auto better = [&](float v, int i) {
            if (v > best || (v == best && i < bi)) {
                best = v;
                bi = i;
            }
        };
        for (int v = lo + lane; v < hi; v += 32) {
            const float4 x = __ldcg(row + v);
            better(x.x, 4 * v);
            better(x.y, 4 * v + 1);
            better(x.z, 4 * v + 2);
            better(x.w, 4 * v + 3);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            better(ov, oi);
        }
        int last = 0;
        if (lane == 0) {
            p.arg_ws[r * kArgSlices + c] = best;
            reinterpret_cast<int*>(p.arg_ws + p.M * kArgSlices)[r * kArgSlices + c] = bi;
            __threadfence();
            last = atomicAdd(&p.arg_tickets[r], 1) == kArgSlices - 1;
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last && lane == 0) {
            __threadfence();
            float fb = -INFINITY;
            int fi = 0x7fffffff;
            const int* pi = reinterpret_cast<const int*>(p.arg_ws + p.M * kArgSlices);
            for (int i = 0; i < kArgSlices; ++i) {
                const float v = __ldcg(p.arg_ws + r * kArgSlices + i);
                const int ix = __ldcg(pi + r * kArgSlices + i);
                if (v > fb || (v == fb && ix < fi)) {
                    fb = v;
                    fi = ix;
                }
            }
            p.arg_tickets[r] = 0;
            p.last_tok[p.row_rid[r]] = fi;
            p.out_tok[p.s_out[r]] = fi;
        }
    }
}

// ---------------------------------------------------------------- the kernel
template <int BN, int GQA>
__global__ void __launch_bounds__(kThreads, 1) mega_decode_kernel(const MegaParams p) {
    using C = MegaCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::kStages * C::kABytes;
    uint8_t* sAttn = smem;  // aliases the ring during the attention phase
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty = full + C::kStages;
    uint64_t* tfull = empty + C::kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    float* small = reinterpret_cast<float*>(tmem_slot + 4);  // 2*64 + 4 floats
    float* red = small + 140;

    const int warp = warp_id(), lane = lane_id();
    if (warp == 0) {
        tmem_alloc(tmem_slot, C::kTmemCols);
        tmem_relinquish();
    } else if (warp == 1 && lane == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int n_gemm = 4 * p.L + 1;

    if (warp == 0) {
        // -------------------------------------------------------- producer
        if (lane == 0) {
            const uint64_t keep = policy_evict_last(), stream = policy_evict_first();
            int stage = 0;
            uint32_t phase = 0;
            // L2 prefetch runs pf_tiles weight tiles ahead of the loads, across GEMM
            // boundaries: HBM keeps streaming while the ring waits on a phase barrier
            TileCursor pf;
            pf.start(p, n_gemm);
            long long n_pf = 0, n_ld = 0;
            auto pump = [&]() {
                if (n_pf < n_ld) {  // lookahead 0 (or a lagging cursor): skip what is loaded
                    while (pf.valid && n_pf < n_ld) {
                        pf.advance(p);
                        ++n_pf;
                    }
                }
                while (pf.valid && n_pf < n_ld + p.pf_tiles) {
                    tma_prefetch_l2(pf.gi.w, pf.kb * kTileK, pf.nt * kTileN);
                    pf.advance(p);
                    ++n_pf;
                }
            };
            for (int g = 0; g < n_gemm; ++g) {
                const GemmInfo gi = gemm_info(p, g);
                UnitIt it = units_begin(gi, p.G);
                // weights of this GEMM start streaming as soon as ring slots free up;
                // activation tiles only after the phase that writes them has published
                int pend_stage[C::kStages], pend_kb[C::kStages];
                int n_pend = 0;
                bool x_ok = false;
                auto release = [&]() {
                    pump();
                    wait_count(p.gbar, gi.x_ready * p.G);
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    for (int i = 0; i < n_pend; ++i)
                        tma_load_2d_hint(sB + pend_stage[i] * C::kBBytes, gi.x, &full[pend_stage[i]],
                                         pend_kb[i] * kTileK, 0, keep);
                    n_pend = 0;
                    x_ok = true;
                };
                // O projection: the ring is the attention phase's scratch until its barrier
                if (g < 4 * p.L && (g & 3) == 1) release();
                int nt, kb0, kb1;
                while (units_next(it, p.G, nt, kb0, kb1)) {
                    for (int kb = kb0; kb < kb1; ++kb) {
                        // every ring slot holds weights waiting for activations: the next
                        // empty slot needs one of them consumed, so wait for the phase now
                        if (!x_ok &&
                            (n_pend == C::kStages || ld_acquire(p.gbar) >= gi.x_ready * static_cast<unsigned>(p.G)))
                            release();
                        pump();
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
                        tma_load_2d_hint(sA + stage * C::kABytes, gi.w, &full[stage], kb * kTileK, nt * kTileN, stream);
                        ++n_ld;
                        if (x_ok) {
                            tma_load_2d_hint(sB + stage * C::kBBytes, gi.x, &full[stage], kb * kTileK, 0, keep);
                        } else {
                            pend_stage[n_pend] = stage;
                            pend_kb[n_pend] = kb;
                            ++n_pend;
                        }
                        if (++stage == C::kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                if (!x_ok && n_pend > 0) release();
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(kTileN, BN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int g = 0; g < n_gemm; ++g) {
                const GemmInfo gi = gemm_info(p, g);
                UnitIt it = units_begin(gi, p.G);
                int nt, kb0, kb1;
                while (units_next(it, p.G, nt, kb0, kb1)) {
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * BN;
                    for (int kb = kb0; kb < kb1; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + stage * C::kABytes), b0 = smem_u32(sB + stage * C::kBBytes);
#pragma unroll
                        for (int k = 0; k < kTileK / 16; ++k)
                            tc_mma_bf16(d_tmem, sdesc_sw128(a0 + k * 32), sdesc_sw128(b0 + k * 32), idesc,
                                        (kb > kb0 || k > 0) ? 1u : 0u);
                        tc_commit(&empty[stage]);
                        if (++stage == C::kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    tc_commit(&tfull[acc]);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
            }
        }
    } else {
        // -------------------------------------------------------- general warps
        const int t = threadIdx.x - 64;  // 0..127
        const int q4 = warp & 3;         // TMEM lane quarter
        unsigned k = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        int g = 0;
        auto epilogue = [&]() {  // this CTA's units of GEMM g -> red.add / store
            if (p.l2pf_kb > 0 && g + 1 < 4 * p.L + 1) {
                // warm L2 with the start of this CTA's share of the next GEMM's weights
                const GemmInfo gn = gemm_info(p, g + 1);
                const char* w = reinterpret_cast<const char*>(p.wptr[g + 1]);
                UnitIt itn = units_begin(gn, p.G);
                long long budget = static_cast<long long>(p.l2pf_kb) * 1024;
                int nt, kb0, kb1;
                while (budget > 0 && units_next(itn, p.G, nt, kb0, kb1)) {
                    const long long seg = static_cast<long long>(kb1 - kb0) * kTileK * 2;
                    const char* row = w + (static_cast<long long>(nt) * kTileN + t) * gn.K * 2 + kb0 * kTileK * 2;
                    for (long long o = 0; o < seg && o < budget / kTileN; o += 128)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(row + o));
                    budget -= seg * kTileN;
                }
            }
            const GemmInfo gi = gemm_info(p, g);
            UnitIt it = units_begin(gi, p.G);
            int nt, kb0, kb1;
            while (units_next(it, p.G, nt, kb0, kb1)) {
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                const int n = nt * kTileN + q4 * 32 + lane;
                const float bias = (gi.bias != nullptr && kb0 == 0) ? bf2f(gi.bias[n]) : 0.f;
#pragma unroll 1
                for (int c = 0; c < BN; c += 16) {
                    if (c >= p.M) break;  // warp-uniform
                    uint32_t v[16];
                    tmem_ld16(tmem_base + (static_cast<uint32_t>(q4 * 32) << 16) + acc * BN + c, v);
                    tmem_ld_wait();
                    const int mlim = min(16, p.M - c);
                    if (!gi.stream_k) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (j < mlim) gi.out[static_cast<size_t>(c + j) * gi.N + n] = __uint_as_float(v[j]) + bias;
                    } else {
                        float a[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) a[j] = __uint_as_float(v[j]) + bias;
                        const int tq = lane & 3;
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            float* r = a + 4 * b;
                            float x0 = __shfl_xor_sync(0xffffffffu, (tq & 1) ? r[0] : r[1], 1);
                            float x1 = __shfl_xor_sync(0xffffffffu, (tq & 1) ? r[2] : r[3], 1);
                            if (tq & 1) {
                                r[0] = x0;
                                r[2] = x1;
                            } else {
                                r[1] = x0;
                                r[3] = x1;
                            }
                            x0 = __shfl_xor_sync(0xffffffffu, (tq & 2) ? r[0] : r[2], 2);
                            x1 = __shfl_xor_sync(0xffffffffu, (tq & 2) ? r[1] : r[3], 2);
                            if (tq & 2) {
                                r[0] = x0;
                                r[1] = x1;
                            } else {
                                r[2] = x0;
                                r[3] = x1;
                            }
                        }
                        const int n4 = nt * kTileN + q4 * 32 + (lane & ~3);
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const int j = 4 * b + tq;
                            if (j < mlim)
                                red_add_v4_f32(gi.out + static_cast<size_t>(c + j) * gi.N + n4, a[4 * b], a[4 * b + 1],
                                               a[4 * b + 2], a[4 * b + 3]);
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
            ++g;
        };

        if (p.trace != nullptr && blockIdx.x == 0 && t == 0) p.trace[0] = globaltimer();
        phase_embed(p, t);
        grid_barrier(p, k, t);
        for (int l = 0; l < p.L; ++l) {
            phase_norm(p, p.attn_norm[l], p.h, t, red);
            grid_barrier(p, k, t);
            epilogue();  // QKV
            grid_barrier(p, k, t);
            phase_rope(p, l, t);
            grid_barrier(p, k, t);
            phase_attn<GQA>(p, l, sAttn, small, t);
            grid_barrier(p, k, t);
            epilogue();  // O (+ residual)
            grid_barrier(p, k, t);
            phase_norm(p, p.ffn_norm[l], p.h, t, red);
            grid_barrier(p, k, t);
            epilogue();  // gate_up
            grid_barrier(p, k, t);
            phase_silu(p, t);
            grid_barrier(p, k, t);
            epilogue();  // down (+ residual)
            grid_barrier(p, k, t);
        }
        phase_norm(p, p.final_norm, p.hs, t, red);
        grid_barrier(p, k, t);
        epilogue();  // LM head
        grid_barrier(p, k, t);
        phase_argmax(p, t);
        if (p.trace != nullptr && blockIdx.x == 0 && t == 0) p.trace[k + 1] = globaltimer();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, C::kTmemCols);
    }
}

// ---------------------------------------------------------------- host
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        return reinterpret_cast<EncodeFn>(f);
    }();
    return fn;
}

int encode(CUtensorMap* m, const void* ptr, long long rows, long long cols, int box_rows) {
    EncodeFn enc = encoder();
    if (!enc) return static_cast<int>(cudaErrorNotSupported);
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
               ? 0
               : static_cast<int>(cudaErrorInvalidValue);
}

template <int BN, int GQA>
int launch_mega(const MegaParams& p, cudaStream_t s) {
    using C = MegaCfg<BN>;
    static unsigned mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(mask & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(mega_decode_kernel<BN, GQA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::kSmem);
        if (e != cudaSuccess) return static_cast<int>(e);
        mask |= 1u << dev;
    }
    // all CTAs must be co-resident (grid barriers): cooperative launch
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, mega_decode_kernel<BN, GQA>, p));
}

}  // namespace

// -------------------------------------------------------------------- C-ABI
struct ck_mega_plan {
    int L;
    CUtensorMap* d_wmaps = nullptr;                    // [4L+1] device
    const void** d_wptr = nullptr;                     // [4L+1] device
    const __nv_bfloat16** d_ptrs = nullptr;           // [3L] device: attn_norm, ffn_norm, bqkv
    std::vector<CUtensorMap*> d_xmaps;                 // per M (1..64): [4] device maps, lazily
    void* x_bufs[4];
    long long x_cols[4];
    unsigned* gbar = nullptr;
    // CRONUS_MEGA_TRACE=1: per-phase durations (CTA 0's view of the barriers), printed at destroy
    unsigned long long* d_trace = nullptr;
    double phase_us[12] = {};
    long long traced = 0;
};

namespace {
int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
const char* kPhaseNames[12] = {"norm1", "qkv", "rope", "attn", "o", "norm2", "gate_up", "silu", "down",
                               "embed", "final_norm+lm", "argmax"};
}  // namespace

extern "C" int ck_mega_plan_create(void** out, int L, const void* const* w_qkv, const void* const* w_o,
                                   const void* const* w_gu, const void* const* w_d, const void* lm_head,
                                   const void* const* attn_norm, const void* const* ffn_norm,
                                   const void* const* bqkv, int H, int NQKV, int NQ, int F, int V, const void* h_buf,
                                   const void* attn_buf, const void* act_buf, const void* hs_buf) {
    auto* pl = new ck_mega_plan{};
    pl->L = L;
    std::vector<CUtensorMap> maps(4 * L + 1);
    for (int l = 0; l < L; ++l) {
        if (encode(&maps[4 * l + 0], w_qkv[l], NQKV, H, kTileN) || encode(&maps[4 * l + 1], w_o[l], H, NQ, kTileN) ||
            encode(&maps[4 * l + 2], w_gu[l], 2LL * F, H, kTileN) || encode(&maps[4 * l + 3], w_d[l], H, F, kTileN)) {
            delete pl;
            return static_cast<int>(cudaErrorInvalidValue);
        }
    }
    if (encode(&maps[4 * L], lm_head, V, H, kTileN)) {
        delete pl;
        return static_cast<int>(cudaErrorInvalidValue);
    }
    std::vector<const void*> wp(4 * L + 1);
    for (int l = 0; l < L; ++l) wp[4 * l] = w_qkv[l], wp[4 * l + 1] = w_o[l], wp[4 * l + 2] = w_gu[l], wp[4 * l + 3] = w_d[l];
    wp[4 * L] = lm_head;
    cudaError_t e = cudaMalloc(&pl->d_wptr, wp.size() * sizeof(void*));
    if (e == cudaSuccess) e = cudaMemcpy(pl->d_wptr, wp.data(), wp.size() * sizeof(void*), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&pl->d_wmaps, maps.size() * sizeof(CUtensorMap));
    if (e == cudaSuccess) e = cudaMemcpy(pl->d_wmaps, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    std::vector<const void*> ptrs(3 * L);
    for (int l = 0; l < L; ++l) {
        ptrs[l] = attn_norm[l];
        ptrs[L + l] = ffn_norm[l];
        ptrs[2 * L + l] = bqkv ? bqkv[l] : nullptr;
    }
    if (e == cudaSuccess) e = cudaMalloc(&pl->d_ptrs, ptrs.size() * sizeof(void*));
    if (e == cudaSuccess) e = cudaMemcpy(pl->d_ptrs, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&pl->gbar, 256);
    pl->x_bufs[0] = const_cast<void*>(h_buf), pl->x_cols[0] = H;
    pl->x_bufs[1] = const_cast<void*>(attn_buf), pl->x_cols[1] = NQ;
    pl->x_bufs[2] = const_cast<void*>(act_buf), pl->x_cols[2] = F;
    pl->x_bufs[3] = const_cast<void*>(hs_buf), pl->x_cols[3] = H;
    pl->d_xmaps.assign(129, nullptr);
    if (e != cudaSuccess) {
        delete pl;
        return static_cast<int>(e);
    }
    *out = pl;
    return 0;
}

extern "C" void ck_mega_plan_destroy(void* plan) {
    auto* pl = static_cast<ck_mega_plan*>(plan);
    if (!pl) return;
    cudaFree(pl->d_wmaps);
    cudaFree(pl->d_wptr);
    cudaFree(pl->d_ptrs);
    cudaFree(pl->gbar);
    if (pl->d_trace) {
        cudaFree(pl->d_trace);
        if (pl->traced > 0) {
            std::fprintf(stderr, "[mega trace] %lld passes, avg us per pass:", pl->traced);
            for (int i = 0; i < 12; ++i) std::fprintf(stderr, " %s=%.1f", kPhaseNames[i], pl->phase_us[i] / pl->traced);
            std::fprintf(stderr, "\n");
        }
    }
    for (CUtensorMap* m : pl->d_xmaps)
        if (m) cudaFree(m);
    delete pl;
}

extern "C" int ck_mega_max_rows(void) { return 64; }

extern "C" int ck_mega_decode(void* plan, const ck_mega_args* a, void* stream) {
    auto* pl = static_cast<ck_mega_plan*>(plan);
    const int M = a->M;
    if (M <= 0 || M > 64) return static_cast<int>(cudaErrorInvalidValue);
    const int BN = M <= 32 ? 32 : 64;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!pl->d_xmaps[M]) {  // activation maps for this row count, built once and never modified
        CUtensorMap xm[4];
        for (int i = 0; i < 4; ++i)
            if (encode(&xm[i], pl->x_bufs[i], M, pl->x_cols[i], BN)) return static_cast<int>(cudaErrorInvalidValue);
        CUtensorMap* d = nullptr;
        cudaError_t e = cudaMalloc(&d, sizeof xm);
        if (e == cudaSuccess) e = cudaMemcpy(d, xm, sizeof xm, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return static_cast<int>(e);
        pl->d_xmaps[M] = d;
    }
    MegaParams p{};
    p.M = M, p.H = a->H, p.NQKV = a->NQKV, p.NQ = a->NQ, p.F = a->F, p.V = a->V, p.nq = a->nq, p.nkv = a->nkv;
    p.L = pl->L, p.G = a->grid, p.eps = a->eps, p.qk_scale_log2 = a->scale * 1.4426950408889634f;
    p.x = a->x, p.h = static_cast<__nv_bfloat16*>(a->h), p.qkv = a->qkv, p.q = static_cast<__nv_bfloat16*>(a->q);
    p.attn = static_cast<__nv_bfloat16*>(a->attn), p.gu = a->gu, p.act = static_cast<__nv_bfloat16*>(a->act);
    p.hs = static_cast<__nv_bfloat16*>(a->hs), p.logits = a->logits;
    p.tm_w = pl->d_wmaps, p.tm_x = pl->d_xmaps[M];
    p.embed = static_cast<const __nv_bfloat16*>(a->embed);
    p.attn_norm = pl->d_ptrs, p.ffn_norm = pl->d_ptrs + pl->L, p.bqkv = pl->d_ptrs + 2 * pl->L;
    p.final_norm = static_cast<const __nv_bfloat16*>(a->final_norm);
    p.cos_tab = a->cos_tab, p.sin_tab = a->sin_tab;
    p.row_rid = a->row_rid, p.row_pos = a->row_pos, p.bt = a->bt, p.d_row = a->d_row, p.d_len = a->d_len, p.d_bt = a->d_bt;
    p.d_item0 = a->d_item0, p.d_work = a->d_work, p.n_work = a->n_work, p.blocks_per_split = a->blocks_per_split;
    p.attn_ws = a->attn_ws, p.attn_tickets = a->attn_tickets, p.pool = static_cast<__nv_bfloat16*>(a->pool);
    p.s_out = a->s_out, p.last_tok = a->last_tok, p.out_tok = a->out_tok, p.arg_ws = a->arg_ws;
    p.arg_tickets = a->arg_tickets, p.gbar = pl->gbar;
    static const int pf_tiles = env_int("CRONUS_MEGA_PF", 0);
    static const bool trace = env_int("CRONUS_MEGA_TRACE", 0) != 0;
    p.pf_tiles = pf_tiles;
    static const int l2pf_kb = env_int("CRONUS_MEGA_L2PF_KB", 0);
    p.l2pf_kb = l2pf_kb;
    p.wptr = reinterpret_cast<const __nv_bfloat16* const*>(pl->d_wptr);
    const int n_trace = 9 * pl->L + 5;
    if (trace && !pl->d_trace) cudaMalloc(&pl->d_trace, n_trace * sizeof(unsigned long long));
    p.trace = trace ? pl->d_trace : nullptr;
    cudaError_t e = cudaMemsetAsync(pl->gbar, 0, 4, s);
    if (e != cudaSuccess) return static_cast<int>(e);
    const int G = a->nq / a->nkv;
    int rc = static_cast<int>(cudaErrorInvalidValue);
#define CK_MEGA(BNV, GV) \
    if (BN == BNV && G == GV) rc = launch_mega<BNV, GV>(p, s);
    CK_MEGA(32, 1) CK_MEGA(32, 2) CK_MEGA(32, 4) CK_MEGA(32, 7) CK_MEGA(32, 8)
    CK_MEGA(64, 1) CK_MEGA(64, 2) CK_MEGA(64, 4) CK_MEGA(64, 7) CK_MEGA(64, 8)
#undef CK_MEGA
    if (rc == 0 && p.trace) {
        std::vector<unsigned long long> t(n_trace);
        cudaMemcpyAsync(t.data(), p.trace, n_trace * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const int L = pl->L;
        pl->phase_us[9] += (t[1] - t[0]) * 1e-3;
        for (int k = 2; k <= 9 * L + 1; ++k) pl->phase_us[(k - 2) % 9] += (t[k] - t[k - 1]) * 1e-3;
        pl->phase_us[10] += (t[9 * L + 3] - t[9 * L + 1]) * 1e-3;
        pl->phase_us[11] += (t[9 * L + 4] - t[9 * L + 3]) * 1e-3;
        pl->traced++;
    }
    return rc;
}
