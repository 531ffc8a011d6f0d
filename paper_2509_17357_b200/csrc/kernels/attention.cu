// Paged attention over the block-major KV pool (see cronus_ck.h for the layout).
//
// Decode (one query token per sequence, HBM bound): split-KV "flash decoding" on
//   mma.sync with a per-warp K/V ring filled by TMA (attn_decode_tma_kernel; the
//   cp.async-ring attn_decode_kernel is kept as ck_attn_decode for comparison). Algorithmic
//   bytes = sum kv_len * 512 B per (layer, kv head) — K and V each read once.
//
// Prefill / chunk (tensor bound): FlashAttention-2 style with mma.sync
//   m16n8k16 bf16 (a CTA = 64 query rows x 1 head; 64-key K/V tiles gathered
//   from paged blocks with cp.async into padded smem, double buffered).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include <cstdlib>

#include <cooperative_groups.h>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "cronus_ck.h"
#include "decode_attn.cuh"

namespace {

using namespace ck;
namespace cg = cooperative_groups;

constexpr float kLog2e = 1.4426950408889634f;
constexpr int kHD = 128;               // head dim
constexpr int kBlk = 16;               // tokens per KV block
constexpr int kTile = kBlk * kHD;      // elements per (block, layer, K|V, head) tile

__device__ __forceinline__ size_t tile_off(int block, int layer, int kv, int head, int n_layers, int nkv) {
    return ((static_cast<size_t>(block) * n_layers + layer) * 2 + kv) * static_cast<size_t>(nkv) * kTile +
           static_cast<size_t>(head) * kTile;
}

// ============================================================== prefill (mma.sync)
constexpr int kPQ = 64;        // query rows per CTA
constexpr int kPK = 64;        // keys per tile
constexpr int kPad = 136;      // padded smem row (bf16 elements): 272 B, conflict-free ldmatrix

// Gather a 64-key K or V tile of (layer, kvh) into padded smem rows.
__device__ __forceinline__ void load_kv_tile(__nv_bfloat16* dst, const __nv_bfloat16* pool, const int* table,
                                             int key0, int n_keys, int layer, int kv, int kvh, int n_layers, int nkv) {
    // 64 keys x 128 dims = 1024 16-byte chunks; 128 threads x 8
    for (int c = threadIdx.x; c < kPK * 16; c += blockDim.x) {
        const int r = c >> 4, col = (c & 15) * 8;
        const int key = key0 + r;
        const bool ok = key < n_keys;
        const int blk = ok ? table[key >> 4] : table[0];
        const __nv_bfloat16* src = pool + tile_off(blk, layer, kv, kvh, n_layers, nkv) + (key & 15) * kHD + col;
        cp_async16(dst + r * kPad + col, src, ok);
    }
}

__global__ void __launch_bounds__(128)
    attn_prefill_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ pool,
                        const int* __restrict__ table, int q_row0, int q_len, int pos0, __nv_bfloat16* __restrict__ out,
                        int nq, int nkv, int layer, int n_layers, float qk_scale_log2) {
    pdl_launch();
    pdl_wait();
    extern __shared__ __align__(16) uint8_t smem_raw[];
    __nv_bfloat16* sQ = reinterpret_cast<__nv_bfloat16*>(smem_raw);
    __nv_bfloat16* sK = sQ + kPQ * kPad;          // [2][64][kPad]
    __nv_bfloat16* sV = sK + 2 * kPK * kPad;      // [2][64][kPad]

    const int qt = blockIdx.x, h = blockIdx.y;
    const int kvh = h / (nq / nkv);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int r_begin = qt * kPQ;
    const int r_end = min(q_len, r_begin + kPQ);
    const int n_keys = pos0 + r_end;  // causal: keys needed by the last row of this tile
    const int n_kt = (n_keys + kPK - 1) / kPK;

    // Q tile
    for (int c = threadIdx.x; c < kPQ * 16; c += blockDim.x) {
        const int r = c >> 4, col = (c & 15) * 8;
        const int row = r_begin + r;
        const bool ok = row < q_len;
        const __nv_bfloat16* src = q + static_cast<size_t>(q_row0 + (ok ? row : r_begin)) * nq * kHD + h * kHD + col;
        cp_async16(sQ + r * kPad + col, src, ok);
    }
    load_kv_tile(sK, pool, table, 0, n_keys, layer, 0, kvh, n_layers, nkv);
    load_kv_tile(sV, pool, table, 0, n_keys, layer, 1, kvh, n_layers, nkv);
    cp_commit();

    uint32_t qf[8][4];
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    const int wrow0 = warp * 16;                      // this warp's first row within the tile
    const int qpos_lo = pos0 + r_begin + wrow0 + g;   // position of row g (row g+8 is +8)

    for (int kt = 0; kt < n_kt; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < n_kt) {
            load_kv_tile(sK + (buf ^ 1) * kPK * kPad, pool, table, (kt + 1) * kPK, n_keys, layer, 0, kvh, n_layers,
                         nkv);
            load_kv_tile(sV + (buf ^ 1) * kPK * kPad, pool, table, (kt + 1) * kPK, n_keys, layer, 1, kvh, n_layers,
                         nkv);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        if (kt == 0) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const __nv_bfloat16* p = sQ + (wrow0 + (lane & 15)) * kPad + kk * 16 + (lane >> 4) * 8;
                ldsm_x4(qf[kk], p);
            }
        }
        const __nv_bfloat16* K = sK + buf * kPK * kPad;
        const __nv_bfloat16* Vt = sV + buf * kPK * kPad;
        // S = Q K^T  (16 x 64 per warp)
        float sc[8][4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) sc[nb][0] = sc[nb][1] = sc[nb][2] = sc[nb][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
            for (int nb = 0; nb < 8; nb += 2) {
                uint32_t b[4];
                const __nv_bfloat16* p =
                    K + (nb * 8 + (lane & 7) + ((lane >> 4) << 3)) * kPad + kk * 16 + ((lane >> 3) & 1) * 8;
                ldsm_x4(b, p);
                mma16816(sc[nb], qf[kk], b[0], b[1]);
                mma16816(sc[nb + 1], qf[kk], b[2], b[3]);
            }
        }
        // scale, causal mask, online softmax (rows g and g+8 of this warp)
        const int key0 = kt * kPK;
        const bool need_mask = key0 + kPK - 1 > qpos_lo;
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float v = sc[nb][e] * qk_scale_log2;
                if (need_mask) {
                    const int key = key0 + nb * 8 + 2 * tq + (e & 1);
                    const int qp = qpos_lo + ((e >> 1) << 3);
                    if (key > qp) v = -INFINITY;
                }
                sc[nb][e] = v;
                mx[e >> 1] = fmaxf(mx[e >> 1], v);
            }
        }
        float corr[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
            mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
            const float mn = fmaxf(mrow[r], mx[r]);
            corr[r] = mn == -INFINITY ? 1.f : exp2f(mrow[r] - mn);
            mrow[r] = mn;
        }
        float rs[2] = {0.f, 0.f};
        uint32_t pf[4][4];
#pragma unroll
        for (int nb = 0; nb < 8; ++nb) {
            float p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float mm = mrow[e >> 1];
                p[e] = mm == -INFINITY ? 0.f : exp2f(sc[nb][e] - mm);
                rs[e >> 1] += p[e];
            }
            const int kk = nb >> 1;
            if ((nb & 1) == 0) {
                pf[kk][0] = pack_bf16x2(p[0], p[1]);
                pf[kk][1] = pack_bf16x2(p[2], p[3]);
            } else {
                pf[kk][2] = pack_bf16x2(p[0], p[1]);
                pf[kk][3] = pack_bf16x2(p[2], p[3]);
            }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
            rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
            lrow[r] = lrow[r] * corr[r] + rs[r];
        }
#pragma unroll
        for (int nd = 0; nd < 16; ++nd) {
            o[nd][0] *= corr[0];
            o[nd][1] *= corr[0];
            o[nd][2] *= corr[1];
            o[nd][3] *= corr[1];
        }
        // O += P V
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
            for (int nd = 0; nd < 16; nd += 2) {
                uint32_t b[4];
                const __nv_bfloat16* p =
                    Vt + (kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * kPad + nd * 8 + (lane >> 4) * 8;
                ldsm_x4_t(b, p);
                mma16816(o[nd], pf[kk], b[0], b[1]);
                mma16816(o[nd + 1], pf[kk], b[2], b[3]);
            }
        }
        __syncthreads();
    }
    // normalize and store
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int row = r_begin + wrow0 + g + r * 8;
        if (row >= q_len) continue;
        const float inv = lrow[r] > 0.f ? 1.f / lrow[r] : 0.f;
        __nv_bfloat16* orow = out + static_cast<size_t>(q_row0 + row) * nq * kHD + h * kHD;
#pragma unroll
        for (int nd = 0; nd < 16; ++nd) {
            const int col = nd * 8 + 2 * tq;
            *reinterpret_cast<uint32_t*>(orow + col) = pack_bf16x2(o[nd][2 * r] * inv, o[nd][2 * r + 1] * inv);
        }
    }
}


// ============================================================== decode (split-KV, mma.sync)
// One CTA = 4 warps owns one (sequence, kv head, split) work item. Each warp streams
// every 4th 16-token block of the split through its own cp.async ring (kDecStages
// deep, 128-B XOR-swizzled rows: conflict-free ldmatrix), and computes
//   S[16 x 16] = Qpad[16 x 128] K^T   (G query heads padded to 16 MMA rows)
//   O[16 x 128] += P[16 x 16] V       with an online softmax in registers,
// i.e. 32 mma.sync per 8 KiB of K+V — the tensor pipe is idle most of the time and
// the kernel is bound by HBM, as it should be. The warps merge in smem; the split
// partials are merged by the last CTA of each (sequence, kv head) (atomic ticket),
// so the whole op is one launch.
constexpr int kDecStages = 3;
constexpr int kDecTile = kDTileBytes;

template <int G>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(DecodeAttnArgs a) {
    pdl_launch();
    pdl_wait();
    extern __shared__ __align__(1024) uint8_t dsm[];
    __shared__ float small[2 * 64 + 4];
    decode_attn_item<G, kDecStages>(a, blockIdx.x, blockIdx.y, dsm, dsm + kDecTile, small, threadIdx.x, 1);
}

template <int G>
int launch_decode(const void* q, const void* pool, const int* bt, const int* seq_row, const int* seq_len,
                  const int* seq_bt, const int* seq_item0, const int* work, int n_work, int bps, float* ws,
                  int* tickets, void* out, int nq, int nkv, int layer, int n_layers, float qk, cudaStream_t st) {
    constexpr int smem = kDecTile + 4 * kDecStages * 2 * kDecTile;
    static_assert(4 * kDecStages * 2 * kDecTile >= 4 * 16 * kHD * 4, "merge scratch must fit in the ring");
    static unsigned mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(mask & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(attn_decode_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return static_cast<int>(e);
        mask |= 1u << dev;
    }
    DecodeAttnArgs a{static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(pool), bt, seq_row, seq_len,
                     seq_bt, seq_item0, work, bps, ws, tickets, static_cast<__nv_bfloat16*>(out), nq, nkv, layer,
                     n_layers, qk};
    return launch_pdl(attn_decode_kernel<G>, dim3(n_work, nkv), dim3(128), smem, st, a);
}


// ------------------------------------------------ decode, TMA + cluster variant (default)
// Same math as attn_decode_kernel. Differences:
//  * each warp's K/V ring is filled by TMA: lane 0 issues four 64x16 SWIZZLE_128B boxes
//    (K and V halves, 8 KiB) per block on the slot's mbarrier, STAGES blocks in flight;
//  * a work item (sequence, part) is served by a CLUSTER of C CTAs, each streaming 1/C
//    of the item's blocks; the C partial results meet in rank 0's registers through
//    distributed shared memory (one cluster barrier, no global round trip), so small
//    batches can spread over many SMs without the split-merge tail. Only sequences too
//    long for one cluster are cut into several parts, merged through the ticketed
//    global path of dec_store;
//  * PDL: every block except the sequence's last (the one the previous kernel appends
//    the new token to) is requested before griddepcontrol.wait.
// Requires finite stale slots in partially filled blocks (read, then masked): the
// engine zero-fills its pools at allocation.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

template <int G, int STAGES>
__global__ void __launch_bounds__(128)
    attn_decode_tma_kernel(const __grid_constant__ CUtensorMap tm, DecodeAttnArgs a) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    __shared__ float small[2 * 64 + 4];
    __shared__ __align__(8) uint64_t bars[4][STAGES];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t C = cluster_size(), rank = cluster_rank();
    const int item = blockIdx.x / C, kvh = blockIdx.y;
    // per-pass metadata comes from host copies ordered before the pass: safe pre-wait
    const int wk = a.work[item];
    const int s = wk >> 16, part = wk & 0xffff;
    const int len = a.seq_len[s];
    const int nblk = (len + kDBlk - 1) / kDBlk;
    const int nparts = a.seq_item0[s + 1] - a.seq_item0[s];
    const int bpp = (nblk + nparts - 1) / nparts;  // blocks per part (parts evened out)
    const int p0 = part * bpp, p1 = min(nblk, p0 + bpp);
    const int bpc = (p1 - p0 + static_cast<int>(C) - 1) / static_cast<int>(C);  // blocks per cluster CTA
    const int b0 = min(p1, p0 + static_cast<int>(rank) * bpc), b1 = min(p1, b0 + bpc);
    const int first = b0 + warp;
    const int mine = first < b1 ? (b1 - first + 3) / 4 : 0;
    const int* table = a.bt + a.seq_bt[s];
    uint8_t* sQ = dsm;
    uint8_t* ring_all = dsm + kDTileBytes;
    uint8_t* ring = ring_all + static_cast<size_t>(warp) * STAGES * 2 * kDTileBytes;
    uint64_t* bar = bars[warp];
    const int v_rows = a.nkv * kDBlk;  // pool rows from a head's K tile to its V tile
    int issued = 0;
    auto load = [&](int i) {  // lane 0
        const int row = ((table[first + 4 * i] * a.n_layers + a.layer) * 2 * a.nkv + kvh) * kDBlk;
        uint8_t* dK = ring + (i % STAGES) * 2 * kDTileBytes;
        uint64_t* bb = &bar[i % STAGES];
        mbar_arrive_expect_tx(bb, 2 * kDTileBytes);
        tma_load_2d(dK, &tm, bb, 0, row);
        tma_load_2d(dK + kDTileBytes / 2, &tm, bb, 64, row);
        tma_load_2d(dK + kDTileBytes, &tm, bb, 0, row + v_rows);
        tma_load_2d(dK + kDTileBytes + kDTileBytes / 2, &tm, bb, 64, row + v_rows);
    };
    const int pre = min(mine, STAGES);
    pdl_launch();
    if (lane == 0) {
        tma_prefetch_desc(&tm);
#pragma unroll
        for (int i = 0; i < STAGES; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
        // fused RoPE: no kernel writes the pool before us -> the last block may go early too
        while (issued < pre && (a.qkv || first + 4 * issued != nblk - 1)) load(issued++);
    }
    pdl_wait();
    if (lane == 0)
        while (issued < pre) load(issued++);
    const int pos = len - 1;  // the decode token
    const int qkv_w = (a.nq + 2 * a.nkv) * kDHD;
    if (a.qkv) {  // Q = RoPE(q) from the fp32 accumulator (G heads x 64 rotate-half pairs)
        const float* qrow = a.qkv + static_cast<size_t>(a.seq_row[s]) * qkv_w + static_cast<size_t>(kvh) * G * kDHD;
        const float* cs = a.cos_tab + static_cast<size_t>(pos) * 64;
        const float* sn = a.sin_tab + static_cast<size_t>(pos) * 64;
        for (int c = t; c < 16 * 64; c += 128) {
            const int r = c >> 6, i = c & 63;
            float lo = 0.f, hi = 0.f;
            if (r < G) {
                const float x = qrow[r * kDHD + i], y = qrow[r * kDHD + i + 64];
                lo = x * cs[i] - y * sn[i];
                hi = y * cs[i] + x * sn[i];
            }
            reinterpret_cast<__nv_bfloat16*>(sQ + swz(r, i >> 3))[i & 7] = f2bf(lo);
            reinterpret_cast<__nv_bfloat16*>(sQ + swz(r, 8 + (i >> 3)))[i & 7] = f2bf(hi);
        }
    } else {  // Q (G rows, zero padded to 16) — written by the previous kernel
        const __nv_bfloat16* qrow =
            a.q + static_cast<size_t>(a.seq_row[s]) * a.nq * kDHD + static_cast<size_t>(kvh) * G * kDHD;
        for (int c = t; c < 16 * 16; c += 128) {
            const int r = c >> 4, ch = c & 15;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (r < G) v = *reinterpret_cast<const uint4*>(qrow + r * kDHD + ch * 8);
            *reinterpret_cast<uint4*>(sQ + swz(r, ch)) = v;
        }
    }
    __syncthreads();
    uint32_t qf[8][4];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) ldsm_x4(qf[kk], sQ + swz(lane & 15, 2 * kk + (lane >> 4)));
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    for (int i = 0; i < mine; ++i) {
        mbar_wait(&bar[i % STAGES], (i / STAGES) & 1);
        uint8_t* K = ring + (i % STAGES) * 2 * kDTileBytes;
        if (a.qkv && first + 4 * i == nblk - 1) {
            // the decode token's K (RoPE) / V: computed from the accumulator, written to
            // its pool slot and patched into the staged block (4 dims per lane)
            const float* krow = a.qkv + static_cast<size_t>(a.seq_row[s]) * qkv_w + (a.nq + kvh) * kDHD;
            const float* vrow = krow + a.nkv * kDHD;
            const int d0 = lane * 4, r = pos & 15;
            float kr[4], vr[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int d = d0 + e, ii = d & 63;
                const float x = krow[d], y = krow[d ^ 64];
                const float c = a.cos_tab[static_cast<size_t>(pos) * 64 + ii];
                const float sn = a.sin_tab[static_cast<size_t>(pos) * 64 + ii];
                kr[e] = d < 64 ? x * c - y * sn : x * c + y * sn;
                vr[e] = vrow[d];
            }
            uint2 kp, vp;
            kp.x = pack_bf16x2(kr[0], kr[1]), kp.y = pack_bf16x2(kr[2], kr[3]);
            vp.x = pack_bf16x2(vr[0], vr[1]), vp.y = pack_bf16x2(vr[2], vr[3]);
            const uint32_t off = (d0 >> 6) * 2048 + r * 128 + ((((d0 & 63) >> 3) ^ (r & 7)) << 4) + (d0 & 7) * 2;
            *reinterpret_cast<uint2*>(K + off) = kp;
            *reinterpret_cast<uint2*>(K + kDTileBytes + off) = vp;
            __nv_bfloat16* slot = const_cast<__nv_bfloat16*>(a.pool) +
                                  kv_tile_off(table[nblk - 1], a.layer, 0, kvh, a.n_layers, a.nkv) + r * kDHD + d0;
            *reinterpret_cast<uint2*>(slot) = kp;
            *reinterpret_cast<uint2*>(slot + static_cast<size_t>(a.nkv) * kDTile) = vp;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before TMA refills the slot
            __syncwarp();
        }
        dec_block<SwzTma128>(K, K + kDTileBytes, qf, o, m_run, l_run, (first + 4 * i) * kDBlk, len,
                             a.qk_scale_log2, lane);
        __syncwarp();
        if (lane == 0 && issued < mine) load(issued++);  // refill the slot just consumed
    }
    float* res = reinterpret_cast<float*>(ring_all + kDResOff);
    dec_merge_warps<G>(ring_all, small, o, m_run, l_run, t, 1, res);
    if (C == 1) {
        dec_store<G>(a, item, kvh, res, small, t, 1);
        return;
    }
    // ---- cluster merge over distributed shared memory: CTA r folds the C per-CTA
    // results for its 1/C slice of the G x 128 outputs (3C independent DSMEM loads
    // per element, pipelined), then writes that slice of the output (or the part's
    // partial, whose ticket rank 0 takes once every slice is written).
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();  // every CTA's res is complete
    const int n_el = G * kDHD;
    const int per = (n_el + static_cast<int>(C) - 1) / static_cast<int>(C);
    const int e_end = min(n_el, (static_cast<int>(rank) + 1) * per);
    const int row = a.seq_row[s];
    const bool single = nparts == 1;
    for (int e = static_cast<int>(rank) * per + t; e < e_end; e += 128) {
        const int h = e / kDHD, d = e % kDHD;
        float pm[16], pl[16], pa[16];
#pragma unroll
        for (int r = 0; r < 16; ++r)
            if (r < static_cast<int>(C)) {
                const float* peer = cl.map_shared_rank(res, r);
                pm[r] = peer[h * kDRes];
                pl[r] = peer[h * kDRes + 1];
                pa[r] = peer[h * kDRes + 2 + d];
            }
        float M = -INFINITY;
#pragma unroll
        for (int r = 0; r < 16; ++r)
            if (r < static_cast<int>(C)) M = fmaxf(M, pm[r]);
        float Ls = 0.f, A = 0.f;
#pragma unroll
        for (int r = 0; r < 16; ++r)
            if (r < static_cast<int>(C)) {
                const float f = pm[r] == -INFINITY ? 0.f : exp2f(pm[r] - M);
                Ls += pl[r] * f;
                A += pa[r] * f;
            }
        if (single) {
            a.out[static_cast<size_t>(row) * a.nq * kDHD + (kvh * G + h) * kDHD + d] = f2bf(Ls > 0.f ? A / Ls : 0.f);
        } else {
            float* prt = a.ws + (static_cast<size_t>(item) * a.nq + kvh * G + h) * kDRes;
            prt[2 + d] = A;
            if (d == 0) {
                prt[0] = M;
                prt[1] = Ls;
            }
        }
    }
    if (!single) __threadfence();
    cl.sync();  // peers' shared memory may be released after this; part's partial complete
    if (single || rank != 0) return;
    // several parts of one sequence: the last part to finish merges all partials
    int* s_last = reinterpret_cast<int*>(small + 128);
    if (t == 0) {
        const int prev = atomicAdd(&a.tickets[s * a.nkv + kvh], 1);
        *s_last = prev == nparts - 1;
        if (*s_last) a.tickets[s * a.nkv + kvh] = 0;  // self-resetting
    }
    __syncthreads();
    if (*s_last) {
        __threadfence();
        const int i0 = a.seq_item0[s], i1 = a.seq_item0[s + 1];
        for (int i = t; i < n_el; i += 128) {
            const int h = i / kDHD, d = i % kDHD;
            const int hq = kvh * G + h;
            float M = -INFINITY;
            for (int it = i0; it < i1; ++it) M = fmaxf(M, __ldcg(a.ws + (static_cast<size_t>(it) * a.nq + hq) * kDRes));
            float Ls = 0.f, A = 0.f;
            for (int it = i0; it < i1; ++it) {
                const float* prt = a.ws + (static_cast<size_t>(it) * a.nq + hq) * kDRes;
                const float pmv = __ldcg(prt);
                const float f = pmv == -INFINITY ? 0.f : exp2f(pmv - M);
                Ls += __ldcg(prt + 1) * f;
                A += __ldcg(prt + 2 + d) * f;
            }
            a.out[static_cast<size_t>(row) * a.nq * kDHD + hq * kDHD + d] = f2bf(Ls > 0.f ? A / Ls : 0.f);
        }
    }
}

template <int G, int STAGES>
int launch_decode_tma(const CUtensorMap& tm, const DecodeAttnArgs& a, int n_work, int cluster, cudaStream_t st) {
    constexpr int smem = kDTileBytes + 4 * STAGES * 2 * kDTileBytes;
    static_assert(4 * STAGES * 2 * kDTileBytes >= kDResOff + 8 * kDRes * 4, "merge scratch must fit in the ring");
    static unsigned mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(mask & (1u << dev))) {
        cudaError_t e =
            cudaFuncSetAttribute(attn_decode_tma_kernel<G, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return static_cast<int>(e);
        e = cudaFuncSetAttribute(attn_decode_tma_kernel<G, STAGES>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return static_cast<int>(e);
        mask |= 1u << dev;
    }
    // The largest cluster the stream's SM set can place (a green-context partition may hold
    // fewer SMs per GPC than the whole device); the kernel derives C from the launch, so the
    // plan's cluster size can be clamped here. Cached per stream: keyed by the handle and
    // re-validated by the stream id (handles get reused) whenever the stream is not being
    // captured (stream queries are not capture-safe; a captured pass was first run plainly).
    {
        struct Entry {
            unsigned long long sid;
            int max_c;
        };
        static std::mutex mu;
        static std::unordered_map<cudaStream_t, Entry> max_cluster;
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        unsigned long long sid = 0;
        if (cs == cudaStreamCaptureStatusNone) cudaStreamGetId(st, &sid);
        std::lock_guard<std::mutex> g(mu);
        auto it = max_cluster.find(st);
        if (it != max_cluster.end() && cs == cudaStreamCaptureStatusNone && it->second.sid != sid) {
            max_cluster.erase(it);
            it = max_cluster.end();
        }
        if (it == max_cluster.end()) {
            if (cs != cudaStreamCaptureStatusNone) return static_cast<int>(cudaErrorStreamCaptureUnsupported);
            cudaLaunchConfig_t q{};
            q.gridDim = dim3(16, a.nkv);
            q.blockDim = dim3(128);
            q.dynamicSmemBytes = smem;
            q.stream = st;
            int mc = 0;
            if (cudaOccupancyMaxPotentialClusterSize(&mc, attn_decode_tma_kernel<G, STAGES>, &q) != cudaSuccess ||
                mc < 1) {
                cudaGetLastError();
                mc = 8;  // portable size
            }
            it = max_cluster.emplace(st, Entry{sid, std::min(mc, 16)}).first;
        }
        while (cluster > it->second.max_c) cluster >>= 1;
    }
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_work * cluster, a.nkv);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    // attribute 0 (PDL) is dropped under CRONUS_NO_PDL, like every other launch
    cfg.attrs = pdl_enabled() ? attr : attr + 1;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    return static_cast<int>(cudaLaunchKernelEx(&cfg, attn_decode_tma_kernel<G, STAGES>, tm, a));
}

// Ring depth per warp: CRONUS_DEC_STAGES (2, 3, 4, 6) if set, else chosen per launch (0).
int dec_stages() {
    static const int v = [] {
        const char* e = std::getenv("CRONUS_DEC_STAGES");
        const int x = e ? std::atoi(e) : 0;
        return (x == 2 || x == 3 || x == 4 || x == 6) ? x : 0;
    }();
    return v;
}

// CTAs of the 3-stage kernel (100 KiB each) the stream's SM set holds at once (2 per SM),
// cached per stream like the cluster clamp (queried only outside stream capture; a captured
// pass was first run plainly, so its stream is known; unknown under capture -> 0).
template <int G>
int resident_ctas_3stage(cudaStream_t st) {
    struct Entry {
        unsigned long long sid;
        int ctas;
    };
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, Entry> cache;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    unsigned long long sid = 0;
    if (cs == cudaStreamCaptureStatusNone) cudaStreamGetId(st, &sid);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(st);
    if (it != cache.end() && (cs != cudaStreamCaptureStatusNone || it->second.sid == sid)) return it->second.ctas;
    if (cs != cudaStreamCaptureStatusNone) return 0;
    constexpr int smem = kDTileBytes + 4 * 3 * 2 * kDTileBytes;
    cudaFuncSetAttribute(attn_decode_tma_kernel<G, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 1;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cudaLaunchConfig_t q{};
    q.gridDim = dim3(1, 1);
    q.blockDim = dim3(128);
    q.dynamicSmemBytes = smem;
    q.stream = st;
    q.attrs = &attr;
    q.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, attn_decode_tma_kernel<G, 3>, &q) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[st] = Entry{sid, n};
    return n;
}

// Default ring depth: 3 stages (2 CTAs per SM), or 2 stages (68 KiB, 3 CTAs per SM) when
// that finishes the grid in fewer waves (many sequences x kv heads, e.g. 32 decoders on the
// 108-SM partition: 256 CTAs = 2 waves at 2 per SM, 1 wave at 3 per SM).
// Measured (tools/pass_sweep.py, 108 SMs): 32 x 2048 decode pass 6.26 -> 5.57 ms, 64 x 2048
// 7.70 -> 7.28 ms with 2 stages; 8-16 sequences (grid within 2 per SM) are 2-4 % faster with 3.
template <int G>
int launch_decode_tma_g(const CUtensorMap& tm, const DecodeAttnArgs& a, int n_work, int cluster, cudaStream_t st) {
    int stages = dec_stages();
    if (stages == 0) {
        // 2 stages only where the third CTA per SM saves a wave (48 x 1024: 384 CTAs on 108 SMs
        // is two waves either way, and 3 stages keep more bytes in flight per CTA: 5.68 vs 5.86 ms)
        const long long r3 = resident_ctas_3stage<G>(st), r2 = r3 * 3 / 2;
        const long long ctas = static_cast<long long>(n_work) * cluster * a.nkv;
        stages = r3 > 0 && (ctas + r2 - 1) / r2 < (ctas + r3 - 1) / r3 ? 2 : 3;
    }
    switch (stages) {
        case 2: return launch_decode_tma<G, 2>(tm, a, n_work, cluster, st);
        case 4: return launch_decode_tma<G, 4>(tm, a, n_work, cluster, st);
        case 6: return launch_decode_tma<G, 6>(tm, a, n_work, cluster, st);
        default: return launch_decode_tma<G, 3>(tm, a, n_work, cluster, st);
    }
}

}  // namespace

extern "C" int ck_attn_decode(const void* q, const void* kv_pool, const int* bt, const int* seq_row,
                              const int* seq_len, const int* seq_bt, const int* seq_item0, const int* work,
                              int n_work, int n_seq, int blocks_per_split, float* ws, int* tickets, void* out,
                              int nq, int nkv, int layer, int n_layers, float scale, void* stream) {
    if (n_seq <= 0 || n_work <= 0) return 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const float qk = scale * kLog2e;
    switch (nq / nkv) {
        case 1: return launch_decode<1>(q, kv_pool, bt, seq_row, seq_len, seq_bt, seq_item0, work, n_work, blocks_per_split, ws, tickets, out, nq, nkv, layer, n_layers, qk, st);
        case 2: return launch_decode<2>(q, kv_pool, bt, seq_row, seq_len, seq_bt, seq_item0, work, n_work, blocks_per_split, ws, tickets, out, nq, nkv, layer, n_layers, qk, st);
        case 4: return launch_decode<4>(q, kv_pool, bt, seq_row, seq_len, seq_bt, seq_item0, work, n_work, blocks_per_split, ws, tickets, out, nq, nkv, layer, n_layers, qk, st);
        case 7: return launch_decode<7>(q, kv_pool, bt, seq_row, seq_len, seq_bt, seq_item0, work, n_work, blocks_per_split, ws, tickets, out, nq, nkv, layer, n_layers, qk, st);
        case 8: return launch_decode<8>(q, kv_pool, bt, seq_row, seq_len, seq_bt, seq_item0, work, n_work, blocks_per_split, ws, tickets, out, nq, nkv, layer, n_layers, qk, st);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

extern "C" int ck_attn_decode_tma(const void* q, const void* kv_pool, long long pool_blocks, const int* bt,
                                  const int* seq_row, const int* seq_len, const int* seq_bt, const int* seq_item0,
                                  const int* work, int n_work, int n_seq, int cluster, float* ws, int* tickets,
                                  void* out, int nq, int nkv, int layer, int n_layers, float scale,
                                  const ck_decode_rope* rope, void* stream) {
    if (n_seq <= 0 || n_work <= 0) return 0;
    if (cluster < 1 || cluster > 16) return static_cast<int>(cudaErrorInvalidValue);
    CUtensorMap tm;
    const unsigned long long pool_rows = static_cast<unsigned long long>(pool_blocks) * n_layers * 2 * nkv * kBlk;
    if (pool_rows >= (1ull << 31)) return static_cast<int>(cudaErrorInvalidValue);  // int32 TMA row coordinate
    int rc = make_map_2d(kv_pool, pool_rows, kHD, kBlk, &tm);
    if (rc) return rc;
    const DecodeAttnArgs a{static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(kv_pool), bt,
                           seq_row, seq_len, seq_bt, seq_item0, work, 0, ws, tickets,
                           static_cast<__nv_bfloat16*>(out), nq, nkv, layer, n_layers, scale * kLog2e,
                           rope ? rope->qkv : nullptr, rope ? rope->cos_tab : nullptr, rope ? rope->sin_tab : nullptr};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    switch (nq / nkv) {
        case 1: return launch_decode_tma_g<1>(tm, a, n_work, cluster, st);
        case 2: return launch_decode_tma_g<2>(tm, a, n_work, cluster, st);
        case 4: return launch_decode_tma_g<4>(tm, a, n_work, cluster, st);
        case 7: return launch_decode_tma_g<7>(tm, a, n_work, cluster, st);
        case 8: return launch_decode_tma_g<8>(tm, a, n_work, cluster, st);
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
}

extern "C" int ck_attn_prefill(const void* q, const void* kv_pool, const int* bt, int q_row0, int q_len, int pos0,
                               void* out, int nq, int nkv, int layer, int n_layers, float scale, void* stream) {
    if (q_len <= 0) return 0;
    constexpr int smem = (kPQ + 4 * kPK) * kPad * 2;
    static unsigned attr_mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_mask & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(attn_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return static_cast<int>(e);
        attr_mask |= 1u << dev;
    }
    const dim3 grid((q_len + kPQ - 1) / kPQ, nq);
    return launch_pdl(attn_prefill_kernel, grid, dim3(128), smem, static_cast<cudaStream_t>(stream),
                      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(kv_pool), bt, q_row0,
                      q_len, pos0, static_cast<__nv_bfloat16*>(out), nq, nkv, layer, n_layers, scale * kLog2e);
}
