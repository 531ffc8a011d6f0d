// Paged attention over the block-major KV pool (see cronus_ck.h for the layout).
//
// Decode (one query token per sequence, HBM bound): split-KV "flash decoding" on
//   mma.sync with a per-warp cp.async ring (see attn_decode_kernel). Algorithmic
//   bytes = sum kv_len * 512 B per (layer, kv head) — K and V each read once.
//
// Prefill / chunk (tensor bound): FlashAttention-2 style with mma.sync
//   m16n8k16 bf16 (a CTA = 64 query rows x 1 head; 64-key K/V tiles gathered
//   from paged blocks with cp.async into padded smem, double buffered).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "cronus_ck.h"
#include "decode_attn.cuh"

namespace {

using namespace ck;

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
    pdl_wait();
    pdl_launch();
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
    pdl_wait();
    pdl_launch();
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
