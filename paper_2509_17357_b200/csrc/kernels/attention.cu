// Paged attention over the block-major KV pool (see cronus_ck.h for the layout).
//
// Decode (one query token per sequence, HBM bound): split-KV "flash decoding".
//   A CTA = 4 warps owns one (sequence, kv head, split) work item of up to
//   `blocks_per_split` 16-token blocks; warps stride over the blocks, each warp
//   consuming a whole 16-token block (4 KiB of K + 4 KiB of V, both contiguous)
//   per step for all G query heads of the GQA group, keeping an online softmax in
//   registers. Partials (m, l, acc) are merged across warps in smem and across
//   splits by a combine kernel. Algorithmic bytes = sum kv_len * 512 B per
//   (layer, kv head) — K and V each read exactly once.
//
// Prefill / chunk (tensor bound): FlashAttention-2 style with mma.sync
//   m16n8k16 bf16 (a CTA = 64 query rows x 1 head; 64-key K/V tiles gathered
//   from paged blocks with cp.async into padded smem, double buffered).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "cronus_ck.h"

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

// ============================================================== decode
template <int G>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ pool,
                       const int* __restrict__ bt, const int* __restrict__ seq_row, const int* __restrict__ seq_len,
                       const int* __restrict__ seq_bt, const int* __restrict__ work, int blocks_per_split,
                       float* __restrict__ ws, int nq, int nkv, int layer, int n_layers, float qscale) {
    // q for the group, split into the two 64-dim halves with a 4-float pad so the
    // two half-warps read different banks.
    __shared__ __align__(16) float qs[G][2][68];
    __shared__ __align__(16) float ps[4][G][16];
    __shared__ float wm[4][G], wl[4][G];
    __shared__ __align__(16) float wacc[4][G][kHD];

    const int item = blockIdx.x;
    const int kvh = blockIdx.y;
    const int w = work[item];
    const int s = w >> 16, split = w & 0xffff;
    const int len = seq_len[s];
    const int nblk = (len + kBlk - 1) / kBlk;
    const int b0 = split * blocks_per_split;
    const int b1 = min(nblk, b0 + blocks_per_split);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int* table = bt + seq_bt[s];

    const __nv_bfloat16* qrow = q + static_cast<size_t>(seq_row[s]) * nq * kHD + static_cast<size_t>(kvh) * G * kHD;
    for (int i = threadIdx.x; i < G * kHD; i += blockDim.x) {
        const int h = i / kHD, d = i % kHD;
        qs[h][d >> 6][d & 63] = bf2f(qrow[i]) * qscale;
    }
    __syncthreads();

    float m[G], l[G], acc[G][4];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        m[h] = -INFINITY;
        l[h] = 0.f;
        acc[h][0] = acc[h][1] = acc[h][2] = acc[h][3] = 0.f;
    }
    const int t = lane & 15, half = lane >> 4;

    for (int b = b0 + warp; b < b1; b += 4) {
        const int blk = table[b];
        const __nv_bfloat16* kt = pool + tile_off(blk, layer, 0, kvh, n_layers, nkv);
        const __nv_bfloat16* vt = kt + static_cast<size_t>(nkv) * kTile;
        // ---- loads (K half-row for QK, V 4-dim column slice for PV)
        uint4 kv4[8];
        const uint4* kp = reinterpret_cast<const uint4*>(kt + t * kHD + half * 64);
#pragma unroll
        for (int i = 0; i < 8; ++i) kv4[i] = __ldg(kp + i);
        uint2 vv[16];
        const uint2* vp = reinterpret_cast<const uint2*>(vt) + lane;  // dims 4*lane..4*lane+3
        const int n_valid = min(kBlk, len - b * kBlk);  // slots past the sequence end hold stale data
#pragma unroll
        for (int j = 0; j < 16; ++j) vv[j] = j < n_valid ? __ldg(vp + j * (kHD / 4)) : make_uint2(0u, 0u);

        // ---- scores
        float sc[G];
#pragma unroll
        for (int h = 0; h < G; ++h) sc[h] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float2 k01 = unpack_bf16x2(kv4[i].x), k23 = unpack_bf16x2(kv4[i].y), k45 = unpack_bf16x2(kv4[i].z),
                         k67 = unpack_bf16x2(kv4[i].w);
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const float4 qa = *reinterpret_cast<const float4*>(&qs[h][half][i * 8]);
                const float4 qb = *reinterpret_cast<const float4*>(&qs[h][half][i * 8 + 4]);
                sc[h] += qa.x * k01.x + qa.y * k01.y + qa.z * k23.x + qa.w * k23.y + qb.x * k45.x + qb.y * k45.y +
                         qb.z * k67.x + qb.w * k67.y;
            }
        }
        const bool valid = b * kBlk + t < len;
#pragma unroll
        for (int h = 0; h < G; ++h) {
            sc[h] += __shfl_xor_sync(0xffffffffu, sc[h], 16);
            if (!valid) sc[h] = -INFINITY;
            float mx = sc[h];
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            const float mn = fmaxf(m[h], mx);
            const float p = exp2f(sc[h] - mn);
            float ps_sum = p;
            ps_sum += __shfl_xor_sync(0xffffffffu, ps_sum, 8);
            ps_sum += __shfl_xor_sync(0xffffffffu, ps_sum, 4);
            ps_sum += __shfl_xor_sync(0xffffffffu, ps_sum, 2);
            ps_sum += __shfl_xor_sync(0xffffffffu, ps_sum, 1);
            const float corr = exp2f(m[h] - mn);
            l[h] = l[h] * corr + ps_sum;
            m[h] = mn;
            acc[h][0] *= corr;
            acc[h][1] *= corr;
            acc[h][2] *= corr;
            acc[h][3] *= corr;
            if (half == 0) ps[warp][h][t] = p;
        }
        __syncwarp();
        // ---- P x V
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float2 v01 = unpack_bf16x2(vv[j].x), v23 = unpack_bf16x2(vv[j].y);
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const float p = ps[warp][h][j];
                acc[h][0] += p * v01.x;
                acc[h][1] += p * v01.y;
                acc[h][2] += p * v23.x;
                acc[h][3] += p * v23.y;
            }
        }
        __syncwarp();
    }

    // ---- merge the 4 warps
#pragma unroll
    for (int h = 0; h < G; ++h) {
        if (lane == 0) {
            wm[warp][h] = m[h];
            wl[warp][h] = l[h];
        }
        *reinterpret_cast<float4*>(&wacc[warp][h][lane * 4]) = make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]);
    }
    __syncthreads();
    // partial layout per (item, q head): [m, l, acc[128]]
    for (int i = threadIdx.x; i < G * kHD; i += blockDim.x) {
        const int h = i / kHD, d = i % kHD;
        float M = -INFINITY;
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) M = fmaxf(M, wm[w2][h]);
        float Lsum = 0.f, A = 0.f;
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) {
            const float f = wm[w2][h] == -INFINITY ? 0.f : exp2f(wm[w2][h] - M);
            Lsum += wl[w2][h] * f;
            A += wacc[w2][h][d] * f;
        }
        float* part = ws + (static_cast<size_t>(item) * nq + kvh * G + h) * (kHD + 2);
        part[2 + d] = A;
        if (d == 0) {
            part[0] = M;
            part[1] = Lsum;
        }
    }
}

// out[row(s), h, :] = sum_splits A * 2^(m - M) / sum_splits l * 2^(m - M)
__global__ void attn_decode_combine_kernel(const float* __restrict__ ws, const int* __restrict__ seq_row,
                                           const int* __restrict__ seq_item0, __nv_bfloat16* __restrict__ out,
                                           int nq) {
    const int s = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
    const int i0 = seq_item0[s], i1 = seq_item0[s + 1];
    float M = -INFINITY;
    for (int i = i0; i < i1; ++i) M = fmaxf(M, ws[(static_cast<size_t>(i) * nq + h) * (kHD + 2)]);
    float L = 0.f, A = 0.f;
    for (int i = i0; i < i1; ++i) {
        const float* part = ws + (static_cast<size_t>(i) * nq + h) * (kHD + 2);
        const float f = part[0] == -INFINITY ? 0.f : exp2f(part[0] - M);
        L += part[1] * f;
        A += part[2 + d] * f;
    }
    out[static_cast<size_t>(seq_row[s]) * nq * kHD + h * kHD + d] = f2bf(L > 0.f ? A / L : 0.f);
}

// ============================================================== prefill (mma.sync)
constexpr int kPQ = 64;        // query rows per CTA
constexpr int kPK = 64;        // keys per tile
constexpr int kPad = 136;      // padded smem row (bf16 elements): 272 B, conflict-free ldmatrix

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

template <int G>
int launch_decode(const void* q, const void* pool, const int* bt, const int* seq_row, const int* seq_len,
                  const int* seq_bt, const int* work, int n_work, int bps, float* ws, int nq, int nkv, int layer,
                  int n_layers, float qscale, cudaStream_t s) {
    attn_decode_kernel<G><<<dim3(n_work, nkv), 128, 0, s>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(pool), bt, seq_row, seq_len, seq_bt,
        work, bps, ws, nq, nkv, layer, n_layers, qscale);
    return static_cast<int>(cudaGetLastError());
}

}  // namespace

extern "C" int ck_attn_decode(const void* q, const void* kv_pool, const int* bt, const int* seq_row,
                              const int* seq_len, const int* seq_bt, const int* seq_item0, const int* work,
                              int n_work, int n_seq, int blocks_per_split, float* ws, void* out, int nq, int nkv,
                              int layer, int n_layers, float scale, void* stream) {
    if (n_seq <= 0 || n_work <= 0) return 0;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int G = nq / nkv;
    const float qscale = scale * kLog2e;
    int rc;
    switch (G) {
        case 1: rc = launch_decode<1>(q, kv_pool, bt, seq_row, seq_len, seq_bt, work, n_work, blocks_per_split, ws, nq, nkv, layer, n_layers, qscale, s); break;
        case 2: rc = launch_decode<2>(q, kv_pool, bt, seq_row, seq_len, seq_bt, work, n_work, blocks_per_split, ws, nq, nkv, layer, n_layers, qscale, s); break;
        case 4: rc = launch_decode<4>(q, kv_pool, bt, seq_row, seq_len, seq_bt, work, n_work, blocks_per_split, ws, nq, nkv, layer, n_layers, qscale, s); break;
        case 7: rc = launch_decode<7>(q, kv_pool, bt, seq_row, seq_len, seq_bt, work, n_work, blocks_per_split, ws, nq, nkv, layer, n_layers, qscale, s); break;
        case 8: rc = launch_decode<8>(q, kv_pool, bt, seq_row, seq_len, seq_bt, work, n_work, blocks_per_split, ws, nq, nkv, layer, n_layers, qscale, s); break;
        default: return static_cast<int>(cudaErrorInvalidValue);
    }
    if (rc) return rc;
    attn_decode_combine_kernel<<<dim3(n_seq, nq), kHD, 0, s>>>(ws, seq_row, seq_item0,
                                                               static_cast<__nv_bfloat16*>(out), nq);
    return static_cast<int>(cudaGetLastError());
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
    attn_prefill_kernel<<<grid, 128, smem, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(kv_pool), bt, q_row0, q_len, pos0,
        static_cast<__nv_bfloat16*>(out), nq, nkv, layer, n_layers, scale * kLog2e);
    return static_cast<int>(cudaGetLastError());
}
