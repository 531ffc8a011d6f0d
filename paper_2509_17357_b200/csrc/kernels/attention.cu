// Paged attention over the block-major KV pool (see cronus_ck.h for the layout).
//
// Decode (one query token per sequence, HBM bound): split-KV "flash decoding" on
//   mma.sync with a per-warp K/V ring filled by TMA (attn_decode_tma_kernel). Algorithmic
//   bytes = sum kv_len * 512 B per (layer, kv head) — K and V each read once.
//
// Prefill / chunk attention (tensor bound) lives in attention_tc.cu (tcgen05 + TMEM).
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

// ------------------------------------------------ decode, TMA + cluster
// A CTA = 4 warps serves one (work item, kv head). Each warp streams every 4th 16-token
// block of its share and computes
//   S[16 x 16] = Qpad[16 x 128] K^T   (G query heads padded to 16 MMA rows)
//   O[16 x 128] += P[16 x 16] V       with an online softmax in registers,
// i.e. 32 mma.sync per 8 KiB of K+V: the tensor pipe is idle most of the time and the
// kernel is bound by HBM, as it should be. The warps merge in smem. Furthermore:
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
    // item-major grid (all kv heads of work item 0, then item 1, ...): the planner lists the
    // heaviest items first, so the block scheduler dispatches them first (LPT)
    const int cid = blockIdx.x / C;
    const int item = cid / a.nkv, kvh = cid % a.nkv;
    // per-pass metadata comes from host copies ordered before the pass: safe pre-wait
    const int wk = a.work[item];
    const int s = wk >> 16, part = wk & 0xff;
    const int len = a.seq_len[s];
    const int nblk = (len + kDBlk - 1) / kDBlk;
    const int nparts = (wk >> 8) & 0xff;
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
    // Loads are issued by the whole (convergent) warp, one elected lane inside the PTX: the
    // block id is made provably warp-uniform (shuffle from lane 0) so the TMA operands live in
    // uniform registers (see tc_mma_bf16_warp).
    // The warp's first 32 block ids come in with ONE parallel load (lane j: its block j) instead
    // of one dependent table read per ring stage (measured neutral at 1-128 sequences; kept as
    // the simpler issue path); later blocks read the table directly.
    const int my_id = lane < mine ? table[first + 4 * lane] : 0;
    auto load = [&](int i) {
        const int id = i < 32 ? __shfl_sync(0xffffffffu, my_id, i) : __shfl_sync(0xffffffffu, table[first + 4 * i], 0);
        const int row = ((id * a.n_layers + a.layer) * 2 * a.nkv + kvh) * kDBlk;
        uint8_t* dK = ring + (i % STAGES) * 2 * kDTileBytes;
        uint64_t* bb = &bar[i % STAGES];
        mbar_expect_tx_warp(bb, 2 * kDTileBytes);
        tma_load_2d_warp(dK, &tm, bb, 0, row);
        tma_load_2d_warp(dK + kDTileBytes / 2, &tm, bb, 64, row);
        tma_load_2d_warp(dK + kDTileBytes, &tm, bb, 0, row + v_rows);
        tma_load_2d_warp(dK + kDTileBytes + kDTileBytes / 2, &tm, bb, 64, row + v_rows);
    };
    const int pre = min(mine, STAGES);
    pdl_launch();
    if (lane == 0) {
        tma_prefetch_desc(&tm);
#pragma unroll
        for (int i = 0; i < STAGES; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // fused RoPE: no kernel writes the pool before us -> the last block may go early too
    while (issued < pre && (a.qkv || first + 4 * issued != nblk - 1)) load(issued++);
    pdl_wait();
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
        if (issued < mine) load(issued++);  // refill the slot just consumed
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
        const int i0 = a.seq_item0[s], i1 = i0 + nparts;
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

// The largest cluster the stream's SM set can place (a green-context partition may hold fewer
// SMs per GPC than the whole device); the kernel derives C from the launch, so the plan's
// cluster size can be clamped at launch. Cached per stream: keyed by the handle and re-validated
// by the stream id (handles get reused) whenever the stream is not being captured (stream
// queries are not capture-safe; a captured pass was first run plainly). -1: unknown under capture.
template <int G, int STAGES>
int decode_max_cluster(cudaStream_t st) {
    constexpr int smem = kDTileBytes + 4 * STAGES * 2 * kDTileBytes;
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
        if (cs != cudaStreamCaptureStatusNone) return -1;
        cudaFuncSetAttribute(attn_decode_tma_kernel<G, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(attn_decode_tma_kernel<G, STAGES>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(16, 1);
        q.blockDim = dim3(128);
        q.dynamicSmemBytes = smem;
        q.stream = st;
        int mc = 0;
        if (cudaOccupancyMaxPotentialClusterSize(&mc, attn_decode_tma_kernel<G, STAGES>, &q) != cudaSuccess || mc < 1) {
            cudaGetLastError();
            mc = 8;  // portable size
        }
        it = max_cluster.emplace(st, Entry{sid, std::min(mc, 16)}).first;
    }
    return it->second.max_c;
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
    const int mc = decode_max_cluster<G, STAGES>(st);
    if (mc < 0) return static_cast<int>(cudaErrorStreamCaptureUnsupported);
    while (cluster > mc) cluster >>= 1;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_work * a.nkv * cluster, 1);
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
        // count the grid with the cluster the launch will actually use (clamped to what the
        // stream's SM set can place), as launch_decode_tma does
        const int mc = decode_max_cluster<G, 3>(st);
        int c = cluster;
        while (mc > 0 && c > mc) c >>= 1;
        const long long r3 = resident_ctas_3stage<G>(st), r2 = r3 * 3 / 2;
        const long long ctas = static_cast<long long>(n_work) * c * a.nkv;
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
