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
#include <cstdlib>
#include <vector>
#include <mutex>
#include <cstdio>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "cronus_ck.h"

namespace {

using namespace ck;

constexpr int kKT = 64;          // keys per K/V sub-tile (one S buffer)
constexpr int kQHalf = 16384;    // one 128-row x 64-col bf16 swizzled region (a Q tile half)
constexpr int kQTileBytes = 2 * kQHalf;
constexpr int kKVHalf = kKT * 128;  // one 64-key x 64-dim half of a K/V sub-tile
constexpr int kKVTileBytes = 2 * kKVHalf;
constexpr int kStages = 5;          // K and V ring depth (sub-tiles)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThreshold = 8.0f;  // log2 units


__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t addr) {
    // MN-major, 128B swizzle: LBO = one sub-tile half (8 KiB) between the two 64-element MN
    // (dim) halves, SBO = 1 KiB between 8-row (key) groups.
    return (static_cast<uint64_t>((addr >> 4) & 0x3FFFu)) | (static_cast<uint64_t>(kKVHalf >> 4) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
           (static_cast<uint64_t>(2) << 61);
}

// kind::f16 instruction descriptor, bf16 A/B, fp32 D, M = 128, N = n, A K-major
__host__ __device__ constexpr uint32_t idesc_attn(bool b_mn_major, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
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
// fp32 pairs on sm_100's paired FMA / add datapath (FFMA2 / FADD2)
__device__ __forceinline__ uint64_t f32x2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float lo_f32(uint64_t v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo;
}
__device__ __forceinline__ float hi_f32(uint64_t v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
// 2^x for a pair on the FMA / ALU pipes only (no MUFU, no F2I / FRND: those share the MUFU's
// quarter-rate pipe): x = n + f with n = rint(x) taken from the low mantissa bits of x + 1.5*2^23,
// f in [-0.5, 0.5], 2^f by a cubic (max relative error 7.5e-5, far below the bf16 rounding P gets
// next), n added into the exponent field. x < -126 -> ~1e-38 (masked keys: -inf); the clamp keeps
// the exponent sum positive (2^f < 1 for f < 0).
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
    constexpr float kMagic = 12582912.f;  // 1.5 * 2^23
    const uint64_t xc = f32x2(fmaxf(lo_f32(x2), -126.f), fmaxf(hi_f32(x2), -126.f));
    const uint64_t t = fadd2(xc, f32x2(kMagic, kMagic));
    const uint64_t r = fadd2(t, f32x2(-kMagic, -kMagic));
    const uint64_t f = ffma2(r, f32x2(-1.f, -1.f), xc);
    uint64_t q = ffma2(f32x2(0.05517588f, 0.05517588f), f, f32x2(0.24261151f, 0.24261151f));
    q = ffma2(q, f, f32x2(0.69326019f, 0.69326019f));
    q = ffma2(q, f, f32x2(0.99992800f, 0.99992800f));
    const int lo = __float_as_int(lo_f32(q)) + (__float_as_int(lo_f32(t)) << 23);
    const int hi = __float_as_int(hi_f32(q)) + (__float_as_int(hi_f32(t)) << 23);
    return f32x2(__int_as_float(lo), __int_as_float(hi));
}
// MUFU.EX2 alone (exp2f adds range fix-ups: 3 more instructions per element)
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One 64-key K or V sub-tile (4 pool blocks x 2 64-dim halves = 8 TMA boxes of 16 rows) and its
// barrier's expect_tx as ONE elected issue: rows r0..r3 are the blocks' pool rows, the boxes land
// at dst + bb * 2 KB (dims 0-63) and dst + 8 KB + bb * 2 KB (dims 64-127).
__device__ __forceinline__ void tma_kv_subtile_warp(void* dst, const CUtensorMap* m, uint64_t* bar, int r0, int r1,
                                                    int r2, int r3, uint64_t policy, uint32_t bytes) {
    asm volatile(
        "{\n"
        ".reg .pred e;\n"
        ".reg .b32 d;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %9;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%2, {%10, %3}], [%1], %7;\n"
        "add.u32 d, %0, 8192;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [d], [%2, {%8, %3}], [%1], %7;\n"
        "add.u32 d, %0, 2048;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [d], [%2, {%10, %4}], [%1], %7;\n"
        "add.u32 d, %0, 10240;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [d], [%2, {%8, %4}], [%1], %7;\n"
        "add.u32 d, %0, 4096;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [d], [%2, {%10, %5}], [%1], %7;\n"
        "add.u32 d, %0, 12288;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [d], [%2, {%8, %5}], [%1], %7;\n"
        "add.u32 d, %0, 6144;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [d], [%2, {%10, %6}], [%1], %7;\n"
        "add.u32 d, %0, 14336;\n"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [d], [%2, {%8, %6}], [%1], %7;\n"
        "}\n" ::"r"(smem_u32(dst)),
        "r"(smem_u32(bar)), "l"(reinterpret_cast<uint64_t>(m)), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(policy), "r"(64),
        "r"(bytes), "r"(0)
        : "memory");
}

// One S = Q K^T tile (M = 128 queries, N = 64 keys, K = 128 dims) as ONE elected issue of 8
// MMAs: the K-step descriptors are the base plus immediates (32 B along K inside a 128-B swizzle
// row = +2, the second 64-dim half = +1024 for Q's 16-KB half, +512 for K's 8-KB half), so the
// whole group costs one ELECT and a handful of uniform adds instead of ~12 instructions per MMA.
__device__ __forceinline__ void mma_s_tile_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred e, pf, pt;\n"
        ".reg .b64 a, b;\n"
        "setp.ne.b32 pf, 0, 0;\n"
        "setp.eq.b32 pt, 0, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pf;\n"
        "add.s64 a, %1, 2;\n add.s64 b, %2, 2;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, 4;\n add.s64 b, %2, 4;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, 6;\n add.s64 b, %2, 6;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, 1024;\n add.s64 b, %2, 512;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, 1026;\n add.s64 b, %2, 514;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, 1028;\n add.s64 b, %2, 516;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n"
        "add.s64 a, %1, 1030;\n add.s64 b, %2, 518;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, pt;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc)
        : "memory");
}
// O += P V for one 64-key sub-tile as ONE elected issue of 4 MMAs (K = 16 keys each): P from
// TMEM (+8 packed columns per step), V MN-major from smem (+2 KB = +128 per step).
__device__ __forceinline__ void mma_pv_tile_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred e, p0, pt;\n"
        ".reg .b64 b;\n"
        ".reg .b32 a;\n"
        "setp.ne.b32 p0, %4, 0;\n"
        "setp.eq.b32 pt, 0, 0;\n"
        "elect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p0;\n"
        "add.s32 a, %1, 8;\n add.s64 b, %2, 128;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.s32 a, %1, 16;\n add.s64 b, %2, 256;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, pt;\n"
        "add.s32 a, %1, 24;\n add.s64 b, %2, 384;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [a], b, %3, pt;\n"
        "}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// ============================================================ ping-pong kernel
// Two 128-row query tiles per CTA, one softmax warpgroup each, sharing the K/V rings. Keys go
// in 64-key sub-tiles and every tile has TWO S buffers in the tensor memory, so the MMA warp
// computes S_i(k+1) while warpgroup i exponentiates S_i(k): the softmax never waits for its
// next scores, and the tensor pipe interleaves the two tiles' PV / S MMAs:
//   PV_0(k), S_0(k+2), PV_1(k), S_1(k+2)
// P never leaves the tensor memory: warpgroup i writes bf16 P over the first 32 columns of the
// S buffer it read (tcgen05.st) and the PV MMA takes A straight from TMEM. MMAs execute in
// issue order, so S_i(k+2) (same buffer as P_i(k)) follows PV_i(k). The lazy O rescale (rare:
// only when a row max grows by more than 2^8) first waits for PV_i(k-1): S_i(k+1), issued right
// after it, retiring says so (one commit per MMA group is all the issue loop can afford: each
// tcgen05.commit costs the issuing thread ~100+ cycles).
// TMEM: S_0a | S_0b | S_1a | S_1b (64 columns each) | O_0 | O_1 (128 each) = 512 columns.
// smem: Q_0, Q_1 (32 KB each), K and V rings of kStages 16-KB sub-tiles, the block ids.
//
// GQA packing: a 128-row tile holds HT query heads x TT = 128/HT tokens of ONE kv head
// (head-major: rows [g*TT, (g+1)*TT) are head g), so a CTA's two tiles cover 2*TT tokens of
// HT heads and every K/V tile it loads serves all of them; HT = 4 for LLaMA (G = 4), 1 for
// Qwen2 (G = 7). A unit = (kv head, head subgroup, token block of 2*TT tokens).
//
// Balanced key split: when the units do not fill the partition (a 448-token chunk is 56 units
// for 108 SMs), each unit's key sub-tiles are cut into pieces of at most steps_cap (the
// smallest cap whose piece count fits one wave, chosen on the host). A piece's unnormalised O
// (fp32, coalesced [tile][dim/4][row] float4 layout) and per-row (max, sum) go to ws; the last
// piece of a unit to finish (self-resetting ticket) folds the others into its own TMEM
// accumulator and writes the bf16 rows. Units run heaviest first (token blocks descending).
//
// PDL: K/V wholly below pos0 was written by earlier passes (a pass starts with a
// stream-ordered metadata copy), so the producer requests those sub-tiles before
// griddepcontrol.wait; Q and the chunk's own keys only after it.
constexpr int kPPOffQ = 0;
constexpr int kPPOffK = kPPOffQ + 2 * kQTileBytes;
constexpr int kPPOffV = kPPOffK + kStages * kKVTileBytes;
constexpr int kPPOffTab = kPPOffV + kStages * kKVTileBytes;  // the piece's block ids (first kPPTabMax)
constexpr int kPPTabMax = 256;                               // 64 sub-tiles = 4k keys (then from global)
constexpr int kPPOffBar = kPPOffTab + kPPTabMax * 4;
constexpr int kPPSmemBytes = kPPOffBar + 512 + 1024;  // barriers (36 x 8 B) + alignment slack
static_assert(kPPSmemBytes <= 232448, "smem budget");
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
    int steps_cap;  // key sub-tiles per piece at most
    float* ws;      // piece partials [grid][kPfWsFloats]
    int* tickets;   // [grid], zero, self-resetting
    long long* probe;  // dev (CRONUS_PF_PROBE=1): per-CTA clock64 stamps [grid][128], else null
    int ablate;        // dev (CRONUS_PF_ABLATE): bit 0 / 2 = no V / K loads, bit 1 = no exp (P = S), bit 3 = all exp on MUFU, bit 4 = parked waits, bit 7 / 8 = no PV / S MMAs; 0 in production
};

// dev probe: clock64 stamp `slot` of this CTA (pipeline events; see launch_prefill)
__device__ __forceinline__ void pf_stamp(const PfParams& p, int slot) {
    if (p.probe != nullptr && slot < 128) p.probe[blockIdx.x * 128 + slot] = clock64();
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}
__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }


// Pipeline waits poll (dev: ablate bit 16 parks the warp with a suspend hint instead, so waiting
// warps leave issue slots to the softmax warps; measured 2-3 % slower). `helper` = the producer /
// MMA warps, which share SM sub-partitions 0 / 1 with softmax warps (dev: ablate bit 5 parks only
// those).
__device__ __forceinline__ void pf_wait(const PfParams& p, uint64_t* bar, uint32_t parity, bool helper = false) {
    if ((p.ablate & 16) || (helper && (p.ablate & 32)))
        mbar_wait_park(bar, parity);
    else
        mbar_wait(bar, parity);
}

// Key tiles of token block tb (its second tile's last valid token).
template <int HT>
__host__ __device__ __forceinline__ int pf_steps(int q_len, int pos0, int tb) {
    constexpr int TT = 128 / HT;
    const int end = (tb + 1) * 2 * TT < q_len ? (tb + 1) * 2 * TT : q_len;
    return (pos0 + end + kKT - 1) / kKT;
}

template <int HT, int NPOLY>
__global__ void __launch_bounds__(kPPThreads, 1)
    attn_prefill_pp_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                           PfParams p) {
    constexpr int TT = 128 / HT;
    constexpr int BPT = kKT / 16;  // 16-token pool blocks per sub-tile
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + kPPOffBar);
    uint64_t* q_full = bar + 0;                // [2] per query tile
    uint64_t* s_full = bar + 2;                // [2 tiles][2 buffers]
    uint64_t* p_full = bar + 6;                // [2 tiles][2 buffers] (4 warp arrivals)
    uint64_t* pv_done = bar + 10;              // [2] per tile, one phase per PV
    uint64_t* o_done = bar + 12;               // [2] per tile
    uint64_t* k_full = bar + 14;               // [kStages]
    uint64_t* k_empty = k_full + kStages;      // [kStages]
    uint64_t* v_full = k_empty + kStages;      // [kStages]
    uint64_t* v_empty = v_full + kStages;      // [kStages]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + kStages);
    int* s_last = reinterpret_cast<int*>(v_empty + kStages + 1);

    const int warp = warp_id(), lane = lane_id();
    if (threadIdx.x == 0) pf_stamp(p, 0);
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
            mbar_init(&pv_done[i], 1);
            mbar_init(&o_done[i], 1);
            for (int bb = 0; bb < 2; ++bb) {
                mbar_init(&s_full[i * 2 + bb], 1);
                mbar_init(&p_full[i * 2 + bb], 4);
            }
        }
        for (int st = 0; st < kStages; ++st) {
            mbar_init(&k_full[st], 1);
            mbar_init(&k_empty[st], 1);
            mbar_init(&v_full[st], 1);
            mbar_init(&v_empty[st], 1);
        }
        fence_mbar_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_launch();
    if (threadIdx.x == 0) pf_stamp(p, 1);

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        // The piece's block ids are staged in smem by the whole warp (coalesced, one round
        // trip; metadata, so before griddepcontrol.wait): a TMA issue loop that reads the
        // table from global pays one dependent L2 round trip per 16-token block.
        const int n_tab = (p.pos0 + min(p.q_len, (tb + 1) * 2 * TT) + 15) / 16;
        int* tab = reinterpret_cast<int*>(sm + kPPOffTab);
        const int t0 = j0 * BPT, n_stage = min(jmax * BPT, kPPTabMax);
        for (int x = lane; x < n_stage; x += 32) {
            const int ti = t0 + x;
            tab[x] = p.table[ti < n_tab ? ti : 0];  // past the end: any finite block (masked)
        }
        __syncwarp();
        {  // whole warp, convergent: one elected lane issues (see mma_ss_warp)
            const uint64_t keep = policy_evict_last();
            auto row_of = [&](int k) {  // lane bb < BPT: pool row of sub-tile k's block bb
                int my_row = 0;
                if (lane < BPT) {
                    const int x = k * BPT + lane, ti = t0 + x;
                    const int id = x < kPPTabMax ? tab[x] : p.table[ti < n_tab ? ti : 0];
                    my_row = ((id * p.n_layers + p.layer) * 2 + 0) * p.nkv * 16 + kvh * 16;
                }
                return my_row;
            };
            auto load_k = [&](int k) {
                const int st = k % kStages;
                const int my_row = row_of(k);
                pf_wait(p, &v_empty[st], ((k / kStages) & 1) ^ 1, true);  // stage free: K(k-5), V(k-5) consumed
                if (k < 16 && lane == 0) pf_stamp(p, 88 + k);
                uint8_t* K = sm + kPPOffK + st * kKVTileBytes;
                if (p.ablate & 4) {  // dev ablation: K = whatever the stage holds
                    if (lane == 0) mbar_arrive(&k_full[st]);
                    return;
                }
                static_assert(BPT == 4 && kKVHalf == 8192, "tma_kv_subtile_warp layout");
                tma_kv_subtile_warp(K, &tmKV, &k_full[st], __shfl_sync(0xffffffffu, my_row, 0),
                                    __shfl_sync(0xffffffffu, my_row, 1), __shfl_sync(0xffffffffu, my_row, 2),
                                    __shfl_sync(0xffffffffu, my_row, 3), keep, kKVTileBytes);
            };
            auto load_v = [&](int k) {
                const int st = k % kStages;
                const int my_row = row_of(k);
                // (the stage was found free by load_k(k), always issued first)
                if (k < 16 && lane == 0) pf_stamp(p, 104 + k);
                if (p.ablate & 1) {  // dev ablation: V = whatever the stage holds
                    if (lane == 0) mbar_arrive(&v_full[st]);
                    return;
                }
                uint8_t* V = sm + kPPOffV + st * kKVTileBytes;
                const int vr = my_row + p.nkv * 16;
                tma_kv_subtile_warp(V, &tmKV, &v_full[st], __shfl_sync(0xffffffffu, vr, 0),
                                    __shfl_sync(0xffffffffu, vr, 1), __shfl_sync(0xffffffffu, vr, 2),
                                    __shfl_sync(0xffffffffu, vr, 3), keep, kKVTileBytes);
            };
            // Issue order = arrival order (the TMA unit serves requests in order): the first
            // two K sub-tiles (if wholly prefix: before griddepcontrol.wait), then Q, then V(0),
            // V(1) and the rest in step order; Q queued behind several stages of K/V arrives
            // microseconds late and holds the first S MMA.
            int pre = 0;
            while (pre < 2 && pre < jmax && (j0 + pre + 1) * kKT <= p.pos0) load_k(pre++);
            pdl_wait();
            for (int i = 0; i < n_qt; ++i) {
                mbar_expect_tx_warp(&q_full[i], kQTileBytes);
                uint8_t* Q = sm + kPPOffQ + i * kQTileBytes;
                const int qrow = p.q_row0 + t_base[i];
#pragma unroll
                for (int g = 0; g < HT; ++g) {
                    tma_load_2d_hint_warp(Q + g * TT * 128, &tmQ, &q_full[i], (h_base + g) * 128, qrow, keep);
                    tma_load_2d_hint_warp(Q + kQHalf + g * TT * 128, &tmQ, &q_full[i], (h_base + g) * 128 + 64, qrow, keep);
                }
            }
            for (int k = 0; k < jmax; ++k) {
                if (k >= pre) load_k(k);
                load_v(k);
            }
        }
    } else if (warp == 1) {
        pdl_wait();
        // ------------------------------------------------------------ MMA issuer (whole warp)
        // Each 64-key S tile (8 MMAs) and PV step (4 MMAs) is one elected issue with uniform
        // descriptor arithmetic (mma_s_tile_warp / mma_pv_tile_warp): the warp shares an SM
        // sub-partition with two softmax warps, and its issue cost set their pace (per-MMA
        // issue: ~2300 cycles per 64-key step; batched: ~1900). Splitting the issue over two
        // warps on two sub-partitions (one per tile) measured 2-3 % slower again.
        {
            const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // provably warp-uniform
            constexpr uint32_t id_s = idesc_attn(false, kKT), id_o = idesc_attn(true, 128);
            for (int i = 0; i < n_qt; ++i) pf_wait(p, &q_full[i], 0, true);
            if (lane == 0) pf_stamp(p, 2);
            auto issue_s = [&](int i, int k) {  // S_i(k) = Q_i K(k)^T -> S buffer (i, k & 1)
                const uint32_t q0 = smem_u32(sm + kPPOffQ + i * kQTileBytes);
                const uint32_t k0 = smem_u32(sm + kPPOffK + (k % kStages) * kKVTileBytes);
                static_assert(kQHalf == 16384 && kKVHalf == 8192, "mma_s_tile_warp immediates");
                if (!(p.ablate & 256))  // dev ablation: no S MMAs (timing only)
                    mma_s_tile_warp(tm + i * 128 + (k & 1) * 64, sdesc_sw128(q0), sdesc_sw128(k0), id_s);
                tc_commit_warp(&s_full[i * 2 + (k & 1)]);
            };
            auto k_ready = [&](int k) {
                pf_wait(p, &k_full[k % kStages], (k / kStages) & 1, true);
                tc_fence_after();
            };
            for (int k = 0; k < 2 && k < jmax; ++k) {
                k_ready(k);
                for (int i = 0; i < 2; ++i)
                    if (k < cnt[i]) issue_s(i, k);
            }
            for (int k = 0; k < jmax; ++k) {
                const bool ahead = k + 2 < jmax;
                pf_wait(p, &v_full[k % kStages], (k / kStages) & 1, true);
                tc_fence_after();
                if (ahead) k_ready(k + 2);
                const uint32_t v0 = smem_u32(sm + kPPOffV + (k % kStages) * kKVTileBytes);
                for (int i = 0; i < 2; ++i) {
                    if (k < cnt[i]) {  // O_i += P_i(k) V(k), P from TMEM (packed bf16 pairs)
                        pf_wait(p, &p_full[i * 2 + (k & 1)], (k >> 1) & 1, true);
                        if (k < 16 && lane == 0) pf_stamp(p, 24 + 16 * i + k);
                        tc_fence_after();
                        static_assert(kKT == 64, "mma_pv_tile_warp issues 4 K = 16 steps");
                        if (!(p.ablate & 128))  // dev ablation: no PV MMAs (timing only)
                            mma_pv_tile_warp(tm + 256 + i * 128, tm + i * 128 + (k & 1) * 64, sdesc_mn_sw128(v0),
                                             id_o, k > 0 ? 1u : 0u);
                        // S_i(k+1) (issued right after PV_i(k-1)) retiring tells the softmax that
                        // PV_i(k-1) did; only the last step has no S_i(k+1): PV_i(cnt-2) commits here
                        if (k == cnt[i] - 2) tc_commit_warp(&pv_done[i]);
                        if (k == cnt[i] - 1) tc_commit_warp(&o_done[i]);
                    }
                    if (k + 2 < cnt[i]) issue_s(i, k + 2);
                }
                if (k < 16 && lane == 0) pf_stamp(p, 8 + k);
                // K(k) and V(k) share one stage, freed by ONE commit once PV(k) (issued after S(k))
                // of both tiles retires: one tcgen05.commit per step fewer than separate K / V
                // releases (the producer still runs K three steps ahead of its use)
                tc_commit_warp(&v_empty[k % kStages]);
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
        for (int k = 0; k < cnt_i; ++k) {
            pf_wait(p, &s_full[i * 2 + (k & 1)], (k >> 1) & 1);
            if (threadIdx.x == 64 && k < 16) pf_stamp(p, 56 + k);
            tc_fence_after();
            const uint32_t sb = s_col + (k & 1) * 64;
            uint32_t sv[2][32];
            tmem_ld32(sb, sv[0]);
            tmem_ld32(sb + 32, sv[1]);
            tmem_ld_wait();
            if (threadIdx.x == 64 && k == 10) pf_stamp(p, 121);  // dev: S in registers
            const int key0 = (j0 + k) * kKT;
            if (key0 + kKT - 1 > warp_q0) {  // diagonal sub-tile: causal mask
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (key0 + c * 32 + e > qpos) sv[c][e] = __float_as_uint(-INFINITY);
            }
            // P = exp2(S * scale - m) -> bf16 pairs over the buffer's first 32 columns, computed
            // speculatively against the running max m_ref while the row max is reduced (8
            // independent chains each: one softmax warp per SM sub-partition and warpgroup has
            // no other latency cover); only when the max grows by more than 2^8 (rare; always
            // on a piece's first sub-tile) is P recomputed against the new max and O rescaled.
            // A row whose keys in this piece are all masked keeps m = -inf: P = 0, not NaN.
            float pmx[8], rsp[8];
            uint32_t pk[2][16];
            // exponentials in fp32 pairs: x = S * scale - m and the row sums on the paired FMA /
            // add pipes (FFMA2 / FADD2: half the instructions of the scalar forms), 2^x on MUFU
            // for 3 of every 4 column groups and on the FMA pipe (cubic) for the 4th
            auto exp_pack = [&](float m_use) {
                const uint64_t sc2 = f32x2(p.scale_log2, p.scale_log2), nm2 = f32x2(-m_use, -m_use);
                uint64_t rs2[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) rs2[e] = 0ull;
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        const bool poly = g >= 4 - NPOLY && !(p.ablate & 8);
#pragma unroll
                        for (int e = 0; e < 8; e += 2) {
                            const uint64_t x2 = ffma2(f32x2(__uint_as_float(sv[c][g * 8 + e]),
                                                            __uint_as_float(sv[c][g * 8 + e + 1])),
                                                      sc2, nm2);
                            const float x0 = lo_f32(x2), x1 = hi_f32(x2);
                            float p0, p1;
                            if (p.ablate & 2) {
                                p0 = x0;
                                p1 = x1;
                            } else if (poly) {
                                const uint64_t e2 = exp2_poly2(x2);
                                p0 = lo_f32(e2);
                                p1 = hi_f32(e2);
                            } else {
                                p0 = ex2_approx(x0);
                                p1 = ex2_approx(x1);
                            }
                            rs2[e >> 1] = fadd2(rs2[e >> 1], f32x2(p0, p1));
                            pk[c][g * 4 + (e >> 1)] = pack_bf16x2(p0, p1);
                        }
                    }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    rsp[2 * e] = lo_f32(rs2[e]);
                    rsp[2 * e + 1] = hi_f32(rs2[e]);
                }
            };
#pragma unroll
            for (int e = 0; e < 8; ++e) pmx[e] = -INFINITY;
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int e = 0; e < 32; ++e) pmx[e & 7] = fmaxf(pmx[e & 7], __uint_as_float(sv[c][e]));
            if (m_ref != -INFINITY) exp_pack(m_ref);
            const float mx = fmaxf(fmaxf(fmaxf(pmx[0], pmx[1]), fmaxf(pmx[2], pmx[3])),
                                   fmaxf(fmaxf(pmx[4], pmx[5]), fmaxf(pmx[6], pmx[7]))) *
                             p.scale_log2;
            const bool need = __any_sync(0xffffffffu, mx > m_ref + kRescaleThreshold || m_ref == -INFINITY);
            if (need) {
                const float m_new = fmaxf(m_ref, mx);
                const float corr = m_ref == -INFINITY ? 0.f : exp2f(m_ref - m_new);
                l_sum *= corr;
                m_ref = m_new;
                exp_pack(m_ref == -INFINITY ? 0.f : m_ref);
                if (k > 0) {
                    // O holds PV_i(0..k-1) once PV_i(k-1) retires (PV_i(k) waits for this P):
                    // S_i(k+1) was issued right after it, or, at the last step, PV_i(k-1) commits
                    if (k + 1 < cnt_i)
                        pf_wait(p, &s_full[i * 2 + ((k + 1) & 1)], ((k + 1) >> 1) & 1);
                    else
                        pf_wait(p, &pv_done[i], 0);
                    tc_fence_after();
#pragma unroll 1
                    for (int c = 0; c < 8; ++c) {  // 16 columns at a time
                        uint32_t o[16];
                        tmem_ld16(o_col + c * 16, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 16; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
                        tmem_st16(o_col + c * 16, o);
                    }
                }
            }
            if (threadIdx.x == 64 && k == 10) pf_stamp(p, 122);  // dev: P computed
            tmem_st16(sb, pk[0]);
            tmem_st16(sb + 16, pk[1]);
            tmem_st_wait();
            if (threadIdx.x == 64 && k == 10) pf_stamp(p, 123);  // dev: P stored
            l_sum += ((rsp[0] + rsp[1]) + (rsp[2] + rsp[3])) + ((rsp[4] + rsp[5]) + (rsp[6] + rsp[7]));
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[i * 2 + (k & 1)]);
            if (threadIdx.x == 64 && k < 16) pf_stamp(p, 72 + k);
        }
        if (cnt_i > 0) {
            pf_wait(p, &o_done[i], 0);
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
                    if (f != 0.f) L += f * lq;
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
                        for (int e = 0; e < 32; ++e) acc[e] = f_own != 0.f ? __uint_as_float(o[e]) * f_own : 0.f;
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
    if (threadIdx.x == 64) pf_stamp(p, 120);
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
// one wave (pieces of 4+ sub-tiles, at most 4 per unit).
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
        // pieces of at least kMinPiece sub-tiles: a piece's setup (Q load, pipeline fill) and the
        // merge cost ~2-3 us, as much as a few hundred keys of work
        // and at most kMaxPieces per unit: the last piece reads every other piece's 128 KB
        // partial from L2 on the kernel's critical path
        static const int kMinPiece = [] {  // dev: CRONUS_PF_MIN_PIECE / CRONUS_PF_MAX_PIECES
            const char* e = std::getenv("CRONUS_PF_MIN_PIECE");
            return e ? std::max(1, std::atoi(e)) : 4;
        }();
        static const int kMaxPieces = [] {
            const char* e = std::getenv("CRONUS_PF_MAX_PIECES");
            return e ? std::max(1, std::atoi(e)) : 4;
        }();
        int c = static_cast<int>(std::max<long long>(std::max(kMinPiece, (n_max + kMaxPieces - 1) / kMaxPieces),
                                                     (total + max_ctas - 1) / max_ctas));
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
    // 2^x column groups (of 4) on the FMA pipe instead of MUFU (dev: CRONUS_PF_NPOLY 1-2; 0, all
    // on MUFU, measured fastest: 448 @ 1024 26.4 vs 27.6 us, 4096 @ 0 163 vs 177 us)
    static const int npoly = [] {
        const char* e = std::getenv("CRONUS_PF_NPOLY");
        return e ? std::min(2, std::max(0, std::atoi(e))) : 0;
    }();
    auto* kern = npoly == 0 ? attn_prefill_pp_kernel<HT, 0> : npoly == 2 ? attn_prefill_pp_kernel<HT, 2>
                                                                         : attn_prefill_pp_kernel<HT, 1>;
    static unsigned mask = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(mask & (1u << dev))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kPPSmemBytes);
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
    static const bool probe = [] {
        const char* e = std::getenv("CRONUS_PF_PROBE");
        return e && e[0] == '1';
    }();
    prm.probe = nullptr;
    static const int ablate = [] {
        const char* e = std::getenv("CRONUS_PF_ABLATE");
        return e ? std::atoi(e) : 0;
    }();
    prm.ablate = ablate;
    if (!probe) return launch_pdl(kern, dim3(grid), dim3(kPPThreads), kPPSmemBytes, st, mq, mkv, prm);
    // dev: clock64 pipeline stamps of CTA 0 (the heaviest piece), relative to kernel entry
    long long* buf = nullptr;
    cudaMalloc(&buf, static_cast<size_t>(grid) * 128 * 8);
    cudaMemsetAsync(buf, 0, static_cast<size_t>(grid) * 128 * 8, st);
    prm.probe = buf;
    int rc2 = launch_pdl(kern, dim3(grid), dim3(kPPThreads), kPPSmemBytes, st, mq, mkv, prm);
    std::vector<long long> h(128);
    cudaMemcpyAsync(h.data(), buf, 128 * 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    cudaFree(buf);
    auto d = [&](int k) { return h[k] ? h[k] - h[0] : -1; };
    std::fprintf(stderr, "[pf probe] q_len=%d pos0=%d grid=%d cap=%d setup=%lld q_full=%lld end=%lld\n", q_len, pos0,
                 grid, prm.steps_cap, d(1), d(2), d(120));
    std::fprintf(stderr, "  step 10, warp 2: S seen %lld, S in registers %lld, P computed %lld, P stored %lld, P arrive %lld\n",
                 d(56 + 10), d(121), d(122), d(123), d(72 + 10));
    for (int jj = 0; jj < 16; ++jj)
        if (h[8 + jj] || h[88 + jj])
            std::fprintf(stderr, "  jj=%2d K_issue=%7lld V_issue=%7lld v_full=%7lld S0_done=%7lld P0_arrive=%7lld "
                                 "p0_seen=%7lld p1_seen=%7lld\n",
                         jj, d(88 + jj), d(104 + jj), d(8 + jj), d(56 + jj), d(72 + jj), d(24 + jj), d(40 + jj));
    return rc2;
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
