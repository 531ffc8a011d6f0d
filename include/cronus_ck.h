/* cronus_ck.h — the thin C-ABI kernel layer of the B200 engine (sm_100a).
 *
 * Every entry point takes raw device pointers, plain sizes and a cudaStream_t
 * passed as void*, never allocates, and returns a cudaError_t as int (0 = ok).
 * The C++ host (csrc/gpu/) is the only production caller; tests call the same
 * symbols through ctypes with torch-allocated buffers.
 *
 * These kernels replace the reference simulator's three cost-model stand-ins
 * (proj/src/costmodel.cpp:9-15 prefill_time / chunked_iter_time and
 * proj/src/model.cpp:11-13 transfer_time): the work those formulas price is
 * what these kernels actually perform.
 *
 * KV cache layout (one pool per worker, block-major, bf16):
 *   pool[block][layer][K=0|V=1][kv_head][16 tokens][128 dims]
 * so a block is one contiguous slab (2 MiB for LLaMA3-8B) — the unit of the
 * PPI -> CPI handoff — and every (block, layer, K|V, head) tile is a contiguous
 * 4 KiB run for the attention kernels.
 */
#ifndef CRONUS_CK_H
#define CRONUS_CK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GEMM epilogues */
enum { CK_EPI_BF16 = 0, CK_EPI_F32 = 1, CK_EPI_RED_F32 = 2, CK_EPI_SILU_BF16 = 3 };

/* out[m, n] (op)= sum_k X[m, k] W[n, k] (+ bias[n]); W [N, K], X [M, K] bf16 row-major.
 * N % 128 == 0, K % 64 == 0. epi: CK_EPI_BF16 (store bf16), CK_EPI_F32 (store
 * fp32), CK_EPI_RED_F32 (red.add fp32 into out — residual add / split-K),
 * CK_EPI_SILU_BF16 (W rows interleaved gate/up: 2i = gate_i, 2i+1 = up_i; out is the
 * bf16 activation [M, ldo] with out[m, i] = silu(gate) * up; splits must be 1 — or, through
 * ck_gemm_fused with splits 0 and a CK_FUSE_SILU fuse: hybrid, whole tiles write fuse->act
 * directly and the tiles of a sparse last wave run as stream-K pieces red.added into `out`
 * (a zeroed fp32 [M, N] accumulator, left zero) and finalized by ticket).
 * splits: K splits (0 = auto; > 1 only with CK_EPI_RED_F32). max_ctas: cap on
 * the persistent grid (0 = all SMs). tcgen05 + TMEM + TMA. */
int ck_gemm(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int ldo, int epi,
            int splits, int max_ctas, void* stream);

/* Fused finalize of a GEMM output tile (128 output columns x BN tokens), run by the
 * last CTA to complete the tile (per-tile ticket counting finished K-blocks):
 *   CK_FUSE_QKV_ROPE: the tile is one 128-dim head of the fp32 qkv accumulator ->
 *                     RoPE(q) -> q_out bf16, RoPE(k) / v -> paged KV slot of each row
 *   CK_FUSE_SILU:     64 interleaved (gate, up) pairs -> act bf16 = silu(g) * u
 *   CK_FUSE_RMSNORM:  (residual red.add GEMM, out = x [M, N] fp32) each tile clears its
 *                     slice of `zero` [M, zero_cols]; the last tile of an m-tile to
 *                     complete (row_tickets: one int per m tile) writes
 *                     norm_out bf16 [M, N] = rmsnorm(x) * gamma, as ck_rmsnorm does —
 *                     the next layer's norm without its own launch. N <= 4096.
 * zero_after clears the accumulator tile after reading it (red.add reuse). tickets:
 * one int per (n tile, m tile), zero before the first call, left zero. */
enum { CK_FUSE_NONE = 0, CK_FUSE_QKV_ROPE = 1, CK_FUSE_SILU = 2, CK_FUSE_RMSNORM = 3 };
typedef struct {
    int kind;
    int zero_after;
    int* tickets;
    /* QKV_ROPE */
    void* q_out;
    void* kv_pool;
    const int* bt;
    const int* row_bt;
    const int* row_pos;
    const float* cos_tab;
    const float* sin_tab;
    int nq, nkv, layer, n_layers;
    /* SILU */
    void* act;
    /* RMSNORM */
    const void* gamma;
    void* norm_out;
    float eps;
    int zero_cols;
    float* zero;
    int* row_tickets;
} ck_gemm_fuse;

int ck_gemm_fused(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int epi,
                  int splits, int max_ctas, const ck_gemm_fuse* fuse, void* stream);

/* Deterministic uniform init: out[i] = bf16(offset + scale * u_i), u_i in [-1, 1)
 * from splitmix64(seed, tensor_id, i) (restated in oracle/numerics.py). */
int ck_init_uniform(void* out_bf16, long long n, unsigned long long seed, unsigned long long tensor_id,
                    float scale, float offset, void* stream);

/* Prompt tokens: tok[i] = splitmix64(seed, req_id[i], pos[i]) % vocab for n rows. */
int ck_prompt_tokens(int* out, const int* req_id, const int* pos, int n, unsigned long long seed, int vocab,
                     void* stream);

/* RoPE cos/sin table [max_pos][64] fp32 each (computed in double). */
int ck_rope_table(float* cos_tab, float* sin_tab, int max_pos, double theta, void* stream);

/* Per-row metadata of one forward pass (device pointers):
 *   row_rid[M]   request slot of the row
 *   row_pos[M]   absolute position of the row's token
 *   row_dec[M]   1: token = last_tok[rid] (decode row); 0: prompt[prompt_off[rid] + pos]
 */
int ck_embed(float* x, const void* emb_bf16, const int* row_rid, const int* row_pos, const int* row_dec,
             const int* prompt, const long long* prompt_off, const int* last_tok, int M, int H, void* stream);

/* out_bf16[r] = rmsnorm(x[rows ? rows[r] : r]) * gamma, r < R. If `zero` is not
 * null, row r of zero[R, zero_cols] (fp32) is also cleared — the accumulation buffer
 * of the next red.add GEMM, so no separate memset launch is needed. */
int ck_rmsnorm(const float* x, const void* gamma, void* out_bf16, const int* rows, int R, int H, float eps,
               float* zero, int zero_cols, void* stream);

/* qkv fp32 [M, (nq + 2 nkv) * 128] (+ bias) -> RoPE(q) bf16 [M, nq*128] and
 * RoPE(k), v appended to the paged pool at each row's position.
 * bt: flat block table; row_bt[M] = offset of the row's sequence in bt.
 * zero_after: clear the qkv rows after reading them (red.add accumulator reuse). */
int ck_qkv_rope_append(float* qkv, const void* bias, void* q_out, void* kv_pool, const int* bt, const int* row_bt,
                       const int* row_pos, const float* cos_tab, const float* sin_tab, int M, int nq, int nkv,
                       int layer, int n_layers, int zero_after, void* stream);

/* Decode attention over the paged pool for S single-token sequences, production path:
 * seq_row[S] (row of q/out), seq_len[S] (keys), seq_bt[S] (offset into bt),
 * seq_item0[S] (first work item of each sequence; its parts are contiguous). ws: fp32 partials,
 * n_work * nq * 130 floats. tickets: n_seq * nkv ints, zero before the first call
 * (the kernel leaves them zero). Output bf16 rows [*, nq*128]. One launch.
 * K/V rings are filled by TMA (2-D map over the pool viewed as
 * [pool_blocks * n_layers * 2 * nkv * 16 rows][128]) and each work item is served by a
 * thread-block CLUSTER of `cluster` CTAs (1..16) that split the item's blocks and merge
 * through distributed shared memory. work[i] = seq << 16 | nparts << 8 | part (nparts <= 255);
 * the grid runs the items in list order (heaviest first is the caller's choice: the engine's
 * planner sorts them, LPT); a sequence's parts are evened out to ceil(nblocks / nparts) blocks; parts of one sequence
 * merge through ws / tickets (the last CTA of a (sequence, kv head) folds them). Partially
 * filled last blocks are read whole and masked, so never-written slots must hold finite
 * values (the engine zero-fills its pools). pool rows must be < 2^31. */
typedef struct {
    const float* qkv;     /* fp32 QKV rows [*, (nq + 2 nkv) * 128] (bias included), row = seq_row */
    const float* cos_tab; /* RoPE tables [max_pos][64] (ck_rope_table) */
    const float* sin_tab;
} ck_decode_rope;
/* rope != NULL: fused RoPE + KV append of the decode token (position seq_len - 1): q, k,
 * v come from rope->qkv (q is unused) and the token's K/V is written to its pool slot
 * (replaces ck_qkv_rope_append for decode-only passes; qkv is left for the caller to clear). */
int ck_attn_decode_tma(const void* q, const void* kv_pool, long long pool_blocks, const int* bt, const int* seq_row,
                       const int* seq_len, const int* seq_bt, const int* seq_item0, const int* work, int n_work,
                       int n_seq, int cluster, float* ws, int* tickets, void* out, int nq, int nkv, int layer,
                       int n_layers, float scale, const ck_decode_rope* rope, void* stream);

/* Prefill/chunk attention, causal, on the 5th-gen tensor cores (tcgen05 + TMEM + TMA):
 * query rows [q_row0, q_row0+q_len) of q (bf16 [q_rows_total, nq*128]) sit at positions
 * [pos0, pos0+q_len) and attend to keys [0, pos0+q_len) of the paged pool via bt.
 * Two 128-row query tiles per CTA with one softmax warpgroup each (ping-pong on the tensor
 * pipe) and P kept in TMEM as the A operand of the PV MMA; a tile packs the query heads of
 * one kv head (4 heads x 32 tokens for GQA groups of 4 / 8, 2 x 64 for 2, 1 x 128 else), so
 * each K/V tile is loaded once for all of them. When the (kv head, token block) units do not
 * fill max_ctas CTAs, their key ranges are cut into balanced pieces whose partials merge
 * through ws (ck_attn_prefill_ws_floats(max_ctas) floats) and tickets (max_ctas ints, zero,
 * left zero); ws = NULL never splits. pool_blocks: blocks in the pool (TMA bound). Stale
 * slots of a sequence's last block are read (and masked): the pool must hold finite values
 * (the engine zero-fills it at allocation). */
int ck_attn_prefill_pp(const void* q, int q_rows_total, const void* kv_pool, long long pool_blocks, const int* bt,
                       int q_row0, int q_len, int pos0, void* out, int nq, int nkv, int layer, int n_layers,
                       float scale, float* ws, int* tickets, int max_ctas, void* stream);
long long ck_attn_prefill_ws_floats(int max_ctas);

/* act[m, i] = silu(gu[m, 2i]) * gu[m, 2i+1]  (gate/up rows interleaved), fp32 in;
 * zero_after: clear gu after reading it. */
int ck_silu_mul(float* gu, void* act_bf16, int M, int F, int zero_after, void* stream);

/* Greedy sampling: token = argmax_v logits[r, v] (lowest index on ties), then
 * last_tok[rid[r]] = token, out_tok[out_idx[r]] = token. ws: 64 * R floats of
 * scratch; tickets: R ints, zero before the first call (left zero). zero_after:
 * clear the R logits rows after reading them (a red.add LM head accumulates into
 * them next). logits_out (nullable, test hook): row r's logits are also stored at
 * logits_out[out_idx[r] * V]. One launch. */
int ck_argmax_emit(float* logits, int R, int V, const int* rid, const long long* out_idx, int* last_tok,
                   int* out_tok, float* ws, int* tickets, int zero_after, float* logits_out, void* stream);

/* KV handoff: copy n_blocks blocks src_pool[src_ids[i]] -> dst_pool[dst_ids[i]]
 * (block_bytes each; src may be a peer-mapped pointer — pull over NVLink). */
int ck_kv_copy(const void* src_pool, const int* src_ids, void* dst_pool, const int* dst_ids, int n_blocks,
               long long block_bytes, void* stream);

/* Copy one int: dst[di] = src[si] (first token travelling with the handoff). */
int ck_copy_token(const int* src, long long si, int* dst, long long di, int* dst2, long long di2, void* stream);

int ck_device_sms(void);

/* Diagnostic: n_ctas CTAs each add 1 to hits[%smid] (hits sized >= 256). Used to
 * verify the SM partition of co-located workers. */
int ck_smid_probe(int* hits, int n_ctas, void* stream);

/* Diagnostic: occupy `stream` for `us` microseconds (one warp spinning on the timer). */
int ck_spin(int us, void* stream);

/* Diagnostic: stream `bytes` of `buf` with `ctas` CTAs; mode 0 = LDG.128, 1 = TMA
 * 128x64 bf16 boxes over a [rows][4096] matrix (the GEMM's weight pattern), 2 =
 * cp.async.bulk 16 KiB chunks. Time it with events on `stream`. */
int ck_bw_probe(const void* buf, long long bytes, int mode, int ctas, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CRONUS_CK_H */
