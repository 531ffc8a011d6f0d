// Decoder model on one B200: shapes, device-resident weights, per-worker
// workspaces and the forward pass over a ragged batch (decode rows + at most one
// prefill chunk) against a paged KV pool. Host orchestration only — every FLOP and
// byte moves in the sm_100a kernels behind include/cronus_ck.h.
#pragma once

#include <cuda_runtime.h>

#include "cronus_ck.h"

#include <cstdint>
#include <map>
#include <set>
#include <string>
#include <vector>

namespace cronus {
namespace gpu {

struct ModelSpec {
    std::string name;
    int hidden = 0;
    int layers = 0;
    int n_heads = 0;
    int n_kv_heads = 0;
    int head_dim = 128;
    int ffn = 0;
    int vocab = 0;
    double rope_theta = 500000.0;
    float rms_eps = 1e-5f;
    bool qkv_bias = false;
    // deterministic random init (uniform with these standard deviations)
    float w_std = 0.02f;
    float emb_std = 0.5f;
    float lm_std = 0.05f;
    uint64_t seed = 1234;
    int max_pos = 65536;

    int qkv_n() const { return (n_heads + 2 * n_kv_heads) * head_dim; }
    int q_n() const { return n_heads * head_dim; }
    long long kv_block_bytes() const { return 2LL * layers * n_kv_heads * 16 * head_dim * 2; }
    long long kv_bytes_per_token() const { return kv_block_bytes() / 16; }
    double linear_flops_per_token() const;  // 2 * (non-embedding linear params), LM head excluded
    long long weight_bytes() const;

    // "llama3-8b", "qwen2-7b", "tiny" (SURVEY.md section 8 model shapes)
    static ModelSpec preset(const std::string& name);
};

// Tensor ids for the deterministic init hash (restated in oracle/numerics.py).
enum : uint64_t { kTidEmbed = 1, kTidLmHead = 2, kTidFinalNorm = 3 };
inline uint64_t layer_tid(int l, int which) { return 16 + 16ull * l + which; }
enum : int { kWqkv = 0, kWo = 1, kWgu = 2, kWd = 3, kAttnNorm = 4, kFfnNorm = 5, kBqkv = 6 };

struct LayerWeights {
    void* wqkv = nullptr;  // [qkv_n, H]
    void* bqkv = nullptr;  // [qkv_n] (Qwen2) or null
    void* wo = nullptr;    // [H, nq*128]
    void* wgu = nullptr;   // [2F, H], row 2i = gate_i, row 2i+1 = up_i
    void* wd = nullptr;    // [H, F]
    void* attn_norm = nullptr;
    void* ffn_norm = nullptr;
};

class Weights {
  public:
    Weights(const ModelSpec& spec, int device);
    ~Weights();
    Weights(const Weights&) = delete;
    Weights& operator=(const Weights&) = delete;

    const ModelSpec& spec() const { return spec_; }
    int device() const { return dev_; }
    void* embed = nullptr;
    void* lm_head = nullptr;
    void* final_norm = nullptr;
    std::vector<LayerWeights> layer;
    float* cos_tab = nullptr;
    float* sin_tab = nullptr;

  private:
    ModelSpec spec_;
    int dev_;
    void* base_ = nullptr;
};

// A paged KV pool: `blocks` slabs of kv_block_bytes on one device.
struct KvPool {
    int device = 0;
    void* base = nullptr;
    long long blocks = 0;
    long long block_bytes = 0;
    KvPool() = default;
    KvPool(int dev, long long n_blocks, long long block_bytes);
    ~KvPool();
    KvPool(const KvPool&) = delete;
    KvPool& operator=(const KvPool&) = delete;
};

// Host description of one forward pass.
struct Batch {
    // rows (decode rows first, then the prefill chunk rows)
    std::vector<int> row_rid, row_pos, row_dec, row_bt;
    // decode sequences
    std::vector<int> d_row, d_len, d_bt, d_item0, d_work;
    int blocks_per_split = 16;
    // cluster size C >= 1 of the decode plan (plan_decode) for ck_attn_decode_tma
    int decode_cluster = 0;
    std::vector<double> plan_heap_;  // plan_decode scratch
    // one prefill sequence: rows [p_row0, p_row0 + p_len) at positions [p_pos0, ...)
    int p_row0 = 0, p_len = 0, p_pos0 = 0, p_bt = 0;
    // flat block table (all sequences)
    std::vector<int> bt;
    // greedy sampling
    std::vector<int> s_row, s_rid;
    std::vector<long long> s_out;

    int rows() const { return static_cast<int>(row_rid.size()); }
    void clear();
    // helpers used by the executor
    int add_table(const std::vector<int32_t>& blocks, long long n_tokens);
    void add_decode(int rid, long long ctx, const std::vector<int32_t>& blocks, long long out_index);
    void add_prefill(int rid, long long pos0, long long len, const std::vector<int32_t>& blocks, bool sample,
                     long long out_index);
    void plan_decode(int n_kv_heads, int slots);
};

// Kernel-time accounting (CUDA events around selected launches, on the launching stream).
struct KernelStat {
    long long launches = 0;
    double ms = 0.0;
    double bytes = 0.0;  // algorithmic bytes
    double flops = 0.0;  // algorithmic flops
};

// Per-worker scratch + metadata staging, sized for `max_rows` rows per pass.
class Worker {
  public:
    Worker(const Weights& w, int max_rows, int max_sample, int max_blocks_per_pass, cudaStream_t stream,
           int max_ctas);
    ~Worker();
    Worker(const Worker&) = delete;
    Worker& operator=(const Worker&) = delete;

    // Enqueue one forward pass on this worker's stream.
    //   pool:      the worker's KV pool
    //   prompt / prompt_off / last_tok / out_tok: request token buffers on this device
    void forward(const Batch& b, const KvPool& pool, const int* prompt, const long long* prompt_off, int* last_tok,
                 int* out_tok);

    int max_rows() const { return max_rows_; }
    cudaStream_t stream() const { return stream_; }
    void set_profiling(bool on) { profile_ = on; }
    // Test hook: sampled rows' logits are also stored at logits_out[out_index * vocab]
    // (device buffer; nullptr = off). Passes with it set are never graph-captured.
    void set_logits_out(float* p) { logits_out_ = p; }
    // Switch the stream / persistent-grid cap later passes launch on (SM lending). The
    // caller orders the streams.
    void set_launch(cudaStream_t s, int max_ctas, cudaStream_t side = nullptr) {
        stream_ = s;
        max_ctas_ = max_ctas;
        side_ = side;
    }
    void collect_stats();  // fold finished profiling events into stats (synchronizes)
    // Drop captured pass graphs (their pointers: the run's token buffers, pools, streams).
    void reset_graphs();
    void reset_stats() {
        stat_decode_attn = stat_prefill_attn = stat_gemm_stream = stat_gemm_tc = stat_other = stat_forward = {};
    }
    // gemm_stream: M <= 128 (weight-streaming, HBM bound); gemm_tc: M > 128 (tensor bound)
    KernelStat stat_decode_attn, stat_prefill_attn, stat_gemm_stream, stat_gemm_tc, stat_other, stat_forward;
    long long launches = 0;  // our kernels launched (always counted)

  private:
    const Weights& w_;
    const ModelSpec& m_;
    int max_rows_, max_sample_, max_bt_;
    cudaStream_t stream_;
    int max_ctas_;
    // Second stream on the same SMs: a mixed pass runs its chunk's prefill attention there,
    // concurrently with the decode attention (independent rows); null = serial.
    cudaStream_t side_ = nullptr;
    cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
    // device activations
    float* x_ = nullptr;
    void* h_ = nullptr;
    float* qkv_ = nullptr;
    void* q_ = nullptr;
    void* attn_ = nullptr;
    float* gu_ = nullptr;
    void* act_ = nullptr;
    void* hs_ = nullptr;
    float* logits_ = nullptr;
    float* attn_ws_ = nullptr;
    long long attn_ws_floats_ = 0;
    int* attn_tickets_ = nullptr;  // split-merge tickets, [max_rows * n_kv_heads], self-resetting
    float* pf_ws_ = nullptr;       // prefill attention piece partials (ck_attn_prefill_ws_floats(kPfSlots))
    int* pf_tickets_ = nullptr;    // [kPfSlots], self-resetting
    static constexpr int kPfSlots = 160;  // >= SMs of any partition (B200: 148)
    // Leading rows of the qkv / gu fp32 accumulators that may be non-zero (left by a
    // tensor-regime pass, which stores instead of red.adding); the weight-streaming
    // regime needs them zero and its consumers re-zero what they read.
    int qkv_dirty_rows_ = 0, gu_dirty_rows_ = 0;
    int* tile_tickets_ = nullptr;  // fused-epilogue tile tickets (self-resetting)
    int* norm_tickets_ = nullptr;  // fused-RMSNorm m-tile tickets (self-resetting)
    float* arg_ws_ = nullptr;      // argmax slice winners [max_sample * 64]
    int* arg_tickets_ = nullptr;   // [max_sample], self-resetting
    float* logits_out_ = nullptr;  // logits test hook (set_logits_out)
    int* meta_dev_ = nullptr;
    long long meta_cap_ = 0;
    // pinned staging ring for per-pass metadata
    static constexpr int kRing = 8;
    int* meta_host_[kRing] = {};
    cudaEvent_t meta_ev_[kRing] = {};
    int ring_ = 0;
    // profiling
    bool profile_ = false;
    struct Pending {
        cudaEvent_t a, b;
        KernelStat* into;
        double bytes, flops;
    };
    std::vector<Pending> pending_;
    std::vector<cudaEvent_t> ev_free_;
    cudaEvent_t ev();
    void mark(cudaEvent_t& a);
    void done(cudaEvent_t a, KernelStat* into, double bytes, double flops);
    // decode-pass CUDA graphs, keyed by the pass shape and the pointers its kernels take
    struct Tally {
        KernelStat* into;
        double bytes, flops;
    };
    struct GraphEntry {
        cudaGraphExec_t exec;
        long long kernels;           // launches one replay stands for
        std::vector<Tally> tallies;  // the stat updates one replay stands for
    };
    std::vector<Tally>* tally_rec_ = nullptr;
    std::map<std::string, GraphEntry> graphs_;
    std::map<std::string, int> graph_seen_;  // shape -> plain (uncaptured) runs so far
    long long graph_hits_ = 0;
    void gemm(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int epi, int splits,
              const ck_gemm_fuse* fuse = nullptr);
};

// Resident decode-attention CTAs per SM the cluster planner assumes (CRONUS_DEC_SLOTS_PER_SM; default 0 = auto).
int decode_slots_per_sm();
// Resident-CTA budget handed to the decode planner for n_seq sequences on `sms` SMs.
int decode_slots(int n_kv_heads, int n_seq, int sms);

void check_cuda(cudaError_t e, const char* what);
void check_ck(int rc, const char* what);

}  // namespace gpu
}  // namespace cronus
