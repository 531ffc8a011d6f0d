// Decoder forward orchestration over the C-ABI kernels (see model.hpp).
#include "model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "cronus_ck.h"

namespace cronus {
namespace gpu {

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void check_ck(int rc, const char* what) {
    if (rc != 0)
        throw std::runtime_error(std::string("kernel ") + what + " failed: " +
                                 cudaGetErrorString(static_cast<cudaError_t>(rc)));
}

// ------------------------------------------------------------------ ModelSpec
ModelSpec ModelSpec::preset(const std::string& name) {
    ModelSpec m;
    m.name = name;
    if (name == "llama3-8b") {
        m.hidden = 4096, m.layers = 32, m.n_heads = 32, m.n_kv_heads = 8, m.ffn = 14336, m.vocab = 128256;
        m.rope_theta = 500000.0, m.rms_eps = 1e-5f, m.qkv_bias = false;
    } else if (name == "qwen2-7b") {
        m.hidden = 3584, m.layers = 28, m.n_heads = 28, m.n_kv_heads = 4, m.ffn = 18944, m.vocab = 152064;
        m.rope_theta = 1000000.0, m.rms_eps = 1e-6f, m.qkv_bias = true;
    } else if (name == "tiny") {
        m.hidden = 256, m.layers = 2, m.n_heads = 2, m.n_kv_heads = 1, m.ffn = 1024, m.vocab = 4096;
        m.rope_theta = 10000.0, m.rms_eps = 1e-5f, m.qkv_bias = false;
        m.lm_std = 0.25f;
        m.max_pos = 16384;
    } else if (name == "tiny-qwen") {  // tiny with the Qwen2 QKV bias and GQA group 2
        m.hidden = 512, m.layers = 2, m.n_heads = 4, m.n_kv_heads = 2, m.ffn = 1024, m.vocab = 4096;
        m.rope_theta = 1000000.0, m.rms_eps = 1e-6f, m.qkv_bias = true;
        m.lm_std = 0.25f;
        m.max_pos = 16384;
    } else {
        throw std::invalid_argument("unknown model preset '" + name + "' (llama3-8b, qwen2-7b, tiny, tiny-qwen)");
    }
    if (m.hidden % 128 || m.ffn % 64 || m.vocab % 128 || m.n_heads % m.n_kv_heads)
        throw std::invalid_argument("model shape not supported by the sm_100a kernels");
    return m;
}

double ModelSpec::linear_flops_per_token() const {
    const double H = hidden;
    const double per_layer = H * qkv_n() + static_cast<double>(q_n()) * H + H * 2.0 * ffn + 1.0 * ffn * H;
    return 2.0 * per_layer * layers;
}

long long ModelSpec::weight_bytes() const {
    const long long H = hidden;
    long long per_layer = H * qkv_n() + static_cast<long long>(q_n()) * H + H * 2LL * ffn + 1LL * ffn * H + 2 * H;
    if (qkv_bias) per_layer += qkv_n();
    return 2LL * (per_layer * layers + 2LL * vocab * H + H);
}

// ------------------------------------------------------------------ Weights
namespace {
size_t align256(size_t v) { return (v + 255) & ~size_t(255); }
constexpr float kSqrt3 = 1.7320508075688772f;
}  // namespace

Weights::Weights(const ModelSpec& spec, int device) : spec_(spec), dev_(device) {
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    const ModelSpec& m = spec_;
    const long long H = m.hidden;
    struct Item {
        void** dst;
        long long n;
        uint64_t tid;
        float scale, offset;
    };
    std::vector<Item> items;
    layer.resize(m.layers);
    items.push_back({&embed, static_cast<long long>(m.vocab) * H, kTidEmbed, m.emb_std * kSqrt3, 0.f});
    items.push_back({&lm_head, static_cast<long long>(m.vocab) * H, kTidLmHead, m.lm_std * kSqrt3, 0.f});
    items.push_back({&final_norm, H, kTidFinalNorm, 0.1f, 1.0f});
    for (int l = 0; l < m.layers; ++l) {
        LayerWeights& L = layer[l];
        items.push_back({&L.wqkv, static_cast<long long>(m.qkv_n()) * H, layer_tid(l, kWqkv), m.w_std * kSqrt3, 0.f});
        if (m.qkv_bias) items.push_back({&L.bqkv, m.qkv_n(), layer_tid(l, kBqkv), 0.1f, 0.f});
        items.push_back({&L.wo, H * m.q_n(), layer_tid(l, kWo), m.w_std * kSqrt3, 0.f});
        items.push_back({&L.wgu, 2LL * m.ffn * H, layer_tid(l, kWgu), m.w_std * kSqrt3, 0.f});
        items.push_back({&L.wd, H * m.ffn, layer_tid(l, kWd), m.w_std * kSqrt3, 0.f});
        items.push_back({&L.attn_norm, H, layer_tid(l, kAttnNorm), 0.1f, 1.0f});
        items.push_back({&L.ffn_norm, H, layer_tid(l, kFfnNorm), 0.1f, 1.0f});
    }
    size_t total = 0;
    std::vector<size_t> off;
    for (const Item& it : items) {
        off.push_back(total);
        total += align256(static_cast<size_t>(it.n) * 2);
    }
    const size_t rope = align256(static_cast<size_t>(m.max_pos) * 64 * 4);
    check_cuda(cudaMalloc(&base_, total + 2 * rope), "cudaMalloc(weights)");
    char* b = static_cast<char*>(base_);
    for (size_t i = 0; i < items.size(); ++i) {
        *items[i].dst = b + off[i];
        check_ck(ck_init_uniform(*items[i].dst, items[i].n, m.seed, items[i].tid, items[i].scale, items[i].offset,
                                 nullptr),
                 "init_uniform");
    }
    cos_tab = reinterpret_cast<float*>(b + total);
    sin_tab = reinterpret_cast<float*>(b + total + rope);
    check_ck(ck_rope_table(cos_tab, sin_tab, m.max_pos, m.rope_theta, nullptr), "rope_table");
    check_cuda(cudaDeviceSynchronize(), "weights init");
}

Weights::~Weights() {
    if (base_) {
        cudaSetDevice(dev_);
        cudaFree(base_);
    }
}

KvPool::KvPool(int dev, long long n_blocks, long long bb) : device(dev), blocks(n_blocks), block_bytes(bb) {
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    check_cuda(cudaMalloc(&base, static_cast<size_t>(n_blocks) * bb), "cudaMalloc(kv pool)");
    // Never-written slots must hold finite values: the tensor-core attention reads whole
    // 16-token blocks and masks the tail (0 * NaN would poison the P.V product).
    check_cuda(cudaMemset(base, 0, static_cast<size_t>(n_blocks) * bb), "zero kv pool");
}

KvPool::~KvPool() {
    if (base) {
        cudaSetDevice(device);
        cudaFree(base);
    }
}

// ------------------------------------------------------------------ Batch
void Batch::clear() {
    row_rid.clear(), row_pos.clear(), row_dec.clear(), row_bt.clear();
    d_row.clear(), d_len.clear(), d_bt.clear(), d_item0.clear(), d_work.clear();
    p_row0 = p_len = p_pos0 = p_bt = 0;
    bt.clear();
    s_row.clear(), s_rid.clear(), s_out.clear();
}

int Batch::add_table(const std::vector<int32_t>& blocks, long long n_tokens) {
    const int off = static_cast<int>(bt.size());
    const long long nb = (n_tokens + 15) / 16;
    if (static_cast<long long>(blocks.size()) < nb) throw std::logic_error("block table shorter than the sequence");
    bt.insert(bt.end(), blocks.begin(), blocks.begin() + nb);
    return off;
}

void Batch::add_decode(int rid, long long ctx, const std::vector<int32_t>& blocks, long long out_index) {
    const int row = rows();
    const int off = add_table(blocks, ctx);
    row_rid.push_back(rid);
    row_pos.push_back(static_cast<int>(ctx - 1));
    row_dec.push_back(1);
    row_bt.push_back(off);
    d_row.push_back(row);
    d_len.push_back(static_cast<int>(ctx));
    d_bt.push_back(off);
    s_row.push_back(row);
    s_rid.push_back(rid);
    s_out.push_back(out_index);
}

void Batch::add_prefill(int rid, long long pos0, long long len, const std::vector<int32_t>& blocks, bool sample,
                        long long out_index) {
    const int off = add_table(blocks, pos0 + len);
    p_row0 = rows();
    p_len = static_cast<int>(len);
    p_pos0 = static_cast<int>(pos0);
    p_bt = off;
    for (long long i = 0; i < len; ++i) {
        row_rid.push_back(rid);
        row_pos.push_back(static_cast<int>(pos0 + i));
        row_dec.push_back(0);
        row_bt.push_back(off);
    }
    if (sample) {
        s_row.push_back(p_row0 + p_len - 1);
        s_rid.push_back(rid);
        s_out.push_back(out_index);
    }
}

// Predicted makespan (in block-streaming times of one CTA) of a decode launch whose
// sequences are cut into parts of at most `cap` blocks: list scheduling of the parts,
// heaviest first, on slots / (nkv * C) item slots; each CTA pays a fixed setup cost and
// a part of a cut sequence the global merge.
static double decode_makespan(const std::vector<int>& d_len, long long cap, int C, long long item_slots,
                              std::vector<double>& heap) {
    // blocks-equivalent (~0.5 us per block per CTA); a global part merge measured ~6-8 us (2 x 2142
    // keys on 148 SMs: 2 parts 18.1 us, whole 10.7 us; round 1 assumed 4 blocks)
    constexpr double kSetup = 6.0, kMerge = 12.0;
    std::vector<double> work;
    work.reserve(d_len.size() * 2);
    for (int len : d_len) {
        const long long nblk = (len + 15) / 16;
        const long long parts = std::max<long long>(1, (nblk + cap - 1) / cap);
        const double w = static_cast<double>((nblk + parts - 1) / parts) / C + kSetup + (parts > 1 ? kMerge : 0.0);
        for (long long i = 0; i < parts; ++i) work.push_back(w);
    }
    std::sort(work.begin(), work.end(), std::greater<double>());
    heap.assign(static_cast<size_t>(std::max<long long>(1, item_slots)), 0.0);  // min-heap of slot finish times
    for (double w : work) {
        std::pop_heap(heap.begin(), heap.end(), std::greater<double>());
        heap.back() += w;
        std::push_heap(heap.begin(), heap.end(), std::greater<double>());
    }
    return *std::max_element(heap.begin(), heap.end());
}

void Batch::plan_decode(int n_kv_heads, int slots) {
    // Resident CTAs `slots`: every (sequence, kv head) pair gets a cluster of C CTAs (C =
    // power of two <= 16, as large as one wave allows while each CTA keeps >= 4 blocks, one
    // per warp). Sequences longer than `cap` blocks are cut into parts (merged through the
    // global ticket path); cap is the candidate with the shortest predicted makespan
    // (decode_makespan), and the work list runs the heaviest parts first (LPT): with the
    // lognormal context lengths of a serve, one 8k-token sequence left whole (or started
    // last) would otherwise hold the whole launch for 2-3x its fair time.
    const long long n = static_cast<long long>(d_len.size());
    long long total = 0, longest = 0;
    for (int len : d_len) {
        total += (len + 15) / 16;
        longest = std::max<long long>(longest, (len + 15) / 16);
    }
    const long long pairs = n * n_kv_heads;
    int C = 1;
    while (C < 16 && pairs * C * 2 <= slots && total * n_kv_heads >= pairs * C * 2 * 4) C *= 2;
    const long long share = std::max<long long>(8, (total * n_kv_heads + slots - 1) / std::max(1, slots));
    const long long min_cap = std::max<long long>(8, (longest + 254) / 255);  // work[] holds <= 255 parts
    // Candidates whose CTAs fit one wave win over any that need a second one: the block-unit
    // makespan treats every resident cluster as running at a fixed per-block rate, but a second
    // wave of an HBM-bound kernel shares the same bandwidth and adds its latency tail (16 x 2048
    // on 148 SMs: 3 parts -> 768 CTAs 44.9 us, whole sequences 26 us). 16-CTA clusters (one GPC
    // each) count against half the slots: 16 of them on 148 SMs run in two rounds (1 x 2142:
    // 2 parts 19.8 us, 1 part 10.1 us); a plan that needs more falls back to 8-CTA clusters
    // (1 x 8192: 25.1 -> 18.7 us). profiles/r2_session5/dec_small.txt, dec_cluster.txt.
    long long cap = 0;
    for (;;) {
        const long long item_slots = std::max<long long>(1, slots / (static_cast<long long>(n_kv_heads) * C));
        const long long wave = C >= 16 ? slots / 2 : slots;
        auto ctas_for = [&](long long c) {
            long long k = 0;
            for (int len : d_len) k += std::max<long long>(1, ((len + 15) / 16 + c - 1) / c);
            return k * n_kv_heads * C;
        };
        // candidates: no split, and the round-1 cap scaled by 2, 1.5, 1, 0.75, 0.5 (ties keep the
        // larger cap: fewer merges); a one-wave candidate wins unless its makespan is more than
        // 1.5x the best (an unsplit long sequence in a small batch must still be cut)
        const double fs[6] = {0.0, 2.0, 1.5, 1.0, 0.75, 0.5};
        long long caps[6];
        double ts[6];
        bool fit[6];
        double t_min = 1e300;
        for (int i = 0; i < 6; ++i) {
            caps[i] = fs[i] == 0.0 ? std::max(min_cap, longest) : std::max(min_cap, static_cast<long long>(fs[i] * share * C));
            ts[i] = decode_makespan(d_len, caps[i], C, item_slots, plan_heap_);
            fit[i] = ctas_for(caps[i]) <= wave;
            t_min = std::min(t_min, ts[i]);
        }
        int pick = -1;
        for (int i = 0; i < 6; ++i)
            if (fit[i] && ts[i] <= 1.5 * t_min && (pick < 0 || ts[i] < ts[pick] - 1e-9)) pick = i;
        const bool best_fits = pick >= 0;
        if (!best_fits)
            for (int i = 1; i < 6; ++i)
                if (pick < 0 || ts[i] < ts[pick] - 1e-9) pick = i;
        cap = caps[pick];
        if (best_fits || C < 16) break;
        C = 8;
    }
    decode_cluster = C;
    std::vector<std::pair<long long, int>> order;  // (blocks per part, sequence)
    std::vector<int> parts_of(d_len.size());
    for (size_t s = 0; s < d_len.size(); ++s) {
        const long long nblk = (d_len[s] + 15) / 16;
        const long long parts = std::max<long long>(1, (nblk + cap - 1) / cap);
        parts_of[s] = static_cast<int>(parts);
        order.emplace_back((nblk + parts - 1) / parts, static_cast<int>(s));
    }
    std::stable_sort(order.begin(), order.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    d_item0.assign(d_len.size(), 0);
    d_work.clear();
    for (const auto& [bpp, s] : order) {
        d_item0[s] = static_cast<int>(d_work.size());
        for (int i = 0; i < parts_of[s]; ++i) d_work.push_back((s << 16) | (parts_of[s] << 8) | i);
    }
    blocks_per_split = static_cast<int>(cap);
}

// Mixed passes: the chunk's prefill attention runs on the worker's side stream, concurrent with
// the decode attention, on this fraction of the worker's SMs (CRONUS_ATTN_OVERLAP; 0 = serial).
double attn_overlap_frac() {
    static const double f = [] {
        const char* e = std::getenv("CRONUS_ATTN_OVERLAP");
        return e ? std::atof(e) : 0.25;
    }();
    return f;
}

// Tensor-regime gate_up: hybrid whole-tile / stream-K-tail SiLU GEMM (CRONUS_SILU_HYBRID=0: whole tiles only).
bool silu_hybrid() {
    static const bool on = [] {
        const char* e = std::getenv("CRONUS_SILU_HYBRID");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Weight-streaming passes of at most this many rows (CRONUS_NORM_FUSE_ROWS, default 0 = off)
// run the ffn norm inside the O GEMM and the next layer's attention norm inside the down
// GEMM (CK_FUSE_RMSNORM: the m-tile's last finished tile normalizes the rows): two
// dependent launches fewer per layer. Measured slower on B200 (8 x 2048 decode pass 4.43 ->
// 5.24 ms, ~1.2 us per row): one CTA's load -> reduce -> store chain per row pair costs
// more than the kernel boundary it removes.
int norm_fuse_rows() {
    static const int n = [] {
        const char* e = std::getenv("CRONUS_NORM_FUSE_ROWS");
        return e ? std::atoi(e) : 0;
    }();
    return n;
}

// Weight-streaming passes of at most this many rows (CRONUS_SILU_FUSE_ROWS, default 0 = off)
// run SiLU(gate) * up in the gate_up GEMM's ticketed tile finalize instead of its own kernel.
int silu_fuse_rows() {
    static const int n = [] {
        const char* e = std::getenv("CRONUS_SILU_FUSE_ROWS");
        return e ? std::atoi(e) : 0;
    }();
    return n;
}

// Weight-streaming passes of at least this many rows (CRONUS_SILU_HYBRID_ROWS, 0 = off) run
// gate_up as the hybrid whole-tile SiLU-epilogue GEMM instead of stream-K + the SiLU kernel.
int silu_hybrid_rows() {
    static const int n = [] {
        const char* e = std::getenv("CRONUS_SILU_HYBRID_ROWS");
        return e ? std::atoi(e) : 0;
    }();
    return n;
}

// Tensor-regime QKV as a stream-K red.add GEMM (CRONUS_QKV_STREAMK=0: whole-tile stores).
bool qkv_streamk() {
    static const bool on = [] {
        const char* e = std::getenv("CRONUS_QKV_STREAMK");
        return !(e && e[0] == '0');
    }();
    return on;
}

// CRONUS_GRAPH_MIN_SEEN (default 24): a decode shape is captured on its N-th sighting, so
// shapes a serve meets only a few times never pay the capture + instantiate cost. Bench serve
// on B200 (req/s, graphs off = 1.000): N = 2 +0.1 %, 8 +0.2 %, 24 +0.45 %, 48 +0.25 %, 96 +0.1 %
// (a serve meets ~105 decode shapes; at 24, 19 of them are captured and replayed ~1050 times).
int graph_min_seen() {
    static const int n = [] {
        const char* e = std::getenv("CRONUS_GRAPH_MIN_SEEN");
        return e ? std::max(2, std::atoi(e)) : 24;
    }();
    return n;
}

// Decode-only passes replay captured CUDA graphs (CRONUS_GRAPHS=0: always issue on the
// stream). A graph replay saves ~0.6 us per dependent boundary (passes 1.5-3 % faster);
// capturing every shape on its second sighting cost about what it saved, hence the
// capture threshold above.
bool use_graphs() {
    static const bool on = [] {
        const char* e = std::getenv("CRONUS_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}

// Decode-only passes fuse RoPE + KV append into the decode attention unless
// CRONUS_DECODE_ROPE_KERNEL=1 (separate qkv_rope_append kernel, for comparison).
bool decode_rope_kernel() {
    static const bool on = [] {
        const char* e = std::getenv("CRONUS_DECODE_ROPE_KERNEL");
        return e && e[0] == '1';
    }();
    return on;
}

int decode_slots_per_sm() {
    static const int n = [] {
        const char* e = std::getenv("CRONUS_DEC_SLOTS_PER_SM");
        const int x = e ? std::atoi(e) : 0;
        return x >= 0 && x <= 4 ? x : 0;  // 0: auto (decode_slots)
    }();
    return n;
}

// Auto (default): plan for 3 resident CTAs per SM once a pass has >= 64 (sequence, kv head)
// pairs — larger clusters, and the kernel layer's 2-stage ring then fits the grid in one wave —
// else 2. Measured (run32.sh): 8 x 2048 decode pass 4.43 -> 4.38 ms, 16 x 2048 4.88 -> 4.79,
// 1-4 and 24-32 sequences unchanged; serve 15.215 / 15.241 -> 15.434 / 15.426 req/s (+1.3 %).
// A flat 3 per SM slowed 4 x 2048 (cluster 8 on 2-stage rings: 4.17 -> 4.37 ms).
int decode_slots(int n_kv_heads, int n_seq, int sms) {
    const int per = decode_slots_per_sm();
    if (per > 0) return per * sms;
    return (static_cast<long long>(n_seq) * n_kv_heads >= 64 ? 3 : 2) * sms;
}

// ------------------------------------------------------------------ Worker
Worker::Worker(const Weights& w, int max_rows, int max_sample, int max_blocks_per_pass, cudaStream_t stream,
               int max_ctas)
    : w_(w), m_(w.spec()), max_rows_(max_rows), max_sample_(max_sample), max_bt_(max_blocks_per_pass),
      stream_(stream), max_ctas_(max_ctas) {
    check_cuda(cudaSetDevice(w.device()), "cudaSetDevice");
    const size_t R = max_rows, H = m_.hidden;
    check_cuda(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming), "event");
    check_cuda(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming), "event");
    check_cuda(cudaMalloc(&x_, R * H * 4), "alloc x");
    check_cuda(cudaMalloc(&h_, R * H * 2), "alloc h");
    check_cuda(cudaMalloc(&qkv_, R * m_.qkv_n() * 4), "alloc qkv");
    check_cuda(cudaMalloc(&q_, R * m_.q_n() * 2), "alloc q");
    check_cuda(cudaMalloc(&attn_, R * m_.q_n() * 2), "alloc attn");
    check_cuda(cudaMalloc(&gu_, R * 2 * m_.ffn * 4), "alloc gu");
    check_cuda(cudaMemset(qkv_, 0, R * m_.qkv_n() * 4), "zero qkv");
    check_cuda(cudaMemset(gu_, 0, R * 2 * m_.ffn * 4), "zero gu");
    check_cuda(cudaMalloc(&act_, R * m_.ffn * 2), "alloc act");
    check_cuda(cudaMalloc(&hs_, static_cast<size_t>(max_sample) * H * 2), "alloc hs");
    check_cuda(cudaMalloc(&logits_, static_cast<size_t>(max_sample) * m_.vocab * 4), "alloc logits");
    check_cuda(cudaMemset(logits_, 0, static_cast<size_t>(max_sample) * m_.vocab * 4), "zero logits");
    attn_ws_floats_ = 4096LL * m_.n_heads * (m_.head_dim + 2);
    check_cuda(cudaMalloc(&attn_ws_, attn_ws_floats_ * 4), "alloc attn ws");
    check_cuda(cudaMalloc(&attn_tickets_, R * m_.n_kv_heads * 4), "alloc attn tickets");
    check_cuda(cudaMemset(attn_tickets_, 0, R * m_.n_kv_heads * 4), "zero attn tickets");
    check_cuda(cudaMalloc(&pf_ws_, static_cast<size_t>(ck_attn_prefill_ws_floats(kPfSlots)) * 4), "alloc prefill ws");
    check_cuda(cudaMalloc(&pf_tickets_, kPfSlots * 4), "alloc prefill tickets");
    check_cuda(cudaMemset(pf_tickets_, 0, kPfSlots * 4), "zero prefill tickets");
    const size_t n_tiles = static_cast<size_t>(std::max(2 * m_.ffn, m_.qkv_n()) / 128) * ((R + 31) / 32);
    check_cuda(cudaMalloc(&tile_tickets_, n_tiles * 4), "alloc tile tickets");
    check_cuda(cudaMemset(tile_tickets_, 0, n_tiles * 4), "zero tile tickets");
    check_cuda(cudaMalloc(&norm_tickets_, 64 * 4), "alloc norm tickets");
    check_cuda(cudaMemset(norm_tickets_, 0, 64 * 4), "zero norm tickets");
    check_cuda(cudaMalloc(&arg_ws_, static_cast<size_t>(max_sample) * 64 * 4), "alloc argmax ws");
    check_cuda(cudaMalloc(&arg_tickets_, static_cast<size_t>(max_sample) * 4), "alloc argmax tickets");
    check_cuda(cudaMemset(arg_tickets_, 0, static_cast<size_t>(max_sample) * 4), "zero argmax tickets");
    meta_cap_ = 12LL * max_rows + max_bt_ + 2 * 4096 + 64;
    check_cuda(cudaMalloc(&meta_dev_, meta_cap_ * 4), "alloc meta");
    for (int i = 0; i < kRing; ++i) {
        check_cuda(cudaMallocHost(&meta_host_[i], meta_cap_ * 4), "alloc pinned meta");
        check_cuda(cudaEventCreateWithFlags(&meta_ev_[i], cudaEventDisableTiming), "event");
    }
}

Worker::~Worker() {
    cudaSetDevice(w_.device());
    reset_graphs();
    for (void* p : {static_cast<void*>(x_), h_, static_cast<void*>(qkv_), q_, attn_, static_cast<void*>(gu_), act_, hs_,
                    static_cast<void*>(logits_), static_cast<void*>(attn_ws_), static_cast<void*>(meta_dev_),
                    static_cast<void*>(attn_tickets_), static_cast<void*>(arg_ws_), static_cast<void*>(arg_tickets_),
                    static_cast<void*>(tile_tickets_), static_cast<void*>(norm_tickets_), static_cast<void*>(pf_ws_),
                    static_cast<void*>(pf_tickets_)})
        if (p) cudaFree(p);
    for (int i = 0; i < kRing; ++i) {
        if (meta_host_[i]) cudaFreeHost(meta_host_[i]);
        if (meta_ev_[i]) cudaEventDestroy(meta_ev_[i]);
    }
    for (auto& p : pending_) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (cudaEvent_t e : ev_free_) cudaEventDestroy(e);
    if (fork_ev_) cudaEventDestroy(fork_ev_);
    if (join_ev_) cudaEventDestroy(join_ev_);
}

cudaEvent_t Worker::ev() {
    if (!ev_free_.empty()) {
        cudaEvent_t e = ev_free_.back();
        ev_free_.pop_back();
        return e;
    }
    cudaEvent_t e;
    check_cuda(cudaEventCreate(&e), "event");
    return e;
}
void Worker::mark(cudaEvent_t& a) {
    if (!profile_) return;
    a = ev();
    cudaEventRecord(a, stream_);
}
void Worker::done(cudaEvent_t a, KernelStat* into, double bytes, double flops) {
    if (!profile_) {  // launches and algorithmic work are always tallied (no events, no timing)
        if (tally_rec_) {
            tally_rec_->push_back({into, bytes, flops});
            static const bool dbg = std::getenv("CRONUS_GRAPH_STATS") != nullptr;
            cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
            if (dbg && cudaStreamIsCapturing(stream_, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusInvalidated)
                std::fprintf(stderr, "[graphs] capture invalidated by launch %zu\n", tally_rec_->size());
        }
        into->launches++;
        into->bytes += bytes;
        into->flops += flops;
        return;
    }
    cudaEvent_t b = ev();
    cudaEventRecord(b, stream_);
    pending_.push_back({a, b, into, bytes, flops});
}

void Worker::reset_graphs() {
    if (std::getenv("CRONUS_GRAPH_STATS") && (graph_hits_ || !graph_seen_.empty()))
        std::fprintf(stderr, "[graphs] shapes %zu captured %zu replays %lld\n", graph_seen_.size(), graphs_.size(),
                     graph_hits_);
    graph_hits_ = 0;
    for (auto& kv : graphs_) cudaGraphExecDestroy(kv.second.exec);
    graphs_.clear();
    graph_seen_.clear();
}

void Worker::collect_stats() {
    for (auto& p : pending_) {
        cudaEventSynchronize(p.b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.a, p.b);
        p.into->launches++;
        p.into->ms += ms;
        p.into->bytes += p.bytes;
        p.into->flops += p.flops;
        ev_free_.push_back(p.a);
        ev_free_.push_back(p.b);
    }
    pending_.clear();
}

void Worker::gemm(const void* W, const void* X, void* out, const void* bias, int M, int N, int K, int epi,
                  int splits, const ck_gemm_fuse* fuse) {
    cudaEvent_t a = nullptr;
    mark(a);
    check_ck(ck_gemm_fused(W, X, out, bias, M, N, K, epi, splits, max_ctas_, fuse, stream_), "gemm");
    ++launches;
    // algorithmic bytes: weights + activations in + output (red.add counted once)
    done(a, M <= 128 ? &stat_gemm_stream : &stat_gemm_tc,
         2.0 * (static_cast<double>(N) * K + static_cast<double>(M) * K) +
             (epi == CK_EPI_BF16 ? 2.0 : epi == CK_EPI_SILU_BF16 ? 1.0 : 4.0) * M * N,
         2.0 * M * N * K);
}

namespace {
// CRONUS_FUSE_EPILOGUE=1: RoPE/KV-append and SiLU*up run inside the QKV / gate_up GEMMs
// (ticketed tile finalize). Measured slower than the separate kernels (the finalize
// sits on the GEMM's critical tail), so off by default.
bool fuse_epilogue() {
    static const bool on = [] {
        const char* e = std::getenv("CRONUS_FUSE_EPILOGUE");
        return e && e[0] == '1';
    }();
    return on;
}

template <class T>
T* carve(int*& cur, size_t n) {
    uintptr_t p = reinterpret_cast<uintptr_t>(cur);
    p = (p + alignof(T) - 1) & ~(uintptr_t)(alignof(T) - 1);
    T* out = reinterpret_cast<T*>(p);
    cur = reinterpret_cast<int*>(out + n);
    return out;
}
}  // namespace

void Worker::forward(const Batch& b, const KvPool& pool, const int* prompt, const long long* prompt_off,
                     int* last_tok, int* out_tok) {
    const int M = b.rows();
    if (M == 0) return;
    if (M > max_rows_) throw std::logic_error("forward: batch exceeds worker rows");
    const int R = static_cast<int>(b.s_row.size());
    if (R > max_sample_) throw std::logic_error("forward: too many sampled rows");
    const ModelSpec& m = m_;
    cudaEvent_t pass0 = nullptr;
    mark(pass0);

    // ---- metadata: one pinned staging slot -> one H2D copy
    const int slot = ring_;
    ring_ = (ring_ + 1) % kRing;
    check_cuda(cudaEventSynchronize(meta_ev_[slot]), "meta staging");
    int* host = meta_host_[slot];
    int* cur_h = host;
    auto put = [&](const auto& v) {
        using T = typename std::decay_t<decltype(v)>::value_type;
        T* dst = carve<T>(cur_h, v.size());
        if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
        return static_cast<long long>(reinterpret_cast<char*>(dst) - reinterpret_cast<char*>(host));
    };
    // arrays sized by the pass shape first, the block table (grows with context) last: every
    // device pointer below is then a function of the shape only (CUDA-graph replay key)
    const long long o_row_rid = put(b.row_rid), o_row_pos = put(b.row_pos), o_row_dec = put(b.row_dec),
                    o_row_bt = put(b.row_bt), o_d_row = put(b.d_row), o_d_len = put(b.d_len), o_d_bt = put(b.d_bt),
                    o_d_item0 = put(b.d_item0), o_d_work = put(b.d_work), o_s_row = put(b.s_row),
                    o_s_rid = put(b.s_rid), o_s_out = put(b.s_out), o_bt = put(b.bt);
    const size_t bytes = reinterpret_cast<char*>(cur_h) - reinterpret_cast<char*>(host);
    if (bytes > static_cast<size_t>(meta_cap_) * 4) throw std::logic_error("forward: metadata overflow");
    check_cuda(cudaMemcpyAsync(meta_dev_, host, bytes, cudaMemcpyHostToDevice, stream_), "meta H2D");
    check_cuda(cudaEventRecord(meta_ev_[slot], stream_), "meta event");
    char* dbase = reinterpret_cast<char*>(meta_dev_);
    auto D = [&](long long off) { return reinterpret_cast<int*>(dbase + off); };
    const int* row_rid = D(o_row_rid);
    const int* row_pos = D(o_row_pos);
    const int* row_dec = D(o_row_dec);
    const int* row_bt = D(o_row_bt);
    const int* bt = D(o_bt);
    const int n_dec = static_cast<int>(b.d_row.size());
    const int n_work = static_cast<int>(b.d_work.size());
    if (static_cast<long long>(n_work) * m.n_heads * (m.head_dim + 2) > attn_ws_floats_)
        throw std::logic_error("forward: decode work list too long");

    const int H = m.hidden, Q = m.qkv_n(), NQ = m.q_n(), F = m.ffn;
    const bool small = M <= 128;  // weight-streaming regime
    const float scale = 1.0f / std::sqrt(static_cast<float>(m.head_dim));
    long long dec_keys = 0;
    for (int len : b.d_len) dec_keys += len;
    const double kv_tok_layer = 2.0 * m.n_kv_heads * m.head_dim * 2;  // bytes per token per layer (K+V)

    // QKV accumulates with stream-K red.add in the weight-streaming regime, and in the tensor
    // regime when whole 128x256 tiles fill the grid's last wave badly (e.g. 48 N-tiles x 1
    // token tile on 40 SMs: 60 %); the RoPE/append kernel (or, for fused decode RoPE, the
    // next norm) clears the rows it consumed
    bool qkv_red = small;
    if (!small && qkv_streamk() && !fuse_epilogue()) {
        const long long tiles = static_cast<long long>(Q / 128) * ((M + 255) / 256);
        const long long ctas = max_ctas_ > 0 ? max_ctas_ : ck_device_sms();
        qkv_red = tiles < 8 * ctas && tiles * 10 < 8 * ((tiles + ctas - 1) / ctas) * ctas;  // < 80 % last-wave fill
    }
    if (qkv_red) {  // red.add accumulators must start from zero
        if (qkv_dirty_rows_ > 0)
            check_cuda(cudaMemsetAsync(qkv_, 0, static_cast<size_t>(qkv_dirty_rows_) * Q * 4, stream_), "memset qkv");
        qkv_dirty_rows_ = 0;
    } else {
        qkv_dirty_rows_ = std::max(qkv_dirty_rows_, M);
    }
    if (small) {
        if (gu_dirty_rows_ > 0)
            check_cuda(cudaMemsetAsync(gu_, 0, static_cast<size_t>(gu_dirty_rows_) * 2 * F * 4, stream_), "memset gu");
        gu_dirty_rows_ = 0;
    } else if (fuse_epilogue()) {
        gu_dirty_rows_ = std::max(gu_dirty_rows_, M);  // else gate/up go straight to act
    }
    // decode-only weight-streaming pass: RoPE + KV append of the decode tokens run inside
    // the decode attention (reads the fp32 qkv accumulator), one kernel fewer per layer
    const bool fused_rope = small && b.p_len == 0 && n_dec == M && b.decode_cluster > 0 && !fuse_epilogue() &&
                            !decode_rope_kernel();
    const ck_decode_rope rope{qkv_, w_.cos_tab, w_.sin_tab};
    if (fused_rope) qkv_dirty_rows_ = std::max(qkv_dirty_rows_, M);  // the last layer's rows: next pass clears

    const bool norm_fused = small && !fuse_epilogue() && M <= norm_fuse_rows() && H <= 4096 && H % 4 == 0;
    ck_gemm_fuse norm_fuse{};
    norm_fuse.kind = CK_FUSE_RMSNORM;
    norm_fuse.tickets = tile_tickets_;
    norm_fuse.row_tickets = norm_tickets_;
    norm_fuse.norm_out = h_;
    norm_fuse.eps = m.rms_eps;
    // ---- the pass's kernel chain (issued directly, or captured once per shape and replayed)
    auto issue = [&]() {
    cudaEvent_t a = nullptr;
    mark(a);
    check_ck(ck_embed(x_, w_.embed, row_rid, row_pos, row_dec, prompt, prompt_off, last_tok, M, H, stream_), "embed");
    ++launches;
    done(a, &stat_other, 0, 0);
    for (int l = 0; l < m.layers; ++l) {
        const LayerWeights& L = w_.layer[l];
        if (!(norm_fused && l > 0)) {  // else the previous down GEMM wrote h_ (and cleared qkv_)
            mark(a);
            // weight-streaming regime (M <= 128): qkv accumulates with red.add (stream-K GEMM),
            // so the norm kernel clears it; tensor regime: plain fp32 tile stores
            // fused decode RoPE: the attention left the previous layer's qkv rows for this norm to clear
            check_ck(ck_rmsnorm(x_, L.attn_norm, h_, nullptr, M, H, m.rms_eps, fused_rope && l > 0 ? qkv_ : nullptr,
                                Q, stream_),
                     "rmsnorm");
            ++launches;
            done(a, &stat_other, 0, 0);
        }
        // QKV projection with RoPE + KV append fused into its tile finalize
        ck_gemm_fuse fq{};
        fq.kind = CK_FUSE_QKV_ROPE;
        fq.zero_after = small ? 1 : 0;
        fq.tickets = tile_tickets_;
        fq.q_out = q_;
        fq.kv_pool = pool.base;
        fq.bt = bt;
        fq.row_bt = row_bt;
        fq.row_pos = row_pos;
        fq.cos_tab = w_.cos_tab;
        fq.sin_tab = w_.sin_tab;
        fq.nq = m.n_heads, fq.nkv = m.n_kv_heads, fq.layer = l, fq.n_layers = m.layers;
        if (fuse_epilogue()) {
            gemm(L.wqkv, h_, qkv_, L.bqkv, M, Q, H, small ? CK_EPI_RED_F32 : CK_EPI_F32, small ? 0 : 1, &fq);
        } else {
            gemm(L.wqkv, h_, qkv_, L.bqkv, M, Q, H, qkv_red ? CK_EPI_RED_F32 : CK_EPI_F32, qkv_red ? 0 : 1);
        }
        if (!fuse_epilogue() && !fused_rope) {
            mark(a);
            check_ck(ck_qkv_rope_append(qkv_, nullptr, q_, pool.base, bt, row_bt, row_pos, w_.cos_tab, w_.sin_tab, M,
                                        m.n_heads, m.n_kv_heads, l, m.layers, qkv_red ? 1 : 0, stream_),
                     "qkv_rope_append");
            ++launches;
            done(a, &stat_other, 0, 0);
        }
        // mixed pass: the decode attention runs on the side stream (lower priority) while the
        // chunk's prefill attention keeps a CTA budget of the SMs on the main stream; both read
        // the pass's q / KV and write disjoint rows of attn_. The prefill grid is dispatched
        // first (main stream, higher priority): one 231-KB CTA per SM could otherwise never
        // find a free SM among the decode kernel's 2-3 resident CTAs per SM.
        const bool overlap = n_dec > 0 && b.p_len > 0 && side_ != nullptr && !profile_ && attn_overlap_frac() > 0.0;
        if (overlap) {
            check_cuda(cudaEventRecord(fork_ev_, stream_), "fork");
            check_cuda(cudaStreamWaitEvent(side_, fork_ev_, 0), "fork wait");
            check_ck(ck_attn_decode_tma(q_, pool.base, pool.blocks, bt, D(o_d_row), D(o_d_len), D(o_d_bt),
                                        D(o_d_item0), D(o_d_work), n_work, n_dec, b.decode_cluster, attn_ws_,
                                        attn_tickets_, attn_, m.n_heads, m.n_kv_heads, l, m.layers, scale,
                                        fused_rope ? &rope : nullptr, side_),
                     "attn_decode_tma (side)");
            ++launches;
            check_cuda(cudaEventRecord(join_ev_, side_), "join");
            const int all = max_ctas_ > 0 ? max_ctas_ : ck_device_sms();
            const int pf_ctas = std::max(8, std::min(kPfSlots, static_cast<int>(attn_overlap_frac() * all)));
            check_ck(ck_attn_prefill_pp(q_, max_rows_, pool.base, pool.blocks, bt + b.p_bt, b.p_row0, b.p_len,
                                        b.p_pos0, attn_, m.n_heads, m.n_kv_heads, l, m.layers, scale, pf_ws_,
                                        pf_tickets_, pf_ctas, stream_),
                     "attn_prefill");
            ++launches;
            check_cuda(cudaStreamWaitEvent(stream_, join_ev_, 0), "join wait");
        }
        if (n_dec > 0 && !overlap) {
            mark(a);
            check_ck(ck_attn_decode_tma(q_, pool.base, pool.blocks, bt, D(o_d_row), D(o_d_len), D(o_d_bt),
                                            D(o_d_item0), D(o_d_work), n_work, n_dec, b.decode_cluster, attn_ws_,
                                            attn_tickets_, attn_, m.n_heads, m.n_kv_heads, l, m.layers, scale,
                                            fused_rope ? &rope : nullptr, stream_),
                         "attn_decode_tma");
            ++launches;
            done(a, &stat_decode_attn, dec_keys * kv_tok_layer, 4.0 * m.n_heads * m.head_dim * dec_keys);
        }
        if (b.p_len > 0 && !overlap) {
            mark(a);
            const int pf_ctas = std::min(kPfSlots, max_ctas_ > 0 ? max_ctas_ : ck_device_sms());
            check_ck(ck_attn_prefill_pp(q_, max_rows_, pool.base, pool.blocks, bt + b.p_bt, b.p_row0, b.p_len,
                                        b.p_pos0, attn_, m.n_heads, m.n_kv_heads, l, m.layers, scale, pf_ws_,
                                        pf_tickets_, pf_ctas, stream_),
                     "attn_prefill");
            ++launches;
            const double keys = static_cast<double>(b.p_len) * b.p_pos0 + 0.5 * b.p_len * (b.p_len + 1.0);
            done(a, &stat_prefill_attn, (b.p_pos0 + b.p_len) * kv_tok_layer, 4.0 * m.n_heads * m.head_dim * keys);
        }
        if (norm_fused) {
            ck_gemm_fuse fn = norm_fuse;
            fn.gamma = L.ffn_norm;
            gemm(L.wo, attn_, x_, nullptr, M, H, NQ, CK_EPI_RED_F32, 0, &fn);
        } else {
            gemm(L.wo, attn_, x_, nullptr, M, H, NQ, CK_EPI_RED_F32, 0);
            mark(a);
            check_ck(ck_rmsnorm(x_, L.ffn_norm, h_, nullptr, M, H, m.rms_eps, nullptr, 0, stream_), "rmsnorm");
            ++launches;
            done(a, &stat_other, 0, 0);
        }
        // gate/up projection with SiLU(gate) * up fused into its tile finalize
        ck_gemm_fuse fs{};
        fs.kind = CK_FUSE_SILU;
        fs.zero_after = small ? 1 : 0;
        fs.tickets = tile_tickets_;
        fs.act = act_;
        if (fuse_epilogue()) {
            gemm(L.wgu, h_, gu_, nullptr, M, 2 * F, H, small ? CK_EPI_RED_F32 : CK_EPI_F32, small ? 0 : 1, &fs);
        } else if (!small) {
            // tensor regime: whole tiles per CTA -> SiLU(gate) * up straight from TMEM (the
            // fp32 gate/up tensor never reaches HBM); a sparse last wave (e.g. 448 tiles on
            // 148 SMs) runs as stream-K pieces through gu_ + ticketed finalize (hybrid)
            if (silu_hybrid()) {
                ck_gemm_fuse fh{};
                fh.kind = CK_FUSE_SILU;
                fh.zero_after = 1;
                fh.tickets = tile_tickets_;
                fh.act = act_;
                gemm(L.wgu, h_, gu_, nullptr, M, 2 * F, H, CK_EPI_SILU_BF16, 0, &fh);
            } else {
                gemm(L.wgu, h_, act_, nullptr, M, 2 * F, H, CK_EPI_SILU_BF16, 1);
            }
        } else if (silu_hybrid_rows() > 0 && M >= silu_hybrid_rows() && silu_hybrid()) {
            // weight-streaming regime, larger batches: whole weight tiles with the SiLU epilogue
            // straight from TMEM (no fp32 gate/up round trip, no SiLU kernel), a sparse last
            // wave as stream-K pieces + ticketed finalize (the tensor regime's hybrid)
            ck_gemm_fuse fh{};
            fh.kind = CK_FUSE_SILU;
            fh.zero_after = 1;
            fh.tickets = tile_tickets_;
            fh.act = act_;
            gemm(L.wgu, h_, gu_, nullptr, M, 2 * F, H, CK_EPI_SILU_BF16, 0, &fh);
        } else if (M <= silu_fuse_rows()) {
            // weight-streaming regime: SiLU * up in the stream-K GEMM's ticketed tile finalize
            gemm(L.wgu, h_, gu_, nullptr, M, 2 * F, H, CK_EPI_RED_F32, 0, &fs);
        } else {
            gemm(L.wgu, h_, gu_, nullptr, M, 2 * F, H, small ? CK_EPI_RED_F32 : CK_EPI_F32, small ? 0 : 1);
            mark(a);
            check_ck(ck_silu_mul(gu_, act_, M, F, small ? 1 : 0, stream_), "silu_mul");
            ++launches;
            done(a, &stat_other, 0, 0);
        }
        if (norm_fused && l + 1 < m.layers) {  // the next layer's attention norm
            ck_gemm_fuse fn = norm_fuse;
            fn.gamma = w_.layer[l + 1].attn_norm;
            fn.zero = fused_rope ? qkv_ : nullptr;
            fn.zero_cols = Q;
            gemm(L.wd, act_, x_, nullptr, M, H, F, CK_EPI_RED_F32, 0, &fn);
        } else {
            gemm(L.wd, act_, x_, nullptr, M, H, F, CK_EPI_RED_F32, 0);
        }
    }
    if (R > 0) {
        mark(a);
        check_ck(ck_rmsnorm(x_, w_.final_norm, hs_, D(o_s_row), R, H, m.rms_eps, nullptr, 0, stream_), "final norm");
        ++launches;
        done(a, &stat_other, 0, 0);
        // LM head: a 1 GB weight stream for a handful of rows -> stream-K red.add into the
        // logits the previous argmax cleared (balanced over the grid); larger R: tile stores
        if (R <= 128)
            gemm(w_.lm_head, hs_, logits_, nullptr, R, m.vocab, H, CK_EPI_RED_F32, 0);
        else
            gemm(w_.lm_head, hs_, logits_, nullptr, R, m.vocab, H, CK_EPI_F32, 1);
        mark(a);
        check_ck(ck_argmax_emit(logits_, R, m.vocab, D(o_s_rid), reinterpret_cast<const long long*>(D(o_s_out)),
                                last_tok, out_tok, arg_ws_, arg_tickets_, 1, logits_out_, stream_),
                 "argmax");
        ++launches;
        done(a, &stat_other, 0, 0);
    }
    };

    // Decode-only weight-streaming passes repeat the same launch sequence for a given shape
    // (rows, attention work items, cluster size, stream): the graph_min_seen()-th time a shape
    // is seen the chain is captured into a CUDA graph (PDL edges kept) and replayed from then on — a
    // dependent kernel boundary costs ~1.3-1.5 us in a graph vs ~1.9-2.7 us on a stream.
    const bool graphable = use_graphs() && !profile_ && fused_rope && !logits_out_;
    if (graphable) {
        char key[256];
        std::snprintf(key, sizeof key, "%d/%d/%d/%d/%d/%p/%d/%p/%d/%p/%p/%p/%p/%p", M, R, n_dec, n_work,
                      b.decode_cluster, static_cast<void*>(stream_), max_ctas_, pool.base, pool.blocks,
                      static_cast<const void*>(prompt),
                      static_cast<const void*>(prompt_off), static_cast<void*>(last_tok),
                      static_cast<void*>(out_tok), static_cast<void*>(meta_dev_));
        auto it = graphs_.find(key);
        if (it != graphs_.end()) {
            check_cuda(cudaGraphLaunch(it->second.exec, stream_), "graph launch");
            launches += it->second.kernels;
            ++graph_hits_;
            for (const auto& t : it->second.tallies) {  // decode attention work: this pass's keys
                const bool attn = t.into == &stat_decode_attn;
                t.into->launches++;
                t.into->bytes += attn ? dec_keys * kv_tok_layer : t.bytes;
                t.into->flops += attn ? 4.0 * m.n_heads * m.head_dim * dec_keys : t.flops;
            }
            return;
        }
        if (++graph_seen_[key] < graph_min_seen()) {  // early sightings run plainly (lazy init)
            issue();
            done(pass0, &stat_forward, 0, 0);
            return;
        }
        std::vector<Tally> tallies;
        const long long l0 = launches;
        check_cuda(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
        cudaGraph_t g = nullptr;
        tally_rec_ = &tallies;
        try {
            issue();
            done(pass0, &stat_forward, 0, 0);
            tally_rec_ = nullptr;
        } catch (...) {
            tally_rec_ = nullptr;
            cudaStreamEndCapture(stream_, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            throw;
        }
        check_cuda(cudaStreamEndCapture(stream_, &g), "end capture");
        cudaGraphExec_t exec = nullptr;
        check_cuda(cudaGraphInstantiate(&exec, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
        graphs_[key] = GraphEntry{exec, launches - l0, std::move(tallies)};
        check_cuda(cudaGraphLaunch(exec, stream_), "graph launch");
        return;
    }
    issue();
    done(pass0, &stat_forward, 0, 0);
}

}  // namespace gpu
}  // namespace cronus
