// GpuEngine: persistent B200 resources (weights, KV pools, workers, streams) and the
// per-run executor that turns the scheduler's work items into device work.
//
// Stream topology per worker pair:
//   ppi stream  (PPI device)  partial prefills; SM-partitioned when co-located
//   cpi stream  (CPI device)  mixed chunk + decode iterations
//   copy stream (CPI device)  KV handoff: pull kernel over NVLink (or D2D)
// Cross-stream ordering is by CUDA events only:
//   handoff  waits  the request's prefill            (its KV exists)
//            waits  the CPI release fence           (destination blocks are free)
//   CPI iter waits  the handoff of every request it touches for the first time
//   PPI pass waits  the PPI release fence           (reused blocks were copied out)
// so the GPU may run arbitrarily far behind the scheduler (virtual clock) and
// still execute exactly the scheduled work, and in wall-clock mode the copy
// stream overlaps CPI compute.
#include <algorithm>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <thread>

#include "../host/scheduler.hpp"
#include "cronus/gpu.hpp"
#include "cronus/policies.hpp"
#include "cronus_ck.h"
#include "model.hpp"
#include "partition.hpp"

namespace cronus {

using gpu::check_ck;
using gpu::check_cuda;

namespace {

struct EngineOptions {
    std::string model = "llama3-8b";
    bool wall = false;
    int ppi_device = 0, cpi_device = 0;
    int ppi_sms = 0;
    int ppi_chunk = 4096;
    long long cpi_pool_blocks = 0, ppi_pool_blocks = 0;
    uint64_t seed = 1234, prompt_seed = 99;
    bool profile = false;
    // co-located pair with a green-context split: CPI iterations launched while the PPI
    // has nothing in flight run on all SMs (the PPI's share is idle); PPI work issued
    // behind such an iteration waits for it, so the two never contend for SMs
    bool sm_lending = true;
    // test hook: treat ppi_device == cpi_device as two separate devices (own weights, pools,
    // token buffers, copy streams): exercises the multi-GPU pair path on one GPU
    bool separate = false;
};

EngineOptions parse_engine_options(const std::string& text) {
    EngineOptions o;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        const size_t hash = line.find('#');
        if (hash != std::string::npos) line = line.substr(0, hash);
        const size_t eq = line.find('=');
        auto strip = [](std::string s) {
            const size_t a = s.find_first_not_of(" \t\r");
            if (a == std::string::npos) return std::string();
            return s.substr(a, s.find_last_not_of(" \t\r") - a + 1);
        };
        if (eq == std::string::npos) {
            if (!strip(line).empty()) throw std::invalid_argument("engine options: expected key = value: " + line);
            continue;
        }
        const std::string k = strip(line.substr(0, eq)), v = strip(line.substr(eq + 1));
        if (k == "model") o.model = v;
        else if (k == "clock") {
            if (v != "virtual" && v != "wall") throw std::invalid_argument("engine options: clock = virtual | wall");
            o.wall = v == "wall";
        } else if (k == "ppi_device") o.ppi_device = std::stoi(v);
        else if (k == "cpi_device") o.cpi_device = std::stoi(v);
        else if (k == "ppi_sms") o.ppi_sms = std::stoi(v);
        else if (k == "ppi_chunk") o.ppi_chunk = std::stoi(v);
        else if (k == "cpi_pool_blocks") o.cpi_pool_blocks = std::stoll(v);
        else if (k == "ppi_pool_blocks") o.ppi_pool_blocks = std::stoll(v);
        else if (k == "seed") o.seed = std::stoull(v);
        else if (k == "prompt_seed") o.prompt_seed = std::stoull(v);
        else if (k == "profile") o.profile = v == "1" || v == "true";
        else if (k == "sm_lending") o.sm_lending = v == "1" || v == "true";
        else if (k == "separate") o.separate = v == "1" || v == "true";
        else throw std::invalid_argument("engine options: unknown key " + k);
    }
    if (o.ppi_chunk < 16 || o.ppi_chunk % 16) throw std::invalid_argument("engine options: ppi_chunk % 16 != 0");
    return o;
}

struct DeviceBuf {
    int dev = 0;
    void* p = nullptr;
    size_t cap = 0;
    void ensure(int device, size_t bytes) {
        if (bytes <= cap && p) return;
        release();
        dev = device;
        check_cuda(cudaSetDevice(dev), "cudaSetDevice");
        check_cuda(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "cudaMalloc(request buffers)");
        cap = std::max<size_t>(bytes, 256);
    }
    void release() {
        if (p) {
            cudaSetDevice(dev);
            cudaFree(p);
        }
        p = nullptr;
        cap = 0;
    }
    ~DeviceBuf() { release(); }
};

// Request-token buffers of one device.
struct TokenBufs {
    DeviceBuf prompt, prompt_off, last_tok, out_tok;
};

}  // namespace

struct GpuEngine::Impl {
    EngineOptions opt;
    gpu::ModelSpec spec;
    bool colocated = true;
    std::shared_ptr<gpu::Weights> w_ppi, w_cpi;
    std::unique_ptr<gpu::KvPool> pool_ppi, pool_cpi;
    cudaStream_t s_ppi = nullptr, s_cpi = nullptr, s_copy = nullptr;
    cudaStream_t s_cpi_full = nullptr;  // primary-context stream for lent (all-SM) CPI iterations
    cudaStream_t s_cpi_side = nullptr, s_cpi_full_side = nullptr;  // their side streams (Worker::side_)
    bool own_cpi_side = false;
    cudaStream_t cpi_side(cudaStream_t main) const { return main == s_cpi_full ? s_cpi_full_side : s_cpi_side; }
    cudaStream_t s_copy_low = nullptr;  // handoffs INTO the low side (disagg-hl) on its own device
    std::unique_ptr<gpu::Worker> ppi, cpi;
    std::unique_ptr<gpu::SmPartition> part;
    std::string partition_mode = "none";
    bool own_cpi_streams = false, own_ppi_stream = false;  // streams created outside a partition
    int ppi_ctas = 0, cpi_ctas = 0;  // persistent-grid caps per worker (0 = whole device)
    int cpi_rows = 0, cpi_samples = 0, ppi_rows = 0, ppi_samples = 0;
    TokenBufs tok_cpi, tok_ppi;
    // pinned staging for handoff block lists
    static constexpr int kRing = 16;
    int* xfer_host[kRing] = {};
    cudaEvent_t xfer_ev[2][kRing] = {};  // per side's device: [low, high]
    int xfer_slot = 0;
    DeviceBuf xfer_dev;      // kRing slices (handoffs into the high side)
    DeviceBuf xfer_dev_low;  // kRing slices (handoffs into the low side, separate devices)
    long long xfer_cap = 0;  // ints per slice
    int sms = 148;
    uint64_t staged_hash = 0;  // trace whose synthesized prompts are resident in tok_*.prompt

    explicit Impl(const std::string& text) : opt(parse_engine_options(text)), spec(gpu::ModelSpec::preset(opt.model)) {
        spec.seed = opt.seed;
        colocated = opt.ppi_device == opt.cpi_device && !opt.separate;
        int ndev = 0;
        check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (opt.ppi_device >= ndev || opt.cpi_device >= ndev)
            throw std::invalid_argument("engine options: device index out of range");
        check_cuda(cudaSetDevice(opt.cpi_device), "cudaSetDevice");
        sms = ck_device_sms();
        w_cpi = std::make_shared<gpu::Weights>(spec, opt.cpi_device);
        w_ppi = colocated ? w_cpi : std::make_shared<gpu::Weights>(spec, opt.ppi_device);
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (colocated && opt.ppi_sms > 0) {
            check_cuda(cudaSetDevice(opt.cpi_device), "cudaSetDevice");
            part = gpu::make_sm_partition(opt.cpi_device, opt.ppi_sms, lo, hi);
            if (part) {
                s_ppi = part->ppi_stream;
                s_cpi = part->cpi_stream;
                s_copy = part->copy_stream;
                ppi_ctas = part->ppi_sms;
                cpi_ctas = part->cpi_sms;
                partition_mode = "green-context";
                s_cpi_side = part->cpi_side_stream;
                if (opt.sm_lending) {
                    check_cuda(cudaStreamCreateWithPriority(&s_cpi_full, cudaStreamNonBlocking, hi), "stream");
                    check_cuda(cudaStreamCreateWithPriority(&s_cpi_full_side, cudaStreamNonBlocking, lo), "stream");
                }
            } else {
                ppi_ctas = opt.ppi_sms;  // fallback: only the PPI's GEMM grid is capped
                partition_mode = "grid-cap";
            }
        }
        if (!colocated && opt.ppi_sms > 0) {
            // separate devices: the low-end worker is emulated by SM-partitioning its own
            // device (north star); only the partition's PPI stream is used
            part = gpu::make_sm_partition(opt.ppi_device, opt.ppi_sms, lo, hi);
            if (part) {
                s_ppi = part->ppi_stream;
                ppi_ctas = part->ppi_sms;
                partition_mode = "green-context (ppi device)";
            } else {
                ppi_ctas = opt.ppi_sms;
                partition_mode = "grid-cap (ppi device)";
            }
        }
        if (!s_cpi) {
            check_cuda(cudaSetDevice(opt.cpi_device), "cudaSetDevice");
            check_cuda(cudaStreamCreateWithPriority(&s_cpi, cudaStreamNonBlocking, hi), "stream");
            check_cuda(cudaStreamCreateWithPriority(&s_copy, cudaStreamNonBlocking, hi), "stream");
            own_cpi_streams = true;
        }
        if (!s_cpi_side) {
            check_cuda(cudaSetDevice(opt.cpi_device), "cudaSetDevice");
            check_cuda(cudaStreamCreateWithPriority(&s_cpi_side, cudaStreamNonBlocking, lo), "stream");
            own_cpi_side = true;
        }
        if (!s_ppi) {
            check_cuda(cudaSetDevice(opt.ppi_device), "cudaSetDevice");
            check_cuda(cudaStreamCreateWithPriority(&s_ppi, cudaStreamNonBlocking, lo), "stream");
            own_ppi_stream = true;
        }
        if (!colocated) {
            int can = opt.ppi_device == opt.cpi_device;  // `separate` test mode: same device
            if (!can) check_cuda(cudaDeviceCanAccessPeer(&can, opt.cpi_device, opt.ppi_device), "peer query");
            if (!can) throw std::runtime_error("CPI device cannot access the PPI device over NVLink (no P2P)");
            for (auto [a, b] : {std::pair{opt.cpi_device, opt.ppi_device}, std::pair{opt.ppi_device, opt.cpi_device}}) {
                if (a == b) continue;  // `separate` test mode on one device
                check_cuda(cudaSetDevice(a), "cudaSetDevice");
                cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) check_cuda(e, "enable peer access");
                cudaGetLastError();
            }
            check_cuda(cudaSetDevice(opt.ppi_device), "cudaSetDevice");
            check_cuda(cudaStreamCreateWithPriority(&s_copy_low, cudaStreamNonBlocking, hi), "stream");
        }
        for (int side = 0; side < 2; ++side) {  // events must live on the device whose streams record them
            check_cuda(cudaSetDevice(side ? opt.cpi_device : opt.ppi_device), "cudaSetDevice");
            for (int i = 0; i < kRing; ++i)
                check_cuda(cudaEventCreateWithFlags(&xfer_ev[side][i], cudaEventDisableTiming), "event");
        }
        check_cuda(cudaSetDevice(opt.cpi_device), "cudaSetDevice");
    }

    ~Impl() {
        for (int i = 0; i < kRing; ++i) {
            if (xfer_host[i]) cudaFreeHost(xfer_host[i]);
            for (int side = 0; side < 2; ++side)
                if (xfer_ev[side][i]) cudaEventDestroy(xfer_ev[side][i]);
        }
        ppi.reset();
        cpi.reset();
        if (s_cpi_full) cudaStreamDestroy(s_cpi_full);
        if (s_cpi_full_side) cudaStreamDestroy(s_cpi_full_side);
        if (own_cpi_side && s_cpi_side) cudaStreamDestroy(s_cpi_side);
        if (s_copy_low) cudaStreamDestroy(s_copy_low);
        if (own_ppi_stream && s_ppi) cudaStreamDestroy(s_ppi);
        if (own_cpi_streams) {
            if (s_cpi) cudaStreamDestroy(s_cpi);
            if (s_copy) cudaStreamDestroy(s_copy);
        }
        part.reset();  // owns the green-context streams
    }

    int cpi_sm_count() const { return cpi_ctas > 0 ? cpi_ctas : sms; }
    int ppi_sm_count() const { return ppi_ctas > 0 ? ppi_ctas : sms; }
    // the two sides of a pair: high = the CPI partition / device, low = the PPI one
    gpu::Worker& worker(bool high) { return high ? *cpi : *ppi; }
    gpu::KvPool& pool(bool high) { return high ? *pool_cpi : *pool_ppi; }
    int device(bool high) const { return high ? opt.cpi_device : opt.ppi_device; }
    TokenBufs& tok(bool high) { return high || colocated ? tok_cpi : tok_ppi; }
    cudaStream_t copy_stream(bool into_high) { return into_high || colocated ? s_copy : s_copy_low; }
    DeviceBuf& xfer_buf(bool into_high) { return into_high || colocated ? xfer_dev : xfer_dev_low; }

    std::string describe(bool probe) {
        std::ostringstream o;
        o << "{\"mode\": \"" << partition_mode << "\", \"device_sms\": " << sms << ", \"ppi_sms\": "
          << (ppi_ctas ? ppi_ctas : sms) << ", \"cpi_sms\": " << cpi_sm_count()
          << ", \"sm_lending\": " << (s_cpi_full ? "true" : "false");
        // CUDA stream ids (as CUPTI / profilers report them) of each worker's streams
        auto sid = [](cudaStream_t st) {
            unsigned long long id = 0;
            if (st) cudaStreamGetId(st, &id);
            return id;
        };
        o << ", \"stream_ids\": {\"ppi\": " << sid(s_ppi) << ", \"cpi\": " << sid(s_cpi)
          << ", \"cpi_full\": " << sid(s_cpi_full) << ", \"copy\": " << sid(s_copy) << "}";
        if (probe) {
            auto seen = [&](int dev, cudaStream_t st) {
                check_cuda(cudaSetDevice(dev), "cudaSetDevice");
                int* hits = nullptr;
                check_cuda(cudaMalloc(&hits, 256 * 4), "alloc");
                check_cuda(cudaMemsetAsync(hits, 0, 256 * 4, st), "memset");
                check_ck(ck_smid_probe(hits, 4 * sms, st), "smid probe");
                int h[256];
                check_cuda(cudaMemcpyAsync(h, hits, sizeof h, cudaMemcpyDeviceToHost, st), "D2H");
                check_cuda(cudaStreamSynchronize(st), "sync");
                cudaFree(hits);
                int n = 0;
                for (int v : h) n += v > 0;
                return n;
            };
            o << ", \"ppi_seen\": " << seen(opt.ppi_device, s_ppi) << ", \"cpi_seen\": " << seen(opt.cpi_device, s_cpi);
        }
        o << "}";
        return o.str();
    }

    // Size pools / workers for this config (reallocating only when they grow).
    void prepare(const ClusterConfig& cfg) {
        if (cfg.high_gpu.kv_block_size != 16 || cfg.low_gpu.kv_block_size != 16)
            throw std::invalid_argument("B200 engine: kv_block_size must be 16 (the kernels' page size)");
        const long long cpi_blocks = opt.cpi_pool_blocks > 0 ? opt.cpi_pool_blocks : cfg.high_gpu.kv_blocks_capacity;
        const long long ppi_blocks = opt.ppi_pool_blocks > 0 ? opt.ppi_pool_blocks : cfg.low_gpu.kv_blocks_capacity;
        if (cpi_blocks < cfg.high_gpu.kv_blocks_capacity || ppi_blocks < cfg.low_gpu.kv_blocks_capacity)
            throw std::invalid_argument("B200 engine: physical KV pools smaller than the profiles' capacities");
        const long long bb = spec.kv_block_bytes();
        // a worker's metadata buffer is sized for its pool's block count: a grown pool
        // rebuilds the worker that indexes it
        bool regrow_cpi = false, regrow_ppi = false;
        if (!pool_cpi || pool_cpi->blocks < cpi_blocks) {
            pool_cpi.reset();
            pool_cpi = std::make_unique<gpu::KvPool>(opt.cpi_device, cpi_blocks, bb);
            regrow_cpi = true;
        }
        if (!pool_ppi || pool_ppi->blocks < ppi_blocks) {
            pool_ppi.reset();
            pool_ppi = std::make_unique<gpu::KvPool>(opt.ppi_device, ppi_blocks, bb);
            regrow_ppi = true;
        }
        // Each side's worker serves the roles the policy puts there: serial prefill in
        // ppi_chunk-row slices and/or chunked iterations of up to B rows (all sampled).
        bool serial[2] = {false, false}, chunked[2] = {false, false};
        for (const InstanceSpec& in : bind_policy(cfg).instances)
            (in.role == Role::PPI || in.role == Role::PurePrefill ? serial : chunked)[in.on_high_gpu] = true;
        const int B[2] = {cfg.max_batched_tokens_low, cfg.max_batched_tokens_high};
        auto rows = [&](int h) { return std::max(serial[h] ? opt.ppi_chunk : 0, chunked[h] ? B[h] : 0); };
        auto samples = [&](int h) { return std::max(1, chunked[h] ? B[h] : 0); };
        if (!cpi || regrow_cpi || cpi_rows < rows(1) || cpi_samples < samples(1)) {
            cpi.reset();
            cpi_rows = std::max(cpi_rows, rows(1));
            cpi_samples = std::max(cpi_samples, samples(1));
            check_cuda(cudaSetDevice(opt.cpi_device), "cudaSetDevice");
            cpi = std::make_unique<gpu::Worker>(*w_cpi, cpi_rows, cpi_samples,
                                                static_cast<int>(pool_cpi->blocks) + cpi_rows, s_cpi, cpi_ctas);
        }
        if (!ppi || regrow_ppi || ppi_rows < rows(0) || ppi_samples < samples(0)) {
            ppi.reset();
            ppi_rows = std::max(ppi_rows, rows(0));
            ppi_samples = std::max(ppi_samples, samples(0));
            check_cuda(cudaSetDevice(opt.ppi_device), "cudaSetDevice");
            ppi = std::make_unique<gpu::Worker>(*w_ppi, ppi_rows, ppi_samples,
                                                static_cast<int>(pool_ppi->blocks) + ppi_rows, s_ppi, ppi_ctas);
        }
        const long long need = 2 * std::max(pool_ppi->blocks, pool_cpi->blocks) + 64;
        if (xfer_cap < need) {
            for (int i = 0; i < kRing; ++i) {
                if (xfer_host[i]) cudaFreeHost(xfer_host[i]);
                check_cuda(cudaMallocHost(&xfer_host[i], need * 4), "pinned xfer");
            }
            xfer_dev.ensure(opt.cpi_device, static_cast<size_t>(need) * 4 * kRing);
            if (!colocated) xfer_dev_low.ensure(opt.ppi_device, static_cast<size_t>(need) * 4 * kRing);
            xfer_cap = need;
        }
    }
};

namespace {

// ---------------------------------------------------------------------------------
class PairExecutor : public sched::Executor {
  public:
    PairExecutor(GpuEngine::Impl& e, const ClusterConfig& cfg, const Trace& t, const GpuRunOptions& o)
        : E(e), trace(t), opts(o) {
        // scheduler instance indices (serial / chunked, in binding order) -> pair side
        for (const InstanceSpec& in : bind_policy(cfg).instances)
            (in.role == Role::PPI || in.role == Role::PurePrefill ? serial_high : chunked_high)
                .push_back(in.on_high_gpu);
        // lending the low side's SMs to high-side iterations: only where the low side
        // runs serial prefills that the lent iteration may delay (cronus, disagg-lh)
        lending = cfg.policy == Policy::Cronus || cfg.policy == Policy::DisaggLowHigh;
        cpi_stream = E.s_cpi;
        const int n = static_cast<int>(t.requests.size());
        prompt_off.resize(n);
        out_off.resize(n);
        long long pin = 0, pout = 0;
        for (int i = 0; i < n; ++i) {
            prompt_off[i] = pin;
            out_off[i] = pout;
            pin += t.requests[i].input_len;
            pout += t.requests[i].output_len;
        }
        total_in = pin;
        total_out = pout;
        prefill_ev.assign(n, nullptr);
        xfer_ev.assign(n, nullptr);
        xfer_pending.assign(n, 0);
        if (opts.host_logits) {
            if (!E.colocated) throw std::invalid_argument("host_logits: co-located pairs only");
            const size_t bytes = static_cast<size_t>(total_out) * E.spec.vocab * 4;
            logits_buf.ensure(E.opt.cpi_device, bytes);
            check_cuda(cudaMemset(logits_buf.p, 0, bytes), "memset logits sink");
            E.cpi->set_logits_out(static_cast<float*>(logits_buf.p));
            E.ppi->set_logits_out(static_cast<float*>(logits_buf.p));
        }
    }

    ~PairExecutor() override {
        E.cpi->set_logits_out(nullptr);
        E.ppi->set_logits_out(nullptr);
        for (auto* v : {&prefill_ev, &xfer_ev})
            for (cudaEvent_t ev : *v)
                if (ev) cudaEventDestroy(ev);
        for (auto& q : done_q)
            for (auto& t : q) cudaEventDestroy(t.ev);
        for (auto& pool : spare)
            for (cudaEvent_t ev : pool) cudaEventDestroy(ev);
        for (cudaEvent_t ev : last_iter)
            if (ev) cudaEventDestroy(ev);
        if (stage_fence) cudaEventDestroy(stage_fence);
        if (t0_cpi) cudaEventDestroy(t0_cpi);
        if (t0_ppi) cudaEventDestroy(t0_ppi);
        if (pinned_prompt) cudaFreeHost(pinned_prompt);
    }

    // Request token buffers on each device; prompts from the host (e2e) or synthesized.
    void upload() {
        const int n = static_cast<int>(trace.requests.size());
        auto setup = [&](TokenBufs& tb, int dev, cudaStream_t s) {
            tb.prompt.ensure(dev, static_cast<size_t>(total_in) * 4);
            tb.prompt_off.ensure(dev, static_cast<size_t>(n) * 8);
            tb.last_tok.ensure(dev, static_cast<size_t>(n) * 4);
            tb.out_tok.ensure(dev, static_cast<size_t>(total_out) * 4);
            check_cuda(cudaSetDevice(dev), "cudaSetDevice");
            check_cuda(cudaMemcpyAsync(tb.prompt_off.p, prompt_off.data(), n * 8, cudaMemcpyHostToDevice, s),
                       "prompt_off H2D");
            check_cuda(cudaMemsetAsync(tb.out_tok.p, 0xff, static_cast<size_t>(total_out) * 4, s), "memset");
            if (opts.host_prompt) {
                if (!pinned_prompt) {
                    check_cuda(cudaMallocHost(&pinned_prompt, static_cast<size_t>(total_in) * 4), "pinned prompt");
                    std::memcpy(pinned_prompt, opts.host_prompt, static_cast<size_t>(total_in) * 4);
                }
                check_cuda(cudaMemcpyAsync(tb.prompt.p, pinned_prompt, static_cast<size_t>(total_in) * 4,
                                           cudaMemcpyHostToDevice, s),
                           "prompt H2D");
                h2d_bytes += total_in * 4;
            } else if (E.staged_hash != trace_hash(trace) || E.staged_hash == 0) {
                synth_prompts(tb, s);  // not staged beforehand: synthesize on the device now
            }
            h2d_bytes += n * 8;
        };
        setup(E.tok_cpi, E.opt.cpi_device, E.s_cpi);
        if (!E.colocated) setup(E.tok_ppi, E.opt.ppi_device, E.s_ppi);
        E.staged_hash = opts.host_prompt ? 0 : trace_hash(trace);
        check_cuda(cudaSetDevice(E.opt.cpi_device), "cudaSetDevice");
        check_cuda(cudaStreamSynchronize(E.s_cpi), "sync");
        check_cuda(cudaSetDevice(E.opt.ppi_device), "cudaSetDevice");
        check_cuda(cudaStreamSynchronize(E.s_ppi), "sync");
    }

    void synth_prompts(TokenBufs& tb, cudaStream_t s) {
        // request id / position per prompt token -> device hash kernel
        std::vector<int> rq(total_in), ps(total_in);
        long long k = 0;
        for (const Request& r : trace.requests)
            for (int p = 0; p < r.input_len; ++p, ++k) {
                rq[k] = r.id;
                ps[k] = p;
            }
        int* d = nullptr;
        check_cuda(cudaMalloc(&d, static_cast<size_t>(total_in) * 8 + 16), "tmp");
        check_cuda(cudaMemcpyAsync(d, rq.data(), total_in * 4, cudaMemcpyHostToDevice, s), "H2D");
        check_cuda(cudaMemcpyAsync(d + total_in, ps.data(), total_in * 4, cudaMemcpyHostToDevice, s), "H2D");
        check_ck(ck_prompt_tokens(static_cast<int*>(tb.prompt.p), d, d + total_in, static_cast<int>(total_in),
                                  E.opt.prompt_seed, E.spec.vocab, s),
                 "prompt_tokens");
        check_cuda(cudaStreamSynchronize(s), "sync");
        cudaFree(d);
    }

    // Disaggregated handoff, second half: copy a request's staged KV into the blocks
    // its decode instance allocated at admission (stream-ordered before its first row).
    void place_staged(int rid, const std::vector<int32_t>& blocks, bool hi, cudaStream_t st) {
        auto it = stage_slots.find(rid);
        if (it == stage_slots.end()) return;
        const std::vector<int32_t>& slots = it->second;
        const int nb = static_cast<int>(slots.size());
        if (static_cast<int>(blocks.size()) < nb) throw std::logic_error("staged handoff: table shorter than prefix");
        const int slot = E.xfer_slot;
        E.xfer_slot = (E.xfer_slot + 1) % GpuEngine::Impl::kRing;
        for (auto& ring : E.xfer_ev) check_cuda(cudaEventSynchronize(ring[slot]), "xfer staging");
        int* h = E.xfer_host[slot];
        std::memcpy(h, slots.data(), nb * 4);
        std::memcpy(h + nb, blocks.data(), nb * 4);
        int* d = static_cast<int*>(E.xfer_buf(hi).p) + slot * E.xfer_cap;
        check_cuda(cudaMemcpyAsync(d, h, 2 * nb * 4, cudaMemcpyHostToDevice, st), "stage ids");
        check_cuda(cudaEventRecord(E.xfer_ev[hi][slot], st), "event");
        check_ck(ck_kv_copy(E.pool(stage_side).base, d, E.pool(hi).base, d + nb, nb, E.pool(hi).block_bytes, st),
                 "kv_copy (staged)");
        ++copy_launches;
        if (!E.colocated && stage_tok[rid]) {  // the first token travels with the KV
            check_ck(ck_copy_token(static_cast<int*>(E.tok(stage_side).last_tok.p), rid,
                                   static_cast<int*>(E.tok(hi).last_tok.p), rid,
                                   static_cast<int*>(E.tok(hi).out_tok.p), out_off[rid], st),
                     "copy_token");
            ++copy_launches;
        }
        stage_fence = record(st, stage_fence);  // slots reusable once this copy ran
        stage_free.insert(stage_free.end(), slots.begin(), slots.end());
        stage_slots.erase(it);
    }

    // Staging region = the upper 3/4 of the prefill side's pool (its serial instance
    // allocates lowest ids first and holds one or two requests at a time).
    void init_staging(bool side) {
        if (staging_ready) {
            if (side != stage_side) throw std::logic_error("staging: prefill side changed within a run");
            return;
        }
        staging_ready = true;
        stage_side = side;
        const long long n = E.pool(side).blocks;
        stage_lo = static_cast<int32_t>(n / 4);
        for (long long b = stage_lo; b < n; ++b) stage_free.push_back(static_cast<int32_t>(b));
    }

    // Stream of a side: the low side has one; the high side's current stream may be
    // the lent all-SM one.
    cudaStream_t side_stream(bool high) const { return high ? cpi_stream : E.s_ppi; }

    // ------------------------------------------------------------- work sites
    uint64_t prefill(const sched::PrefillWork& w) override {
        const bool hi = serial_high.at(w.instance);
        check_cuda(cudaSetDevice(E.device(hi)), "cudaSetDevice");
        cudaStream_t st = side_stream(hi);
        if (serial_fence[hi]) {
            check_cuda(cudaStreamWaitEvent(st, serial_fence[hi], 0), "wait fence");
            serial_fence[hi] = nullptr;
        }
        if (!hi && last_lent && last_iter[1]) {  // the in-flight lent iteration holds these SMs too
            check_cuda(cudaStreamWaitEvent(st, last_iter[1], 0), "wait lent iteration");
            last_lent = false;
        }
        if (staging_ready && hi == stage_side)
            for (int32_t b : *w.blocks)
                if (b >= stage_lo) throw std::runtime_error("serial prefill reached the staging region of its pool");
        TokenBufs& tb = E.tok(hi);
        gpu::Worker& W = E.worker(hi);
        const long long slice = std::min<long long>(E.opt.ppi_chunk, W.max_rows());
        for (long long start = 0; start < w.tokens; start += slice) {
            const long long len = std::min<long long>(slice, w.tokens - start);
            const bool last = start + len == w.tokens;
            batch.clear();
            batch.add_prefill(w.rid, start, len, *w.blocks, last && w.sample_last, out_off[w.rid]);
            W.forward(batch, E.pool(hi), static_cast<int*>(tb.prompt.p), static_cast<long long*>(tb.prompt_off.p),
                      static_cast<int*>(tb.last_tok.p), static_cast<int*>(tb.out_tok.p));
        }
        prefill_ev[w.rid] = record(st, prefill_ev[w.rid]);
        if (hi) last_iter[1] = record(st, last_iter[1]);  // keeps the high side's stream order
        prefill_tokens += w.tokens;
        return complete(st, hi ? 2 : 0, hi);
    }

    uint64_t transfer(const sched::TransferWork& w) override {
        const bool src_hi = serial_high.at(w.src_instance), dst_hi = chunked_high.at(w.dst_instance);
        // the pull kernel runs on the destination device (NVLink read of the source pool)
        check_cuda(cudaSetDevice(E.device(dst_hi)), "cudaSetDevice");
        cudaStream_t cs = E.copy_stream(dst_hi);
        if (prefill_ev[w.rid]) check_cuda(cudaStreamWaitEvent(cs, prefill_ev[w.rid], 0), "wait prefill");
        if (chunked_fence[dst_hi]) check_cuda(cudaStreamWaitEvent(cs, chunked_fence[dst_hi], 0), "wait fence");
        const int nb = static_cast<int>((w.tokens + 15) / 16);
        if (static_cast<int>(w.src_blocks->size()) < nb) throw std::logic_error("handoff: source table too short");
        // Cronus: the CPI reserved and allocated the prefix blocks before the link started.
        // Disaggregated: the decode instance allocates only at admission, later. The
        // prefill side then keeps the KV (moved into its pool's staging region, whose
        // blocks its serial instance never reaches) until the decode side pulls it into
        // the admitted request's blocks (place_staged) — the pull model of real
        // disaggregated deployments; the link carries the bytes at that point.
        const bool staged = static_cast<int>(w.dst_blocks->size()) < nb;
        const std::vector<int32_t>* dst_ids = w.dst_blocks;
        gpu::KvPool* dst_pool = &E.pool(dst_hi);
        if (staged) {
            check_cuda(cudaSetDevice(E.device(src_hi)), "cudaSetDevice");
            cs = E.copy_stream(src_hi);
            if (prefill_ev[w.rid]) check_cuda(cudaStreamWaitEvent(cs, prefill_ev[w.rid], 0), "wait prefill");
            init_staging(src_hi);
            if (static_cast<int>(stage_free.size()) < nb)
                throw std::runtime_error("handoff: staging region of the prefill pool exhausted");
            std::vector<int32_t>& slots = stage_slots[w.rid];
            slots.assign(stage_free.end() - nb, stage_free.end());
            stage_free.resize(stage_free.size() - nb);
            dst_ids = &slots;
            dst_pool = &E.pool(src_hi);
            if (stage_fence) check_cuda(cudaStreamWaitEvent(cs, stage_fence, 0), "wait staging reuse");
        }
        const int slot = E.xfer_slot;
        E.xfer_slot = (E.xfer_slot + 1) % GpuEngine::Impl::kRing;
        for (auto& ring : E.xfer_ev) check_cuda(cudaEventSynchronize(ring[slot]), "xfer staging");
        int* h = E.xfer_host[slot];
        std::memcpy(h, w.src_blocks->data(), nb * 4);
        std::memcpy(h + nb, dst_ids->data(), nb * 4);
        int* d = static_cast<int*>(E.xfer_buf(staged ? src_hi : dst_hi).p) + slot * E.xfer_cap;
        check_cuda(cudaMemcpyAsync(d, h, 2 * nb * 4, cudaMemcpyHostToDevice, cs), "xfer ids");
        check_cuda(cudaEventRecord(E.xfer_ev[staged ? src_hi : dst_hi][slot], cs), "event");
        check_ck(ck_kv_copy(E.pool(src_hi).base, d, dst_pool->base, d + nb, nb, dst_pool->block_bytes, cs), "kv_copy");
        ++copy_launches;
        const Request& r = trace.requests[w.rid];
        if (!E.colocated && w.tokens == r.input_len && !staged) {
            // the prefill side sampled the first token: it travels with the KV
            check_ck(ck_copy_token(static_cast<int*>(E.tok(src_hi).last_tok.p), w.rid,
                                   static_cast<int*>(E.tok(dst_hi).last_tok.p), w.rid,
                                   static_cast<int*>(E.tok(dst_hi).out_tok.p), out_off[w.rid], cs),
                     "copy_token");
            ++copy_launches;
        }
        xfer_ev[w.rid] = record(cs, xfer_ev[w.rid]);
        xfer_pending[w.rid] = 1;
        if (staged) stage_tok[w.rid] = w.tokens == r.input_len;
        handoff_bytes += static_cast<double>(nb) * E.pool(dst_hi).block_bytes;
        handoffs++;
        return complete(cs, 1, staged ? src_hi : dst_hi);
    }

    uint64_t iteration(const sched::IterWork& w) override {
        const bool hi = chunked_high.at(w.instance);
        check_cuda(cudaSetDevice(E.device(hi)), "cudaSetDevice");
        // SM lending: nothing in flight on the low side -> this iteration may use every SM
        const bool lend = hi && lending && E.opt.wall && E.s_cpi_full && done_q[0].empty();
        cudaStream_t cur = E.s_ppi;
        if (hi) {
            cur = lend ? E.s_cpi_full : E.s_cpi;
            if (cur != cpi_stream) {  // keep high-side work in order across the two streams
                if (last_iter[1]) check_cuda(cudaStreamWaitEvent(cur, last_iter[1], 0), "wait previous iteration");
                cpi_stream = cur;
                E.cpi->set_launch(cur, lend ? 0 : E.cpi_ctas, E.cpi_side(cur));
            }
        }
        auto need = [&](int rid, const std::vector<int32_t>* blocks) {
            if (xfer_pending[rid]) {
                check_cuda(cudaStreamWaitEvent(cur, xfer_ev[rid], 0), "wait handoff");
                xfer_pending[rid] = 0;
            }
            if (blocks) place_staged(rid, *blocks, hi, cur);
        };
        batch.clear();
        for (const sched::DecodeRow& d : w.decoders) {
            need(d.rid, d.blocks);
            const long long emitted = d.ctx - trace.requests[d.rid].input_len;
            batch.add_decode(d.rid, d.ctx, *d.blocks, out_off[d.rid] + emitted);
        }
        if (w.chunk_rid >= 0) {
            need(w.chunk_rid, w.chunk_blocks);
            batch.add_prefill(w.chunk_rid, w.chunk_start, w.chunk_len, *w.chunk_blocks, w.chunk_samples,
                              out_off[w.chunk_rid]);
        }
        for (int rid : w.finishers) need(rid, nullptr);  // zero rows: its KV is placed when it decodes
        if (!batch.d_len.empty())
            batch.plan_decode(E.spec.n_kv_heads, gpu::decode_slots(E.spec.n_kv_heads, static_cast<int>(batch.d_len.size()), lend ? E.sms : hi ? E.cpi_sm_count() : E.ppi_sm_count()));
        if (E.opt.wall && hi) {  // device-side start of this iteration (busy time = end - start)
            iter_start = take_event(true);
            check_cuda(cudaEventRecord(iter_start, cur), "event record");
        }
        TokenBufs& tb = E.tok(hi);
        E.worker(hi).forward(batch, E.pool(hi), static_cast<int*>(tb.prompt.p),
                             static_cast<long long*>(tb.prompt_off.p), static_cast<int*>(tb.last_tok.p),
                             static_cast<int*>(tb.out_tok.p));
        iters++;
        lent_iters += lend ? 1 : 0;
        if (hi) last_lent = lend;
        iter_rows += batch.rows();
        decode_rows += static_cast<long long>(w.decoders.size());
        for (const sched::DecodeRow& d : w.decoders) decode_keys += d.ctx;
        chunk_rows += w.chunk_len;
        last_iter[hi] = record(cur, last_iter[hi]);
        return complete(cur, hi ? 2 : 0, hi);
    }

    void release(int instance, int rid) override {
        if (instance >= 1000) {
            // serial-instance blocks of rid were read by its handoff (none: it failed before one)
            if (xfer_ev[rid]) serial_fence[serial_high.at(instance - 1000)] = xfer_ev[rid];
        } else {
            const bool hi = chunked_high.at(instance);
            chunked_fence[hi] = last_iter[hi];  // freed at the end of the latest launched work there
        }
    }

    // ------------------------------------------------------------- clocks
    bool wall_clock() const override { return E.opt.wall; }

    void start() override {
        E.cpi->set_launch(E.s_cpi, E.cpi_ctas, E.s_cpi_side);
        cpi_stream = E.s_cpi;
        launches0_cpi = E.cpi->launches;
        launches0_ppi = E.ppi->launches;
        check_cuda(cudaSetDevice(E.opt.cpi_device), "cudaSetDevice");
        check_cuda(cudaEventCreate(&t0_cpi), "event");
        check_cuda(cudaEventRecord(t0_cpi, E.s_cpi), "event");
        check_cuda(cudaSetDevice(E.opt.ppi_device), "cudaSetDevice");
        check_cuda(cudaEventCreate(&t0_ppi), "event");
        check_cuda(cudaEventRecord(t0_ppi, E.s_ppi), "event");
        check_cuda(cudaEventSynchronize(t0_ppi), "sync");
        check_cuda(cudaSetDevice(E.opt.cpi_device), "cudaSetDevice");
        check_cuda(cudaEventSynchronize(t0_cpi), "sync");
        host_t0 = std::chrono::steady_clock::now();
    }

    double now_ms() override {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    }

    bool poll(sched::Completion& out) override {
        int best = -1;
        double best_t = 0;
        for (int q = 0; q < 3; ++q) {
            if (done_q[q].empty()) continue;
            Tick& t = done_q[q].front();
            if (!t.done) {
                const cudaError_t st = cudaEventQuery(t.ev);
                if (st == cudaErrorNotReady) continue;
                check_cuda(st, "event query");
                float ms = 0.f;
                check_cuda(cudaEventElapsedTime(&ms, t.high ? t0_cpi : t0_ppi, t.ev), "elapsed");
                t.t = ms;
                t.done = true;
                if (t.start) {
                    float busy = 0.f;
                    check_cuda(cudaEventElapsedTime(&busy, t.start, t.ev), "elapsed");
                    cpi_busy_ms += busy;
                    spare[1].push_back(t.start);
                    t.start = nullptr;
                }
            }
            if (best < 0 || t.t < best_t) {
                best = q;
                best_t = t.t;
            }
        }
        if (best < 0) return false;
        Tick t = done_q[best].front();
        done_q[best].pop_front();
        spare[t.high].push_back(t.ev);
        out.ticket = t.ticket;
        out.t_ms = t.t;
        return true;
    }

    void wait(double until_ms) override {
        // Completions are polled by the scheduler; here we only pass time. The host thread
        // has nothing else to do, so it spins (yielding) rather than sleeping: the next
        // iteration is enqueued within ~1-2 us of the device finishing the previous one.
        while (now_ms() < until_ms) {
            for (int q = 0; q < 3; ++q)
                if (!done_q[q].empty() && (done_q[q].front().done || cudaEventQuery(done_q[q].front().ev) == cudaSuccess))
                    return;
            std::this_thread::yield();
        }
    }

    void finish() override {
        check_cuda(cudaSetDevice(E.opt.ppi_device), "cudaSetDevice");
        check_cuda(cudaStreamSynchronize(E.s_ppi), "sync ppi");
        check_cuda(cudaSetDevice(E.opt.cpi_device), "cudaSetDevice");
        check_cuda(cudaStreamSynchronize(E.s_copy), "sync copy");
        check_cuda(cudaStreamSynchronize(E.s_cpi), "sync cpi");
        if (E.s_cpi_full) check_cuda(cudaStreamSynchronize(E.s_cpi_full), "sync cpi (lent)");
        float ms = 0.f;
        cudaEvent_t end;
        check_cuda(cudaEventCreate(&end), "event");
        check_cuda(cudaEventRecord(end, cpi_stream ? cpi_stream : E.s_cpi), "event");
        check_cuda(cudaEventSynchronize(end), "sync");
        check_cuda(cudaEventElapsedTime(&ms, t0_cpi, end), "elapsed");
        cudaEventDestroy(end);
        gpu_ms = ms;
        E.cpi->set_launch(E.s_cpi, E.cpi_ctas, E.s_cpi_side);
        if (opts.host_tokens) {
            check_cuda(cudaMemcpy(opts.host_tokens, E.tok_cpi.out_tok.p, static_cast<size_t>(total_out) * 4,
                                  cudaMemcpyDeviceToHost),
                       "tokens D2H");
            d2h_bytes += total_out * 4;
            if (!E.colocated) {  // requests decoded on the low side (dp, disagg-hl) left their tokens there
                std::vector<int> low(static_cast<size_t>(total_out));
                check_cuda(cudaSetDevice(E.opt.ppi_device), "cudaSetDevice");
                check_cuda(cudaMemcpy(low.data(), E.tok_ppi.out_tok.p, low.size() * 4, cudaMemcpyDeviceToHost),
                           "tokens D2H (low side)");
                d2h_bytes += total_out * 4;
                for (size_t i = 0; i < low.size(); ++i)
                    if (opts.host_tokens[i] < 0) opts.host_tokens[i] = low[i];
            }
        }
        if (opts.host_logits) {
            check_cuda(cudaMemcpy(opts.host_logits, logits_buf.p, static_cast<size_t>(total_out) * E.spec.vocab * 4,
                                  cudaMemcpyDeviceToHost),
                       "logits D2H");
        }
        E.cpi->collect_stats();
        E.ppi->collect_stats();
    }

    std::string stats() const {
        std::ostringstream s;
        auto ks = [&](const char* name, const gpu::KernelStat& k, bool comma = true) {
            s << "\"" << name << "\": {\"launches\": " << k.launches << ", \"ms\": " << k.ms
              << ", \"bytes\": " << k.bytes << ", \"flops\": " << k.flops << "}" << (comma ? ", " : "");
        };
        s.precision(10);
        s << "{\"gpu_ms\": " << gpu_ms << ", \"cpi_busy_ms\": " << cpi_busy_ms << ", \"cpi_iterations\": " << iters << ", \"cpi_lent_iterations\": " << lent_iters << ", \"iter_rows\": " << iter_rows
          << ", \"decode_rows\": " << decode_rows << ", \"decode_keys\": " << decode_keys
          << ", \"chunk_rows\": " << chunk_rows << ", \"prefill_tokens\": " << prefill_tokens
          << ", \"handoffs\": " << handoffs << ", \"handoff_bytes\": " << handoff_bytes
          << ", \"h2d_bytes\": " << h2d_bytes << ", \"d2h_bytes\": " << d2h_bytes
          << ", \"gpu_launches\": " << (E.cpi->launches - launches0_cpi) + (E.ppi->launches - launches0_ppi) + copy_launches
          << ", \"colocated\": " << (E.colocated ? "true" : "false") << ", \"sms\": " << E.sms
          // bytes one pass streams regardless of its rows (all layers' weights + LM head) and
          // the KV bytes one token adds (all layers): the pass-level roofline terms
          << ", \"pass_weight_bytes\": "
          << E.spec.weight_bytes() - 2LL * E.spec.vocab * E.spec.hidden
          << ", \"kv_bytes_per_token\": " << E.spec.kv_bytes_per_token()
          << ", \"partition\": " << E.describe(false) << ", \"cpi\": {";
        ks("decode_attn", E.cpi->stat_decode_attn);
        ks("prefill_attn", E.cpi->stat_prefill_attn);
        ks("gemm_stream", E.cpi->stat_gemm_stream);
        ks("gemm_tc", E.cpi->stat_gemm_tc);
        ks("other", E.cpi->stat_other);
        ks("forward", E.cpi->stat_forward, false);
        s << "}, \"ppi\": {";
        ks("prefill_attn", E.ppi->stat_prefill_attn);
        ks("gemm_stream", E.ppi->stat_gemm_stream);
        ks("gemm_tc", E.ppi->stat_gemm_tc);
        ks("other", E.ppi->stat_other);
        ks("forward", E.ppi->stat_forward, false);
        s << "}}";
        return s.str();
    }

  private:
    GpuEngine::Impl& E;
    const Trace& trace;
    const GpuRunOptions& opts;
    std::vector<long long> prompt_off, out_off;
    long long total_in = 0, total_out = 0;
    DeviceBuf logits_buf;  // logits test hook (opts.host_logits)
    int* pinned_prompt = nullptr;
    gpu::Batch batch;
    std::vector<cudaEvent_t> prefill_ev, xfer_ev;
    std::vector<char> xfer_pending;
    std::vector<char> serial_high, chunked_high;  // scheduler instance index -> on the high side
    std::map<int, std::vector<int32_t>> stage_slots;  // rid -> staging slots holding its handed-off KV
    std::map<int, bool> stage_tok;                    // rid -> the prefill side sampled its first token
    std::vector<int32_t> stage_free;
    bool staging_ready = false, stage_side = false;
    int32_t stage_lo = 0;  // lowest staging block id of the prefill-side pool
    cudaEvent_t stage_fence = nullptr;
    bool lending = false;
    // per side [low, high]: block-reuse fences and the latest work launched there
    cudaEvent_t serial_fence[2] = {}, chunked_fence[2] = {}, last_iter[2] = {};
    struct Tick {
        uint64_t ticket;
        cudaEvent_t ev;
        bool done;
        double t;
        cudaEvent_t start;  // CPI iterations: event recorded before the first kernel
        bool high;          // recorded on the high side's device (its t0 is the time base)
    };
    cudaEvent_t iter_start = nullptr;
    cudaStream_t cpi_stream = nullptr;  // stream the latest CPI iteration went to
    bool last_lent = false;
    long long lent_iters = 0;
    std::deque<Tick> done_q[3];
    std::vector<cudaEvent_t> spare[2];  // reusable timing events per side's device
    uint64_t next_ticket = 1;
    cudaEvent_t t0_cpi = nullptr, t0_ppi = nullptr;
    std::chrono::steady_clock::time_point host_t0;

  public:
    long long launches0_cpi = 0, launches0_ppi = 0, copy_launches = 0;
    double gpu_ms = 0, cpi_busy_ms = 0;
    long long iters = 0, iter_rows = 0, decode_rows = 0, decode_keys = 0, chunk_rows = 0, prefill_tokens = 0;
    long long handoffs = 0;
    double handoff_bytes = 0, h2d_bytes = 0, d2h_bytes = 0;

  private:
    // One reusable event per request role, re-recorded (never timing-critical).
    cudaEvent_t record(cudaStream_t s, cudaEvent_t ev) {
        if (!ev) check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        check_cuda(cudaEventRecord(ev, s), "event record");
        return ev;
    }
    // `high`: the side whose device `s` belongs to (and is current).
    uint64_t complete(cudaStream_t s, int q, bool high) {
        const uint64_t t = next_ticket++;
        if (!E.opt.wall) return t;  // virtual clock: completions come from the cost model
        cudaEvent_t ev = take_event(high);
        check_cuda(cudaEventRecord(ev, s), "event record");
        done_q[q].push_back(Tick{t, ev, false, 0.0, q == 2 ? iter_start : nullptr, high});
        if (q == 2) iter_start = nullptr;
        return t;
    }
    // A timing event on `high`'s device (the caller has made that device current).
    cudaEvent_t take_event(bool high) {
        cudaEvent_t ev;
        if (!spare[high].empty()) {
            ev = spare[high].back();
            spare[high].pop_back();
        } else {
            check_cuda(cudaEventCreate(&ev), "event");
        }
        return ev;
    }
};

}  // namespace

GpuEngine::GpuEngine(const std::string& engine_options) : impl_(std::make_unique<Impl>(engine_options)) {}
GpuEngine::~GpuEngine() = default;

std::string GpuEngine::describe(bool probe) { return impl_->describe(probe); }

// Calibration sample: one synthetic forward pass on a worker,
// timed with CUDA events on that worker's stream; median of `reps`.
double GpuEngine::time_pass(const ClusterConfig& cfg, int worker, int n_dec, int dec_ctx, int chunk_len,
                            int chunk_pos0, int reps) {
    Impl& E = *impl_;
    E.prepare(cfg);
    gpu::Worker& W = worker == 0 ? *E.ppi : *E.cpi;
    gpu::KvPool& pool = worker == 0 ? *E.pool_ppi : *E.pool_cpi;
    if (worker != 0) E.cpi->set_launch(E.s_cpi, E.cpi_ctas, E.s_cpi_side);  // as a serve's CPI iterations
    const int dev = worker == 0 ? E.opt.ppi_device : E.opt.cpi_device;
    TokenBufs& tb = worker == 0 && !E.colocated ? E.tok_ppi : E.tok_cpi;
    check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    const long long span = std::max<long long>(chunk_pos0 + chunk_len, dec_ctx) + 16;
    const int n_req = n_dec + 1;
    tb.prompt.ensure(dev, static_cast<size_t>(span) * 4);
    tb.prompt_off.ensure(dev, static_cast<size_t>(n_req) * 8);
    tb.last_tok.ensure(dev, static_cast<size_t>(n_req) * 4);
    tb.out_tok.ensure(dev, static_cast<size_t>(n_req) * 4 + static_cast<size_t>(span) * 4);
    cudaStream_t st = W.stream();
    check_cuda(cudaMemsetAsync(tb.prompt.p, 0, static_cast<size_t>(span) * 4, st), "memset");
    check_cuda(cudaMemsetAsync(tb.prompt_off.p, 0, static_cast<size_t>(n_req) * 8, st), "memset");
    check_cuda(cudaMemsetAsync(tb.last_tok.p, 0, static_cast<size_t>(n_req) * 4, st), "memset");
    E.staged_hash = 0;
    // disjoint block ranges per sequence
    long long next = 0;
    auto blocks_for = [&](long long tokens) {
        std::vector<int32_t> b;
        for (long long i = 0; i < (tokens + 15) / 16; ++i) b.push_back(static_cast<int32_t>(next++ % pool.blocks));
        return b;
    };
    gpu::Batch batch;
    std::vector<std::vector<int32_t>> tables;
    tables.reserve(n_dec + 1);
    for (int i = 0; i < n_dec; ++i) {
        tables.push_back(blocks_for(dec_ctx));
        batch.add_decode(i + 1, dec_ctx, tables.back(), i + 1);
    }
    if (chunk_len > 0) {
        tables.push_back(blocks_for(chunk_pos0 + chunk_len));
        batch.add_prefill(0, chunk_pos0, chunk_len, tables.back(), true, 0);
    }
    if (n_dec > 0)
        batch.plan_decode(E.spec.n_kv_heads, gpu::decode_slots(E.spec.n_kv_heads, static_cast<int>(batch.d_len.size()), worker == 0 ? (E.ppi_ctas ? E.ppi_ctas : E.sms) : E.cpi_sm_count()));
    cudaEvent_t a, b;
    check_cuda(cudaEventCreate(&a), "event");
    check_cuda(cudaEventCreate(&b), "event");
    std::vector<float> t;
    // CRONUS_PASS_PRELOAD=1: hold the stream while the host enqueues the pass, so the
    // measurement excludes host launch throughput (compare with the default).
    const char* pre = std::getenv("CRONUS_PASS_PRELOAD");
    const bool preload = pre && pre[0] == '1';
    for (int r = 0; r < reps + 1; ++r) {
        if (preload) check_ck(ck_spin(20000, st), "spin");
        check_cuda(cudaEventRecord(a, st), "event");
        W.forward(batch, pool, static_cast<int*>(tb.prompt.p), static_cast<long long*>(tb.prompt_off.p),
                  static_cast<int*>(tb.last_tok.p), static_cast<int*>(tb.out_tok.p));
        check_cuda(cudaEventRecord(b, st), "event");
        check_cuda(cudaEventSynchronize(b), "sync");
        float ms = 0.f;
        check_cuda(cudaEventElapsedTime(&ms, a, b), "elapsed");
        if (r > 0) t.push_back(ms);  // first pass warms caches / descriptors
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (const char* e = std::getenv("CRONUS_PASS_STATS"); e && e[0] == '1') {  // dev: per-kernel-class split
        W.reset_stats();
        W.set_profiling(true);
        W.forward(batch, pool, static_cast<int*>(tb.prompt.p), static_cast<long long*>(tb.prompt_off.p),
                  static_cast<int*>(tb.last_tok.p), static_cast<int*>(tb.out_tok.p));
        W.collect_stats();
        W.set_profiling(false);
        auto pr = [](const char* n, const gpu::KernelStat& k) {
            if (k.launches)
                std::fprintf(stderr, " %s: n=%lld ms=%.3f GB/s=%.0f", n, k.launches, k.ms, k.bytes / std::max(k.ms, 1e-9) / 1e6);
        };
        std::fprintf(stderr, "[pass stats n_dec=%d ctx=%d chunk=%d]", n_dec, dec_ctx, chunk_len);
        pr("decode_attn", W.stat_decode_attn);
        pr("prefill_attn", W.stat_prefill_attn);
        pr("gemm_stream", W.stat_gemm_stream);
        pr("gemm_tc", W.stat_gemm_tc);
        pr("other", W.stat_other);
        pr("forward", W.stat_forward);
        std::fprintf(stderr, "\n");
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

void GpuEngine::stage(const ClusterConfig& cfg, const Trace& trace) {
    impl_->prepare(cfg);
    GpuRunOptions o;
    impl_->staged_hash = 0;
    PairExecutor ex(*impl_, cfg, trace, o);
    ex.upload();  // synthesizes the prompts on the device and marks them staged
}

void GpuEngine::staged_prompts(int* out, long long n) {
    if (!impl_->staged_hash) throw std::logic_error("staged_prompts: no staged trace");
    if (static_cast<size_t>(n) * 4 > impl_->tok_cpi.prompt.cap)
        throw std::invalid_argument("staged_prompts: more tokens than the staged trace holds");
    check_cuda(cudaSetDevice(impl_->opt.cpi_device), "cudaSetDevice");
    check_cuda(cudaMemcpy(out, impl_->tok_cpi.prompt.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost),
               "prompt D2H");
}

RunReport GpuEngine::run(const ClusterConfig& cfg, const Trace& trace, const GpuRunOptions& opts) {
    // every policy but pp runs on the pair (the scheduler rejects pp: out of scope)
    const auto errs = validate_config(cfg);
    if (!errs.empty() || trace.requests.empty()) return cronus::run(cfg, trace, opts);  // throws the same errors
    impl_->prepare(cfg);
    impl_->cpi->set_profiling(opts.profile || impl_->opt.profile);
    impl_->ppi->set_profiling(opts.profile || impl_->opt.profile);
    impl_->cpi->reset_stats();
    impl_->ppi->reset_stats();
    impl_->cpi->reset_graphs();  // captured passes hold the previous run's buffers
    impl_->ppi->reset_graphs();
    PairExecutor ex(*impl_, cfg, trace, opts);
    ex.upload();
    sched::SchedulerHooks hooks;
    hooks.executor = &ex;
    std::vector<sched::IterRecord> iters;
    hooks.iterations = &iters;
    RunReport rep = sched::run_scheduler(cfg, trace, opts, hooks);
    if (opts.stats_json) {
        // iteration-shape histogram: (chunk?, decoders bucket) -> count, wall ms
        struct Bin {
            long long n = 0;
            double ms = 0;
            long long rows = 0, ctx = 0;
        };
        std::map<std::string, Bin> bins;
        for (const auto& it : iters) {
            const int d = it.n_decode;
            const char* db = d == 0 ? "0" : d <= 16 ? "1-16" : d <= 64 ? "17-64" : d <= 128 ? "65-128" : ">128";
            Bin& b = bins[std::string(it.chunk_len > 0 ? "chunk+" : "decode ") + db];
            b.n++;
            b.ms += it.t_end - it.t_start;
            b.rows += it.n_decode;
            b.ctx += it.decode_ctx_sum;
        }
        std::string js = ex.stats();
        std::ostringstream h;
        h << ", \"iteration_shapes\": {";
        bool first = true;
        for (const auto& [k, b] : bins) {
            // [iterations, wall ms, mean decoders per iteration, mean decode context]
            h << (first ? "" : ", ") << "\"" << k << "\": [" << b.n << ", " << b.ms << ", "
              << static_cast<double>(b.rows) / std::max<long long>(1, b.n) << ", "
              << static_cast<double>(b.ctx) / std::max<long long>(1, b.rows) << "]";
            first = false;
        }
        h << "}}";
        js.pop_back();  // '}'
        *opts.stats_json = js + h.str();
    }
    return rep;
}

RunReport run(const ClusterConfig& cfg, const Trace& trace, const GpuRunOptions& opts,
              const std::string& engine_options) {
    GpuEngine eng(engine_options);
    return eng.run(cfg, trace, opts);
}

}  // namespace cronus
