// The executor seam: the three places where the reference simulator prices GPU
// work with a cost formula are where the B200 engine launches real work.
//
//   reference call site (proj/src/engine.cpp)     work item here
//   :551 prefill_time(low, L_p)   serial prefill   PrefillWork   (PPI partial prefill)
//   :580 transfer_time(link, L_p) KV handoff       TransferWork  (NVLink / D2D block copy)
//   :473 chunked_iter_time(...)   CPI iteration    IterWork      (mixed chunk + decode batch)
//
// Clock modes:
//   * Virtual (lockstep): the scheduler advances by cost-model time exactly as the
//     oracle does; every work item is still launched on the device, asynchronously
//     and in dependency order, so the GPU executes precisely the oracle's schedule.
//   * Wall: the same scheduler is driven by device completion timestamps (CUDA
//     events); this is the mode that measures req/s, TTFT and TBT on B200.
#pragma once

#include <cstdint>
#include <vector>

namespace cronus {
namespace sched {

// Serial (PPI / pure-prefill) instance: prefill prompt tokens [0, tokens) of one
// request into `blocks` of that instance's KV pool. If `sample_last`, also run the
// LM head on the last row (L_p == L_in: the first output token comes from the PPI).
struct PrefillWork {
    int instance = 0;
    int rid = 0;  // index into the trace
    long long tokens = 0;
    bool sample_last = false;
    const std::vector<int32_t>* blocks = nullptr;
};

// KV handoff of the first `tokens` positions of request `rid`: src blocks on the
// prefill instance, dst blocks on the chunked instance (same count, ceil(tokens/N)).
struct TransferWork {
    int rid = 0;
    long long tokens = 0;
    int src_instance = 0;
    int dst_instance = 0;
    const std::vector<int32_t>* src_blocks = nullptr;
    const std::vector<int32_t>* dst_blocks = nullptr;
};

struct DecodeRow {
    int rid = 0;
    long long ctx = 0;  // keys attended = need + emitted; row position = ctx - 1
    const std::vector<int32_t>* blocks = nullptr;
};

// One chunked-instance iteration (reference engine.cpp:437-480 composition):
// every decoder contributes one row; at most one prefill chunk contributes
// `chunk_len` rows at positions [chunk_start, chunk_start + chunk_len); handoff
// finishers contribute no rows (their first token was sampled by the PPI).
struct IterWork {
    int instance = 0;
    std::vector<DecodeRow> decoders;
    int chunk_rid = -1;
    long long chunk_start = 0;
    long long chunk_len = 0;
    bool chunk_samples = false;  // chunk completes the prompt -> LM head on its last row
    const std::vector<int32_t>* chunk_blocks = nullptr;
    std::vector<int> finishers;  // zero-row entries emitting their PPI-sampled token
};

// A finished device operation (wall-clock mode).
struct Completion {
    uint64_t ticket = 0;
    double t_ms = 0.0;  // completion time on the run clock
};

class Executor {
  public:
    virtual ~Executor() = default;

    // Each returns a ticket identifying the launched operation.
    virtual uint64_t prefill(const PrefillWork& w) = 0;
    virtual uint64_t transfer(const TransferWork& w) = 0;
    virtual uint64_t iteration(const IterWork& w) = 0;
    // KV blocks of `rid` on `instance` were released by the ledger; the device may
    // reuse them once every operation launched so far that touches them is done.
    virtual void release(int instance, int rid) { (void)instance; (void)rid; }

    // --- wall-clock mode -------------------------------------------------------
    virtual bool wall_clock() const { return false; }
    // Current time on the run clock (ms since start()).
    virtual double now_ms() { return 0.0; }
    // Non-blocking: the next finished operation, in completion order.
    virtual bool poll(Completion& out) { (void)out; return false; }
    // Block until something finishes or the run clock reaches `until_ms`.
    virtual void wait(double until_ms) { (void)until_ms; }

    virtual void start() {}
    // Drain all outstanding device work (end of run).
    virtual void finish() {}
};

}  // namespace sched
}  // namespace cronus
