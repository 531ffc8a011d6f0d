// The serving scheduler behind cronus::run — a deterministic event-driven core
// whose decisions reproduce the reference simulator bit-for-bit on the virtual
// clock (reference proj/src/engine.cpp:152-1033), restructured for a device
// backend:
//   * per-request state lives in one flat table indexed by trace position, so
//     iteration bookkeeping is O(batch) instead of the reference's O(n^2)
//     find-per-decoder (engine.cpp:483-487);
//   * every instance owns a paged KV block pool with deterministic lowest-free-id
//     allocation; physical block tables track the reference's ledger
//     (blocks(req) = ceil((done_tok + emitted) / N), engine.cpp:522-531) exactly;
//   * the three work sites call an Executor (executor.hpp) instead of only
//     pricing the work, and the clock is either virtual (cost model) or the
//     device's completion timestamps.
#pragma once

#include <cstdint>
#include <deque>
#include <functional>
#include <map>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "cronus/engine.hpp"
#include "cronus/policies.hpp"
#include "executor.hpp"

namespace cronus {
namespace sched {

// Lowest-free-id block allocator over [0, capacity). Lazy: ids are minted in
// order and recycled through a min-heap, so construction is O(1).
class BlockPool {
  public:
    explicit BlockPool(long long capacity = 0) : cap_(capacity) {}
    long long capacity() const { return cap_; }
    long long in_use() const { return in_use_; }
    bool alloc(int32_t& id);
    void release(int32_t id);

  private:
    long long cap_ = 0;
    long long minted_ = 0;
    long long in_use_ = 0;
    std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_;
};

// One record per chunked-instance iteration (diagnostics, bench accounting and the
// GPU parity tests). Captured only when SchedulerHooks::iterations is set.
struct IterRecord {
    int instance = 0;
    double t_start = 0.0;
    double t_end = 0.0;
    int n_decode = 0;
    long long decode_ctx_sum = 0;
    int chunk_rid = -1;
    long long chunk_start = 0;
    long long chunk_len = 0;
    int n_finishers = 0;
    long long alloc_blocks = 0;  // instance ledger right after the iteration
};

struct PrefillRecord {
    int instance = 0;
    int rid = 0;
    long long tokens = 0;
    double t_start = 0.0;
    double t_end = 0.0;
};

struct TransferRecord {
    int rid = 0;
    long long tokens = 0;
    double t_start = 0.0;
    double t_end = 0.0;
};

struct SchedulerHooks {
    Executor* executor = nullptr;  // null: pure virtual-clock simulation
    std::vector<IterRecord>* iterations = nullptr;
    std::vector<PrefillRecord>* prefills = nullptr;
    std::vector<TransferRecord>* transfers = nullptr;
    // Per-request block tables are checked against the reference ledger formula
    // after every ledger update (cheap; on by default).
    bool check_ledger = true;
};

RunReport run_scheduler(const ClusterConfig& cfg, const Trace& trace, const RunOptions& opts,
                        const SchedulerHooks& hooks);

}  // namespace sched
}  // namespace cronus
