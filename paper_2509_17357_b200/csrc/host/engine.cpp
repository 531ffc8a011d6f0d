// cronus/engine.hpp: the drop-in entry point and the standalone saturation
// diagnostics (reference proj/src/engine.cpp:1030-1133).
#include <algorithm>
#include <deque>

#include "cronus/costmodel.hpp"
#include "cronus/engine.hpp"
#include "scheduler.hpp"

namespace cronus {

RunReport run(const ClusterConfig& cfg, const Trace& trace, const RunOptions& opts) {
    sched::SchedulerHooks hooks;  // virtual clock, no device work
    return sched::run_scheduler(cfg, trace, opts, hooks);
}

namespace {

long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

// Saturation run of one chunked instance with the whole trace queued at t=0
// (reference engine.cpp:1051-1121). `decode_only` starts every request with its
// KV present and first token emitted (the disaggregated decode instance).
double saturate(const GpuProfile& g, int budget, const Trace& trace, bool decode_only) {
    struct Job {
        int in, out;
        long long prefilled;
        int emitted;
        long long life;
    };
    std::deque<Job> queue;
    for (const Request& q : trace.requests) {
        const long long life = cdiv(q.input_len + q.output_len, g.kv_block_size);
        if (life > g.kv_blocks_capacity) continue;
        queue.push_back(Job{q.input_len, q.output_len, decode_only ? q.input_len : 0, decode_only ? 1 : 0, life});
    }
    std::vector<Job> live;
    long long reserved = 0;
    double clock = 0.0;
    int served = 0;
    auto admit = [&] {
        while (!queue.empty() && static_cast<long long>(live.size()) < budget &&
               reserved + queue.front().life <= g.kv_blocks_capacity) {
            Job j = queue.front();
            queue.pop_front();
            if (j.emitted >= j.out) {  // single-token request: done on arrival
                ++served;
                continue;
            }
            reserved += j.life;
            live.push_back(j);
        }
    };
    admit();
    while (!live.empty()) {
        int n_d = 0;
        long long ctx = 0;
        Job* head = nullptr;
        for (Job& j : live) {
            if (j.prefilled == j.in) {
                if (j.emitted >= 1) {
                    ++n_d;
                    ctx += j.in + j.emitted;
                }
            } else if (!head) {
                head = &j;
            }
        }
        const long long chunk = head ? std::min<long long>(budget - n_d, head->in - head->prefilled) : 0;
        const double pctx = chunk > 0 ? static_cast<double>(head->prefilled + chunk) : 0.0;
        clock += chunked_iter_time(g, pctx, static_cast<double>(ctx));
        if (head) head->prefilled += chunk;
        for (Job& j : live)
            if (j.prefilled == j.in) j.emitted++;
        size_t keep = 0;
        for (size_t i = 0; i < live.size(); ++i) {
            if (live[i].emitted >= live[i].out && live[i].prefilled == live[i].in) {
                reserved -= live[i].life;
                ++served;
            } else {
                live[keep++] = live[i];
            }
        }
        live.resize(keep);
        admit();
    }
    if (served == 0 || clock <= 0) return 0.0;
    return served / (clock / 1000.0);
}

}  // namespace

double standalone_prefill_rps(const GpuProfile& prof, const Trace& trace) {
    double ms = 0.0;
    int n = 0;
    for (const Request& q : trace.requests) {
        if (cdiv(q.input_len, prof.kv_block_size) > prof.kv_blocks_capacity) continue;
        ms += prefill_time(prof, q.input_len);
        ++n;
    }
    return (n == 0 || ms <= 0) ? 0.0 : n / (ms / 1000.0);
}

double standalone_decode_rps(const GpuProfile& prof, int max_batched_tokens, const Trace& trace) {
    return saturate(prof, max_batched_tokens, trace, true);
}

double standalone_chunked_rps(const GpuProfile& prof, int max_batched_tokens, const Trace& trace) {
    return saturate(prof, max_batched_tokens, trace, false);
}

}  // namespace cronus
