// Cronus balancer, paper Alg. 1; observable behaviour follows
// reference proj/src/balancer.cpp:12-76 (guards, candidate grid, strict-< argmin,
// FP64 expression order — the split point is a bit-exact parity target).
//
// The candidate sweep is the only per-request host cost on the admission path:
// 512 candidates x ~12 flops. It runs once per dispatched request, off the GPU
// critical path (the CPI keeps iterating while the frontend admits).
#include <cmath>
#include <stdexcept>

#include "cronus/balancer.hpp"

namespace cronus {

namespace {
constexpr int kGrid = 512;

void require_positive_len(int input_len) {
    if (input_len < 1) throw std::invalid_argument("input_len must be >= 1");
}

SplitDecision whole_prompt_on_ppi(const GpuProfile& low, int input_len) {
    SplitDecision d;
    d.partial_len = input_len;
    d.predicted_t_prefill = prefill_time(low, input_len);
    d.predicted_t_chunked = 0.0;
    return d;
}
}  // namespace

std::vector<int> candidate_lengths(int input_len) {
    require_positive_len(input_len);
    std::vector<int> lens(kGrid);
    for (int i = 0; i < kGrid; ++i) {
        const long long scaled = static_cast<long long>(i + 1) * input_len;
        lens[i] = static_cast<int>((scaled + kGrid - 1) / kGrid);  // ceil
    }
    return lens;
}

SplitDecision choose_split(const GpuProfile& low, const GpuProfile& high, const CpiStats& stats,
                           int input_len) {
    require_positive_len(input_len);

    // Guard 1: the CPI could not even hold the prompt's KV -> no split.
    const long long prompt_blocks = (input_len + high.kv_block_size - 1) / high.kv_block_size;
    if (stats.free_kv_blocks < prompt_blocks) {
        SplitDecision d = whole_prompt_on_ppi(low, input_len);
        d.full_on_ppi = true;
        return d;
    }
    // Guard 2: decoders consume the whole token budget -> no chunk slot.
    const long long per_iter = static_cast<long long>(stats.max_batched_tokens) - stats.n_decode;
    if (per_iter <= 0) {
        SplitDecision d = whole_prompt_on_ppi(low, input_len);
        d.cpi_saturated = true;
        return d;
    }

    // Per-iteration CPI cost that does not depend on the candidate.
    const double decode_term = high.chunked_k_ctxd * static_cast<double>(stats.decode_ctx_sum);
    const std::vector<int> lens = candidate_lengths(input_len);
    SplitDecision best;
    double best_gap = 0.0;
    bool have = false;
    for (int i = 0; i < kGrid; ++i) {
        const long long lp = lens[i];
        const long long rest = input_len - lp;
        const double t_ppi = prefill_time(low, static_cast<double>(lp));
        long long iters = (rest + per_iter - 1) / per_iter;
        if (iters < 1) iters = 1;  // lp == input_len: one zero-budget handoff iteration
        const long long last_ctx = lp + (rest / per_iter) * per_iter;
        // Arithmetic series of iteration times from the first to the last chunk,
        // grouped exactly as (k_ctxp*(L+l_last)/2 + k_ctxd*ctxd + b) * n_iter.
        const double t_cpi =
            iters * (high.chunked_k_ctxp * (input_len + last_ctx) / 2.0 + decode_term + high.chunked_b);
        const double gap = std::fabs(t_ppi - t_cpi);
        if (!have || gap < best_gap) {
            have = true;
            best_gap = gap;
            best.partial_len = static_cast<int>(lp);
            best.predicted_t_prefill = t_ppi;
            best.predicted_t_chunked = t_cpi;
        }
    }
    return best;
}

}  // namespace cronus
