// include/cronus_capi.h: C-ABI wrappers over the C++ API (host side).
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>

#include "cronus/balancer.hpp"
#include "cronus/costmodel.hpp"
#include "cronus/engine.hpp"
#include "cronus/metrics.hpp"
#include "cronus_capi.h"

namespace {

thread_local std::string g_error;

char* to_c(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.c_str(), s.size() + 1);
    return p;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_error = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_error = e.what();
        return 3;
    }
}

}  // namespace

namespace cronus {
namespace capi {
Trace trace_from(int n, const int* id, const double* arr, const int* in, const int* out, const char* name) {
    Trace t;
    t.name = name ? name : "";
    t.requests.resize(n);
    for (int i = 0; i < n; ++i) t.requests[i] = Request{id[i], arr[i], in[i], out[i]};
    return t;
}
void set_error(const std::string& m) { g_error = m; }
}  // namespace capi
}  // namespace cronus

extern "C" {

const char* cronus_last_error(void) { return g_error.c_str(); }
void cronus_free(char* p) { std::free(p); }
const char* cronus_version(void) { return "cronus-b200 0.1 (sm_100a)"; }

int cronus_synth_trace(int n, double mean_in, double mean_out, int fixed_interval, double interval_ms,
                       long long seed, int* id, double* arrival_ms, int* input_len, int* output_len,
                       char* name, int name_cap) {
    return guarded([&] {
        const cronus::Trace t = cronus::synth_trace(
            n, mean_in, mean_out,
            fixed_interval ? cronus::ArrivalMode::FixedInterval : cronus::ArrivalMode::AllAtZero,
            interval_ms, seed);
        for (int i = 0; i < n; ++i) {
            id[i] = t.requests[i].id;
            arrival_ms[i] = t.requests[i].arrival_ms;
            input_len[i] = t.requests[i].input_len;
            output_len[i] = t.requests[i].output_len;
        }
        if (name && name_cap > 0) {
            std::strncpy(name, t.name.c_str(), name_cap - 1);
            name[name_cap - 1] = 0;
        }
    });
}

unsigned long long cronus_trace_hash(int n, const int* id, const double* arrival_ms, const int* input_len,
                                     const int* output_len) {
    return cronus::trace_hash(cronus::capi::trace_from(n, id, arrival_ms, input_len, output_len, ""));
}

int cronus_run_virtual(const char* cfg_text, int n, const int* id, const double* arrival_ms,
                       const int* input_len, const int* output_len, const char* trace_name, int want_events,
                       int compute_utilization, char** json_out, char** events_out, char** csv_out) {
    return guarded([&] {
        const cronus::ClusterConfig cfg = cronus::parse_config(cfg_text);
        const cronus::Trace t = cronus::capi::trace_from(n, id, arrival_ms, input_len, output_len, trace_name);
        std::ostringstream ev;
        cronus::RunOptions o;
        o.compute_utilization = compute_utilization != 0;
        o.event_log = want_events ? &ev : nullptr;
        const cronus::RunReport rep = cronus::run(cfg, t, o);
        if (json_out) *json_out = to_c(cronus::report_to_json(rep, true));
        if (events_out) *events_out = to_c(ev.str());
        if (csv_out) *csv_out = to_c(cronus::csv_row(rep));
    });
}

int cronus_choose_split(const char* cfg_text, int n_decode, long long decode_ctx_sum, long long free_kv_blocks,
                        int max_batched_tokens, int input_len, int* partial_len, double* t_prefill,
                        double* t_chunked, int* flags) {
    return guarded([&] {
        const cronus::ClusterConfig cfg = cronus::parse_config(cfg_text);
        cronus::CpiStats st;
        st.n_decode = n_decode;
        st.decode_ctx_sum = decode_ctx_sum;
        st.free_kv_blocks = free_kv_blocks;
        st.max_batched_tokens = max_batched_tokens;
        const cronus::SplitDecision d = cronus::choose_split(cfg.low_gpu, cfg.high_gpu, st, input_len);
        *partial_len = d.partial_len;
        *t_prefill = d.predicted_t_prefill;
        *t_chunked = d.predicted_t_chunked;
        *flags = (d.full_on_ppi ? 1 : 0) | (d.cpi_saturated ? 2 : 0);
    });
}

int cronus_fit(int kind, int n, const double* x0, const double* x1, const double* y, double* coef, double* r2,
               double* mape) {
    return guarded([&] {
        cronus::FitReport rep;
        if (kind == 0) {
            std::vector<cronus::PrefillSample> s;
            for (int i = 0; i < n; ++i) s.push_back({x0[i], y[i]});
            rep = cronus::fit_prefill(s);
        } else {
            std::vector<cronus::ChunkedSample> s;
            for (int i = 0; i < n; ++i) s.push_back({x0[i], x1[i], y[i]});
            rep = cronus::fit_chunked(s);
        }
        for (size_t i = 0; i < rep.coefficients.size(); ++i) coef[i] = rep.coefficients[i];
        *r2 = rep.r2;
        *mape = rep.mape;
    });
}

int cronus_percentile(const double* v, int n, double p, double* out) {
    return guarded([&] { *out = cronus::percentile(std::vector<double>(v, v + n), p); });
}

int cronus_config_roundtrip(const char* cfg_text, char** out) {
    return guarded([&] { *out = to_c(cronus::serialize_config(cronus::parse_config(cfg_text))); });
}

}  // extern "C"
