// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the *unmodified* reference simulator
// (/root/reference/proj/src/*.cpp, compiled out-of-tree by oracle/Makefile into
// oracle/_ref/libcronus_ref.so). It lets the Python tests, smoke() and the
// bench's reference arm call the reference's own public API
// (proj/include/cronus/engine.hpp:18 `cronus::run`, balancer.hpp:31
// `choose_split`, trace.hpp:24 `synth_trace`, costmodel.hpp:38-39 `fit_*`)
// through plain pointers. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load it.
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>

#include "cronus/balancer.hpp"
#include "cronus/costmodel.hpp"
#include "cronus/engine.hpp"
#include "cronus/metrics.hpp"
#include "cronus/model.hpp"
#include "cronus/trace.hpp"

namespace {

thread_local std::string g_err;

char* dup_str(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size() + 1);
    return p;
}

cronus::Trace make_trace(int n, const int* id, const double* arr, const int* in,
                         const int* out, const char* name) {
    cronus::Trace t;
    t.name = name ? name : "";
    t.requests.resize(n);
    for (int i = 0; i < n; ++i) t.requests[i] = {id[i], arr[i], in[i], out[i]};
    return t;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// 0 ok, 1 invalid_argument, 2 runtime_error, 3 other
int ref_run(const char* cfg_text, int n, const int* id, const double* arr, const int* in,
            const int* out, const char* trace_name, int want_events, int compute_util,
            char** json_out, char** events_out, char** csv_out) {
    try {
        cronus::ClusterConfig cfg = cronus::parse_config(cfg_text);
        cronus::Trace t = make_trace(n, id, arr, in, out, trace_name);
        std::ostringstream ev;
        cronus::RunOptions opts;
        opts.compute_utilization = compute_util != 0;
        if (want_events) opts.event_log = &ev;
        cronus::RunReport rep = cronus::run(cfg, t, opts);
        if (json_out) *json_out = dup_str(cronus::report_to_json(rep, true));
        if (events_out) *events_out = dup_str(ev.str());
        if (csv_out) *csv_out = dup_str(cronus::csv_row(rep));
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

int ref_synth_trace(int n, double mean_in, double mean_out, int fixed_interval,
                    double interval_ms, long long seed, int* id, double* arr, int* in,
                    int* out, char* name, int name_cap) {
    try {
        cronus::Trace t = cronus::synth_trace(
            n, mean_in, mean_out,
            fixed_interval ? cronus::ArrivalMode::FixedInterval : cronus::ArrivalMode::AllAtZero,
            interval_ms, seed);
        for (int i = 0; i < n; ++i) {
            id[i] = t.requests[i].id;
            arr[i] = t.requests[i].arrival_ms;
            in[i] = t.requests[i].input_len;
            out[i] = t.requests[i].output_len;
        }
        if (name && name_cap > 0) {
            std::strncpy(name, t.name.c_str(), name_cap - 1);
            name[name_cap - 1] = 0;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

unsigned long long ref_trace_hash(int n, const int* id, const double* arr, const int* in,
                                  const int* out) {
    return cronus::trace_hash(make_trace(n, id, arr, in, out, ""));
}

// low/high profiles are given as config text (the reference parser fills them).
int ref_choose_split(const char* cfg_text, int n_decode, long long decode_ctx_sum,
                     long long free_kv_blocks, int max_batched_tokens, int input_len,
                     int* partial_len, double* t_prefill, double* t_chunked, int* flags) {
    try {
        cronus::ClusterConfig cfg = cronus::parse_config(cfg_text);
        cronus::CpiStats st;
        st.n_decode = n_decode;
        st.decode_ctx_sum = decode_ctx_sum;
        st.free_kv_blocks = free_kv_blocks;
        st.max_batched_tokens = max_batched_tokens;
        cronus::SplitDecision d = cronus::choose_split(cfg.low_gpu, cfg.high_gpu, st, input_len);
        *partial_len = d.partial_len;
        *t_prefill = d.predicted_t_prefill;
        *t_chunked = d.predicted_t_chunked;
        *flags = (d.full_on_ppi ? 1 : 0) | (d.cpi_saturated ? 2 : 0);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// kind 0: prefill (x0 = len); kind 1: chunked (x0 = prefill_ctx, x1 = decode_ctx_sum)
int ref_fit(int kind, int n, const double* x0, const double* x1, const double* y,
            double* coef, double* r2, double* mape) {
    try {
        cronus::FitReport rep;
        if (kind == 0) {
            std::vector<cronus::PrefillSample> s(n);
            for (int i = 0; i < n; ++i) s[i] = {x0[i], y[i]};
            rep = cronus::fit_prefill(s);
        } else {
            std::vector<cronus::ChunkedSample> s(n);
            for (int i = 0; i < n; ++i) s[i] = {x0[i], x1[i], y[i]};
            rep = cronus::fit_chunked(s);
        }
        for (size_t i = 0; i < rep.coefficients.size(); ++i) coef[i] = rep.coefficients[i];
        *r2 = rep.r2;
        *mape = rep.mape;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

double ref_percentile(const double* v, int n, double p) {
    return cronus::percentile(std::vector<double>(v, v + n), p);
}

}  // extern "C"
