/* C-ABI of libcronus_b200.so — the boundary a non-C++ caller (Python ctypes in
 * tests/ and bench.py, or any FFI) binds. Plain pointers and sizes only.
 *
 * Each entry point wraps one function of the reference's C++ API
 * (proj/include/cronus/*.hpp); the C++ API itself (include/cronus/*.hpp) is the
 * primary drop-in boundary for C++ callers. Return codes: 0 ok,
 * 1 std::invalid_argument, 2 std::runtime_error, 3 other error; the message is
 * available from cronus_last_error(). Strings returned through char** are
 * malloc'd and released with cronus_free().
 */
#ifndef CRONUS_CAPI_H
#define CRONUS_CAPI_H

#ifdef __cplusplus
extern "C" {
#endif

const char* cronus_last_error(void);
void cronus_free(char* p);
const char* cronus_version(void);

/* trace.hpp:24 synth_trace. Arrays have n entries; name gets the trace name. */
int cronus_synth_trace(int n, double mean_in, double mean_out, int fixed_interval,
                       double interval_ms, long long seed, int* id, double* arrival_ms,
                       int* input_len, int* output_len, char* name, int name_cap);

/* trace.hpp:27 trace_hash. */
unsigned long long cronus_trace_hash(int n, const int* id, const double* arrival_ms,
                                     const int* input_len, const int* output_len);

/* engine.hpp:18 run() on the virtual clock, no device work (replaces the CPU
 * simulator call; bit-identical outputs). Outputs: report_to_json(rep, true),
 * the event log, csv_row(rep). Any output pointer may be NULL. */
int cronus_run_virtual(const char* cfg_text, int n, const int* id, const double* arrival_ms,
                       const int* input_len, const int* output_len, const char* trace_name,
                       int want_events, int compute_utilization, char** json_out,
                       char** events_out, char** csv_out);

/* balancer.hpp:31 choose_split; profiles come from config text (low/high). flags:
 * bit0 full_on_ppi, bit1 cpi_saturated. */
int cronus_choose_split(const char* cfg_text, int n_decode, long long decode_ctx_sum,
                        long long free_kv_blocks, int max_batched_tokens, int input_len,
                        int* partial_len, double* t_prefill, double* t_chunked, int* flags);

/* costmodel.hpp:38-39 fit_prefill (kind 0: x0 = len) / fit_chunked (kind 1:
 * x0 = prefill_ctx, x1 = decode_ctx_sum). coef receives 2 or 3 values. */
int cronus_fit(int kind, int n, const double* x0, const double* x1, const double* y,
               double* coef, double* r2, double* mape);

/* metrics.hpp:44 percentile (nearest rank, p in (0, 1]) -> *out. Errors as in the
 * reference (std::invalid_argument for an empty set or p outside (0, 1]) come back as a
 * non-zero return with cronus_last_error() set. */
int cronus_percentile(const double* v, int n, double p, double* out);

/* config round trip (model.hpp:78-80): parse then serialize. */
int cronus_config_roundtrip(const char* cfg_text, char** out);

#ifdef __cplusplus
}
#endif

#endif /* CRONUS_CAPI_H */
