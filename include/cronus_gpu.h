/* cronus_gpu.h — C-ABI of the B200 serving engine (libcronus_b200.so).
 *
 * Wraps cronus::GpuEngine (include/cronus/gpu.hpp): the reference's `run`
 * (proj/include/cronus/engine.hpp:18) with its three cost-model work sites
 * (engine.cpp:473, :551, :580) executed on B200 workers. Return codes as in
 * cronus_capi.h (0 ok, 1 invalid argument, 2 runtime error, 3 other).
 */
#ifndef CRONUS_GPU_H
#define CRONUS_GPU_H

#ifdef __cplusplus
extern "C" {
#endif

/* engine_options: `key = value` lines (see include/cronus/gpu.hpp). Allocates the
 * model weights on the worker device(s). */
int cronus_engine_create(const char* engine_options, void** engine_out);
void cronus_engine_destroy(void* engine);

/* Serve one trace. host_prompt (nullable): concatenated prompt tokens in trace
 * order (e2e mode: copied H2D inside the call); host_tokens (nullable): receives
 * the generated tokens (output_len per request, concatenated). Outputs are the
 * reference's report_to_json(rep, true), event log and csv_row, plus a stats JSON
 * (kernel timings when profiling). flags: bit0 = write the event log, bit1 = time
 * kernel classes with CUDA events during this run. */
int cronus_engine_serve(void* engine, const char* cfg_text, int n, const int* id, const double* arrival_ms,
                        const int* input_len, const int* output_len, const char* trace_name,
                        const int* host_prompt, int* host_tokens, int flags, char** json_out,
                        char** events_out, char** csv_out, char** stats_out);

/* Test hook: serve() (prompts synthesized on the device, no event log) that also
 * returns the fp32 logits each generated token was sampled from, host_logits =
 * [sum(output_len)][vocab] in host_tokens order. Co-located pairs only. */
int cronus_engine_serve_logits(void* engine, const char* cfg_text, int n, const int* id, const double* arrival_ms,
                               const int* input_len, const int* output_len, const char* trace_name, int* host_tokens,
                               float* host_logits, char** json_out);

/* Pre-synthesize the trace's prompt tokens on the device (see GpuEngine::stage). */
int cronus_engine_stage(void* engine, const char* cfg_text, int n, const int* id, const double* arrival_ms,
                        const int* input_len, const int* output_len);

/* Host copy of the staged prompt tokens (n = total input tokens of the staged trace). */
int cronus_engine_staged_prompts(void* engine, int* out, long long n);

/* Calibration sample (see GpuEngine::time_pass): median ms of one forward pass. */
int cronus_engine_time_pass(void* engine, const char* cfg_text, int worker, int n_dec, int dec_ctx, int chunk_len,
                            int chunk_pos0, int reps, double* ms_out);

/* JSON description of the engine's SM partition; probe = 1 launches an %smid probe
 * on each worker stream and reports the SMs actually used. */
int cronus_engine_describe(void* engine, int probe, char** json_out);

/* The engine's decode-attention planner (gpu::Batch::plan_decode) on n context lengths for
 * `slots` resident CTAs: writes the ck_attn_decode_tma work list (work_out: capacity
 * work_cap entries) and seq_item0 (item0_out[n]); *n_work_out, *cluster_out. Host only
 * (tools and tests drive the kernel with the production plan through it). */
int cronus_plan_decode(const int* lens, int n, int n_kv_heads, int slots, int* work_out, int work_cap,
                       int* item0_out, int* n_work_out, int* cluster_out);

#ifdef __cplusplus
}
#endif

#endif /* CRONUS_GPU_H */
