// B200 extension of the drop-in API: the same scheduler
// as cronus::run, with its three work sites executed on B200 workers.
//
//   cronus::GpuEngine eng("model = llama3-8b\nclock = wall\nppi_sms = 40\n");
//   cronus::RunReport rep = eng.run(cfg, trace);          // same RunReport as the CPU simulator
//
// Engine options are a separate `key = value` text (never part of ClusterConfig:
// the shared config format rejects unknown keys):
//   model        llama3-8b | qwen2-7b | tiny | tiny-qwen      (default llama3-8b)
//   clock        virtual | wall   virtual: cost-model clock, oracle-identical
//                                 schedule, every batch executed on the GPU;
//                                 wall: scheduler driven by CUDA-event times
//   ppi_device, cpi_device        CUDA devices of the two workers (equal = co-located)
//   ppi_sms      SMs granted to the PPI when co-located (0 = no partition)
//   ppi_chunk    max rows per PPI forward pass (longer prefixes run in sub-passes)
//   cpi_pool_blocks, ppi_pool_blocks   physical KV pool sizes (0 = the profile's capacity)
//   seed, prompt_seed                  weight / prompt-token hash seeds
//   profile      1: time kernel classes with CUDA events (stats JSON)
#pragma once

#include <cstdint>
#include <memory>
#include <string>

#include "cronus/engine.hpp"

namespace cronus {

struct GpuRunOptions : RunOptions {
    // e2e mode: prompt tokens come from this host array (concatenated per request in
    // trace order) and generated tokens are written back to `host_tokens`
    // (concatenated, output_len per request). Null: prompts are synthesized on the
    // device (splitmix64 of (prompt_seed, request id, position)).
    const int32_t* host_prompt = nullptr;
    int32_t* host_tokens = nullptr;
    // Test hook (co-located pair only): the fp32 logits every generated token was sampled
    // from, [total output tokens][vocab] in host_tokens order.
    float* host_logits = nullptr;
    std::string* stats_json = nullptr;  // kernel / iteration statistics
    bool profile = false;               // time kernel classes with CUDA events this run
};

class GpuEngine {
  public:
    explicit GpuEngine(const std::string& engine_options);
    ~GpuEngine();
    GpuEngine(const GpuEngine&) = delete;
    GpuEngine& operator=(const GpuEngine&) = delete;

    RunReport run(const ClusterConfig& cfg, const Trace& trace, const GpuRunOptions& opts = {});

    // JSON: SM partition in effect ("green-context" | "grid-cap" | "none") and SM
    // counts; with probe = true also the SMs each worker's kernels actually ran on.
    std::string describe(bool probe = false);

    // Synthesize this trace's prompt tokens on the device ahead of run() (the
    // "inputs already resident in HBM" measurement); run() then skips that step.
    void stage(const ClusterConfig& cfg, const Trace& trace);
    // The staged trace's prompt tokens copied back to the host (n = total input tokens,
    // trace order): the host buffers of an end-to-end serve (run with host_prompt).
    void staged_prompts(int* out, long long n);

    // Calibration sample: median time (ms, CUDA events) of one forward pass on the
    // PPI (worker 0) or CPI (worker 1) with n_dec decode rows of context dec_ctx and
    // an optional prefill chunk [chunk_pos0, chunk_pos0 + chunk_len).
    double time_pass(const ClusterConfig& cfg, int worker, int n_dec, int dec_ctx, int chunk_len, int chunk_pos0,
                     int reps);

    struct Impl;

  private:
    std::unique_ptr<Impl> impl_;
};

// One-shot convenience: build an engine, serve, tear down.
RunReport run(const ClusterConfig& cfg, const Trace& trace, const GpuRunOptions& opts,
              const std::string& engine_options);

}  // namespace cronus
