// SM partitioning of one B200 between the co-located PPI and CPI workers.
//
// The paper's heterogeneity (a low-end GPU running partial prefill next to a
// high-end GPU) is emulated on one device by giving the PPI a fixed set of SMs and
// the CPI the rest, with CUDA green contexts (driver API, resolved at run time via
// cudaGetDriverEntryPoint so the library still loads on machines without a driver):
//   cuDeviceGetDevResource(SM) -> cuDevSmResourceSplitByCount(k) ->
//   cuDevResourceGenerateDesc -> cuGreenCtxCreate -> cuGreenCtxStreamCreate
// Both workers share the device's HBM (weights are one copy) — exactly the
// co-located configuration of BASELINE.json configs[1]. If green contexts are not
// available the engine falls back to capping the PPI GEMM grid (reported).
#include "partition.hpp"

#include <cuda.h>

#include <stdexcept>
#include <string>

namespace cronus {
namespace gpu {

namespace {

template <class F>
F entry(const char* name) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<F>(f);
}

using GetDevResource = CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType);
using SplitByCount = CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned);
using GenerateDesc = CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned);
using GreenCreate = CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned);
using GreenStream = CUresult (*)(CUstream*, CUgreenCtx, unsigned, int);
using GreenDestroy = CUresult (*)(CUgreenCtx);

}  // namespace

SmPartition::~SmPartition() {
    auto destroy = entry<GreenDestroy>("cuGreenCtxDestroy");
    if (ppi_stream) cudaStreamDestroy(ppi_stream);
    if (cpi_stream) cudaStreamDestroy(cpi_stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (cpi_side_stream) cudaStreamDestroy(cpi_side_stream);
    if (destroy) {
        if (g_ppi) destroy(static_cast<CUgreenCtx>(g_ppi));
        if (g_cpi) destroy(static_cast<CUgreenCtx>(g_cpi));
    }
}

std::unique_ptr<SmPartition> make_sm_partition(int device, int ppi_sms, int prio_ppi, int prio_cpi) {
    auto get = entry<GetDevResource>("cuDeviceGetDevResource");
    auto split = entry<SplitByCount>("cuDevSmResourceSplitByCount");
    auto desc = entry<GenerateDesc>("cuDevResourceGenerateDesc");
    auto create = entry<GreenCreate>("cuGreenCtxCreate");
    auto stream = entry<GreenStream>("cuGreenCtxStreamCreate");
    if (!get || !split || !desc || !create || !stream) return nullptr;
    CUdevResource all{};
    if (get(static_cast<CUdevice>(device), &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS) return nullptr;
    CUdevResource part{}, rest{};
    unsigned groups = 1;
    if (split(&part, &groups, &all, &rest, 0, static_cast<unsigned>(ppi_sms)) != CUDA_SUCCESS || groups != 1)
        return nullptr;
    auto out = std::make_unique<SmPartition>();
    CUdevResourceDesc d_ppi = nullptr, d_cpi = nullptr;
    if (desc(&d_ppi, &part, 1) != CUDA_SUCCESS || desc(&d_cpi, &rest, 1) != CUDA_SUCCESS) return nullptr;
    CUgreenCtx g1 = nullptr, g2 = nullptr;
    if (create(&g1, d_ppi, static_cast<CUdevice>(device), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return nullptr;
    out->g_ppi = g1;
    if (create(&g2, d_cpi, static_cast<CUdevice>(device), CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS) return nullptr;
    out->g_cpi = g2;
    CUstream s1 = nullptr, s2 = nullptr;
    if (stream(&s1, g1, CU_STREAM_NON_BLOCKING, prio_ppi) != CUDA_SUCCESS) return nullptr;
    out->ppi_stream = reinterpret_cast<cudaStream_t>(s1);
    if (stream(&s2, g2, CU_STREAM_NON_BLOCKING, prio_cpi) != CUDA_SUCCESS) return nullptr;
    out->cpi_stream = reinterpret_cast<cudaStream_t>(s2);
    CUstream s3 = nullptr;
    if (stream(&s3, g2, CU_STREAM_NON_BLOCKING, prio_cpi) != CUDA_SUCCESS) return nullptr;
    out->copy_stream = reinterpret_cast<cudaStream_t>(s3);
    CUstream s4 = nullptr;
    // lower priority than the CPI's main stream: its kernels take the SMs the main stream's leave
    if (stream(&s4, g2, CU_STREAM_NON_BLOCKING, prio_ppi) != CUDA_SUCCESS) return nullptr;
    out->cpi_side_stream = reinterpret_cast<cudaStream_t>(s4);
    out->ppi_sms = static_cast<int>(part.sm.smCount);
    out->cpi_sms = static_cast<int>(rest.sm.smCount);
    return out;
}

}  // namespace gpu
}  // namespace cronus
