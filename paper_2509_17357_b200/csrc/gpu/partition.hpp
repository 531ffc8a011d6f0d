// SM partitioning of a device between co-located workers (see partition.cpp).
#pragma once

#include <cuda_runtime.h>

#include <memory>

namespace cronus {
namespace gpu {

struct SmPartition {
    void* g_ppi = nullptr;  // CUgreenCtx
    void* g_cpi = nullptr;
    cudaStream_t ppi_stream = nullptr;  // kernels launched here run on ppi_sms SMs only
    cudaStream_t cpi_stream = nullptr;  // ... and here on the remaining cpi_sms SMs
    cudaStream_t copy_stream = nullptr; // handoff copies, inside the CPI partition
    cudaStream_t cpi_side_stream = nullptr;  // CPI kernels overlapped with the main chain (same SMs)
    int ppi_sms = 0, cpi_sms = 0;
    ~SmPartition();
};

// nullptr when green contexts are unavailable (old driver) or the split is invalid
// (ppi_sms must be a multiple of 8 on sm_100).
std::unique_ptr<SmPartition> make_sm_partition(int device, int ppi_sms, int prio_ppi, int prio_cpi);

}  // namespace gpu
}  // namespace cronus
