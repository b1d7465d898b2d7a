// Shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <mutex>
#include <set>
#include <string>
#include <utility>

#include "errors.hpp"

#define NRR_CUDA_CHECK(expr)                                                              \
    do {                                                                                  \
        const cudaError_t nrr_e_ = (expr);                                                \
        if (nrr_e_ != cudaSuccess)                                                        \
            throw ::nrr_b200::CudaError(std::string("CUDA error: ") +                     \
                                        cudaGetErrorString(nrr_e_) + " at " __FILE__ ":" + \
                                        std::to_string(__LINE__));                        \
    } while (0)

namespace nrr_b200 {

// Opt a kernel into the device's full dynamic shared memory, once per
// (kernel, device). The attribute is process-global: setting it per launch to
// the launch's own size races when several contexts launch the same kernel
// from several host threads (config 3 batches), so it is set to the maximum.
inline void allow_max_smem(const void* fn) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    NRR_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (!done.insert({fn, dev}).second) return;
    int optin = 0;
    NRR_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    NRR_CUDA_CHECK(cudaFuncGetAttributes(&fa, fn));
    NRR_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        optin - static_cast<int>(fa.sharedSizeBytes)));
}

constexpr int kWarp = 32;

// Fixed-size grids keep every two-level reduction in the same order on every
// run and every device, which makes the energies bitwise reproducible
// (reference README.md:181-182, "deterministic reduction order").
constexpr int kTermBlocks = 296;  // 2 x 148 SMs
constexpr int kTermThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// deterministic block sum of one value per thread (fixed tree); result valid
// in thread 0. `sh` needs blockDim.x/32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// atomic max for non-negative doubles via their IEEE bit patterns
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace nrr_b200
