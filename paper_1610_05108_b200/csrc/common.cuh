// Shared device/host helpers of the xyz engine (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

namespace xyzb {

typedef uint64_t u64;
typedef uint32_t u32;

struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct data_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct internal_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct guard_error : std::runtime_error {  // xyz::guard_error (errors.hpp:15-18)
    using std::runtime_error::runtime_error;
};

#define XYZB_CUDA(call)                                                                         \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            throw ::xyzb::cuda_error(std::string(#call) + ": " + cudaGetErrorString(e_) +       \
                                     " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")");   \
    } while (0)

#define XYZB_LAUNCH_CHECK() XYZB_CUDA(cudaGetLastError())

// cudaFuncSetAttribute applies to the CURRENT device only. Datasets on
// several devices (and concurrent host threads) launch the same kernels, so
// every (kernel, device, attribute) keeps the largest value requested so far,
// raised under a lock before the launch that needs it (dynamic shared memory
// limits and cluster opt-ins only ever need to grow).
inline void func_attr(const void* fn, cudaFuncAttribute attr, int value) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int>, int> cur;
    int dev = 0;
    XYZB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(fn, dev, int(attr));
    const auto it = cur.find(key);
    if (it != cur.end() && it->second >= value) return;
    XYZB_CUDA(cudaFuncSetAttribute(fn, attr, value));
    cur[key] = value;
}
template <class F>
inline void func_smem(F* fn, size_t bytes) {
    func_attr(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
}

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

__host__ __device__ inline u64 ceil_div(u64 a, u64 b) { return (a + b - 1) / b; }
__host__ __device__ inline u64 minu(u64 a, u64 b) { return a < b ? a : b; }

#ifdef __CUDACC__
__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
#endif

} // namespace xyzb
