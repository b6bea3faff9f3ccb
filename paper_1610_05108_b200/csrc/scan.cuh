// Exclusive scan of a device array whose length lives in device memory (no
// host round trip): fixed persistent grid, reduce -> scan partials -> scan.
#pragma once

#include "common.cuh"

namespace xyzb {
namespace scan {

constexpr int kBlock = 256;
constexpr int kGrid = kSMs * 4;

template <class T>
__device__ __forceinline__ T block_exclusive(T v, T* smem_warp, T* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) smem_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        T x = lane < nw ? smem_warp[lane] : T(0);
        T xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < nw) smem_warp[lane] = xi - x;
        if (lane == nw - 1) smem_warp[32] = xi;
    }
    __syncthreads();
    const T out = smem_warp[wid] + incl - v;
    *total = smem_warp[32];
    __syncthreads();
    return out;
}

template <class T>
__device__ __forceinline__ void chunk_of(u64 n, u64& b, u64& e) {
    const u64 per = (n + gridDim.x - 1) / gridDim.x;
    b = minu(n, per * blockIdx.x);
    e = minu(n, b + per);
}

template <class T>
__global__ void __launch_bounds__(kBlock) reduce_chunks(const T* __restrict__ in, const u32* __restrict__ count,
                                                        T* __restrict__ partial) {
    __shared__ T sw[33];
    u64 b, e;
    chunk_of<T>(*count, b, e);
    T acc = 0;
    for (u64 i = b + threadIdx.x; i < e; i += kBlock) acc += in[i];
    T tot;
    block_exclusive<T>(acc, sw, &tot);
    if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

template <class T>
__global__ void __launch_bounds__(kBlock) scan_partials(T* __restrict__ partial, int n, const u32* __restrict__ count,
                                                        T* __restrict__ out) {
    __shared__ T sw[33];
    // n <= kGrid; each thread handles ceil(n / kBlock) consecutive entries
    const int per = (n + kBlock - 1) / kBlock;
    const int b = threadIdx.x * per, e = min(n, b + per);
    T loc = 0;
    for (int i = b; i < e; ++i) loc += partial[i];
    T tot;
    T run = block_exclusive<T>(loc, sw, &tot);
    for (int i = b; i < e; ++i) {
        const T t = partial[i];
        partial[i] = run;
        run += t;
    }
    if (threadIdx.x == 0) out[*count] = tot;
}

template <class T>
__global__ void __launch_bounds__(kBlock) scan_chunks(const T* __restrict__ in, const u32* __restrict__ count,
                                                      const T* __restrict__ partial, T* __restrict__ out) {
    __shared__ T sw[33];
    u64 b, e;
    chunk_of<T>(*count, b, e);
    T base = partial[blockIdx.x];
    for (u64 i0 = b; i0 < e; i0 += kBlock) {
        const u64 i = i0 + threadIdx.x;
        const T v = i < e ? in[i] : T(0);
        T tot;
        const T ex = block_exclusive<T>(v, sw, &tot);
        if (i < e) out[i] = base + ex;
        base += tot;
    }
}

// out[i] = sum_{t<i} in[t] for i < *count; out[*count] = total. partial: kGrid scratch.
template <class T>
void exclusive(const T* in, const u32* count, T* out, T* partial, cudaStream_t st, u64* launches = nullptr) {
    reduce_chunks<T><<<kGrid, kBlock, 0, st>>>(in, count, partial);
    XYZB_LAUNCH_CHECK();
    scan_partials<T><<<1, kBlock, 0, st>>>(partial, kGrid, count, out);
    XYZB_LAUNCH_CHECK();
    scan_chunks<T><<<kGrid, kBlock, 0, st>>>(in, count, partial, out);
    XYZB_LAUNCH_CHECK();
    if (launches) *launches += 3;
}

} // namespace scan
} // namespace xyzb
