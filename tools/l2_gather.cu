// Microbenchmark: the L2 -> SM bandwidth a verify-shaped access pattern can
// reach on this GPU. A 51.2 MB column matrix (1e5 columns x 512 B, L2
// resident) is read as random column pairs by 8-lane teams (4 x 16 B per lane
// per column), XOR-popcounted like verify_pairs_*; plus a sequential sweep.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_gather l2_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int G>
__global__ void __launch_bounds__(256) gather(const ulonglong2* __restrict__ X, uint32_t ncols, uint32_t npairs,
                                              uint32_t seed, unsigned long long* sink) {
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t nteams = (gridDim.x * blockDim.x) / G;
    uint32_t acc = 0;
    for (uint32_t q = team; q < npairs; q += nteams) {
        const uint32_t j = hash32(q * 2 + seed) % ncols, k = hash32(q * 2 + 1 + seed) % ncols;
        const ulonglong2* a = X + size_t(j) * 32;
        const ulonglong2* b = X + size_t(k) * 32;
        ulonglong2 va[32 / G], vb[32 / G];
#pragma unroll
        for (int it = 0; it < 32 / G; ++it) {
            va[it] = __ldg(a + it * G + tl);
            vb[it] = __ldg(b + it * G + tl);
        }
#pragma unroll
        for (int it = 0; it < 32 / G; ++it) acc += __popcll(va[it].x ^ vb[it].x) + __popcll(va[it].y ^ vb[it].y);
    }
    if (acc == 0xffffffffu) atomicAdd(sink, acc);
}

// The verify shape: pair record (16 B) -> column ids through the grouped
// positions (sv) -> the two columns.
template <int G>
__global__ void __launch_bounds__(256) gather_indirect(const ulonglong2* __restrict__ X, const uint4* __restrict__ pr,
                                                       const uint32_t* __restrict__ sv, uint32_t npairs,
                                                       unsigned long long* sink) {
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t nteams = (gridDim.x * blockDim.x) / G;
    uint32_t acc = 0;
    for (uint32_t c0 = team * 32; c0 < npairs; c0 += nteams * 32) {
        const uint32_t c1 = min(npairs, c0 + 32);
        for (uint32_t q = c0; q < c1; ++q) {
            const uint4 r = pr[q];
            const uint32_t j = sv[r.x], k = sv[r.y];
            const ulonglong2* a = X + size_t(j) * 32;
            const ulonglong2* b = X + size_t(k) * 32;
            ulonglong2 va[32 / G], vb[32 / G];
#pragma unroll
            for (int it = 0; it < 32 / G; ++it) {
                va[it] = __ldg(a + it * G + tl);
                vb[it] = __ldg(b + it * G + tl);
            }
#pragma unroll
            for (int it = 0; it < 32 / G; ++it) acc += __popcll(va[it].x ^ vb[it].x) + __popcll(va[it].y ^ vb[it].y);
        }
    }
    if (acc == 0xffffffffu) atomicAdd(sink, acc);
}

__global__ void fill_pairs(uint4* pr, uint32_t* sv, uint32_t npairs, uint32_t nsv, uint32_t ncols) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < npairs; i += gridDim.x * blockDim.x)
        pr[i] = make_uint4(hash32(2 * i) % nsv, hash32(2 * i + 1) % nsv, 0, 0);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nsv; i += gridDim.x * blockDim.x)
        sv[i] = hash32(i ^ 0x9e3779b9u) % ncols;
}

// 256-bit loads (LDG.E.ENL2.256): G lanes x (512 / (32 G)) loads of 32 B per column.
__device__ __forceinline__ void ld256(const void* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
template <int G>
__global__ void __launch_bounds__(256) gather256(const ulonglong2* __restrict__ X, uint32_t ncols, uint32_t npairs,
                                                 uint32_t seed, unsigned long long* sink) {
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t nteams = (gridDim.x * blockDim.x) / G;
    constexpr int NL = 16 / G;  // 32-byte loads per lane per column
    uint32_t acc = 0;
    for (uint32_t q = team; q < npairs; q += nteams) {
        const uint32_t j = hash32(q * 2 + seed) % ncols, k = hash32(q * 2 + 1 + seed) % ncols;
        const char* a = reinterpret_cast<const char*>(X + size_t(j) * 32);
        const char* b = reinterpret_cast<const char*>(X + size_t(k) * 32);
        uint64_t va[NL][4], vb[NL][4];
#pragma unroll
        for (int it = 0; it < NL; ++it) {
            ld256(a + (it * G + tl) * 32, va[it][0], va[it][1], va[it][2], va[it][3]);
            ld256(b + (it * G + tl) * 32, vb[it][0], vb[it][1], vb[it][2], vb[it][3]);
        }
#pragma unroll
        for (int it = 0; it < NL; ++it)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc += __popcll(va[it][e] ^ vb[it][e]);
    }
    if (acc == 0xffffffffu) atomicAdd(sink, acc);
}

__global__ void sweep(const ulonglong2* __restrict__ X, size_t n, unsigned long long* sink) {
    uint64_t acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const ulonglong2 v = __ldg(X + i);
        acc ^= v.x + v.y;
    }
    if (acc == 0x12345) atomicAdd(sink, acc);
}

int main() {
    const uint32_t ncols = 100000, npairs = 16000000;
    const size_t words2 = size_t(ncols) * 32;
    ulonglong2* X;
    unsigned long long* sink;
    cudaMalloc(&X, words2 * 16);
    cudaMalloc(&sink, 8);
    cudaMemset(X, 0x5a, words2 * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        sweep<<<148 * 8, 256>>>(X, words2, sink);
        for (int r = 0; r < 9; ++r) sweep<<<148 * 8, 256>>>(X, words2, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("sequential sweep of L2-resident 51.2 MB: %.1f GB/s\n", 10 * words2 * 16 / (ms * 1e-3) / 1e9);
    }
    for (int g : {4, 8, 16, 32}) {
        for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
          for (int w = 0; w < 2; ++w) {
            cudaEventRecord(e0);
            for (int r = 0; r < 5; ++r) {
                if (g == 4) gather<4><<<grid, 256>>>(X, ncols, npairs, r, sink);
                if (g == 8) gather<8><<<grid, 256>>>(X, ncols, npairs, r, sink);
                if (g == 16) gather<16><<<grid, 256>>>(X, ncols, npairs, r, sink);
                if (g == 32) gather<32><<<grid, 256>>>(X, ncols, npairs, r, sink);
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
          }
            printf("random 512 B column pairs, team %2d lanes, grid %5d: %.1f GB/s (%.3f ms per 16M pairs)\n", g,
                   grid, 5.0 * npairs * 1024 / (ms * 1e-3) / 1e9, ms / 5);
        }
    }
    for (int g : {4, 8, 16}) {
        for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
            for (int w = 0; w < 2; ++w) {
                cudaEventRecord(e0);
                for (int r = 0; r < 5; ++r) {
                    if (g == 4) gather256<4><<<grid, 256>>>(X, ncols, npairs, r, sink);
                    if (g == 8) gather256<8><<<grid, 256>>>(X, ncols, npairs, r, sink);
                    if (g == 16) gather256<16><<<grid, 256>>>(X, ncols, npairs, r, sink);
                }
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            printf("random 512 B column pairs, 256-bit loads, team %2d lanes, grid %5d: %.1f GB/s (%.3f ms per 16M pairs)\n",
                   g, grid, 5.0 * npairs * 1024 / (ms * 1e-3) / 1e9, ms / 5);
        }
    }
    {
        const uint32_t nsv = 20000000;
        uint4* pr;
        uint32_t* sv;
        cudaMalloc(&pr, size_t(npairs) * 16);
        cudaMalloc(&sv, size_t(nsv) * 4);
        fill_pairs<<<148 * 8, 256>>>(pr, sv, npairs, nsv, ncols);
        for (int g : {8, 16}) {
            for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
                for (int w = 0; w < 2; ++w) {
                    cudaEventRecord(e0);
                    for (int r = 0; r < 5; ++r) {
                        if (g == 8) gather_indirect<8><<<grid, 256>>>(X, pr, sv, npairs, sink);
                        if (g == 16) gather_indirect<16><<<grid, 256>>>(X, pr, sv, npairs, sink);
                    }
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    cudaEventElapsedTime(&ms, e0, e1);
                }
                printf("pair list + sv indirection, team %2d lanes, grid %5d: %.1f GB/s of columns (%.3f ms per 16M pairs)\n",
                       g, grid, 5.0 * npairs * 1024 / (ms * 1e-3) / 1e9, ms / 5);
            }
        }
    }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
