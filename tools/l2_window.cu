// Microbenchmark: random column-pair XOR-popcount gathers confined to a
// window of `win` columns (the L2-tiled verify's working set) over an X of
// 1e6 columns x 1280 B (config 4): rate vs window size.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_window tools/l2_window.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int G, int NIT>
__global__ void __launch_bounds__(256) win(const ulonglong2* __restrict__ X, uint32_t ncols, uint32_t w2,
                                           uint32_t npairs, uint32_t wcols, uint32_t per_win, uint32_t seed,
                                           unsigned long long* sink) {
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t nteams = (gridDim.x * blockDim.x) / G;
    uint32_t acc = 0;
    for (uint32_t q = team; q < npairs; q += nteams) {
        const uint32_t wb = (q / per_win) * wcols % (ncols - wcols + 1);
        const uint32_t j = wb + __umulhi(mix32(2 * q + seed), wcols), k = wb + __umulhi(mix32(2 * q + 1 + seed), wcols);
        ulonglong2 a[NIT], b[NIT];
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const uint32_t wi = it * G + tl;
            a[it] = wi < w2 ? __ldg(X + size_t(j) * w2 + wi) : make_ulonglong2(0, 0);
            b[it] = wi < w2 ? __ldg(X + size_t(k) * w2 + wi) : make_ulonglong2(0, 0);
        }
        uint32_t s = 0;
#pragma unroll
        for (int it = 0; it < NIT; ++it) s += __popcll(a[it].x ^ b[it].x) + __popcll(a[it].y ^ b[it].y);
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        acc += s;
    }
    if (acc == 0xffffffffu) atomicAdd(sink, acc);
}

int main() {
    const uint32_t ncols = 1000000, words = 160, w2 = words / 2, npairs = 31000000;
    ulonglong2* X; cudaMalloc(&X, size_t(ncols) * words * 8); cudaMemset(X, 0x5a, size_t(ncols) * words * 8);
    unsigned long long* sink; cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (uint32_t wc : {6000u, 12000u, 24000u, 36000u, 49000u, 70000u, 98000u, 200000u, 1000000u}) {
        const uint32_t per_win = 400000;  // pairs per window (a tile)
        float best = 1e30f;
        for (int grid : {148 * 4, 148 * 8}) {
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(e0);
                win<32, 3><<<grid, 256>>>(X, ncols, w2, npairs, wc, per_win, rep, sink);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (rep && ms < best) best = ms;
            }
        }
        printf("window %7u cols (%6.1f MB): %.3f ms  %.0f GB/s algorithmic\n", wc, wc * 1280.0 / 1e6, best,
               double(npairs) * 2 * 1256 / (best * 1e-3) / 1e9);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
