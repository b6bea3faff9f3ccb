// Microbenchmark (round 2): random column-pair XOR-popcount gathers confined
// to a window of `wc` columns over an X of 1e6 columns x 1280 B (config 4),
// for several team shapes (G lanes per pair, PR pairs in flight per team), to
// decide whether an L2-tiled pair order can beat the HBM-bound verify.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_window2 tools/l2_window2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// the window a pair falls in: consecutive blocks of per_win pairs share a window
template <int G, int PR, int U>
__global__ void __launch_bounds__(256) win(const ulonglong2* __restrict__ X, uint32_t ncols, uint32_t w2,
                                           uint32_t npairs, uint32_t wcols, uint32_t per_win, uint32_t seed,
                                           unsigned long long* sink) {
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t nteams = (gridDim.x * blockDim.x) / G;
    uint32_t acc = 0;
    for (uint32_t q0 = team * PR; q0 < npairs; q0 += nteams * PR) {
        const ulonglong2* a[PR];
        const ulonglong2* b[PR];
#pragma unroll
        for (int r = 0; r < PR; ++r) {
            const uint32_t q = q0 + r;
            const uint32_t wb = (q / per_win) * wcols % (ncols - wcols + 1);
            const uint32_t j = wb + __umulhi(mix32(2 * q + seed), wcols);
            const uint32_t k = wb + __umulhi(mix32(2 * q + 1 + seed), wcols);
            a[r] = X + size_t(j) * w2;
            b[r] = X + size_t(k) * w2;
        }
        for (uint32_t w0 = 0; w0 < w2; w0 += U * G) {
            ulonglong2 va[PR][U], vb[PR][U];
#pragma unroll
            for (int r = 0; r < PR; ++r)
#pragma unroll
                for (int it = 0; it < U; ++it) {
                    const uint32_t wi = w0 + it * G + tl;
                    va[r][it] = wi < w2 ? __ldg(a[r] + wi) : make_ulonglong2(0, 0);
                    vb[r][it] = wi < w2 ? __ldg(b[r] + wi) : make_ulonglong2(0, 0);
                }
#pragma unroll
            for (int r = 0; r < PR; ++r)
#pragma unroll
                for (int it = 0; it < U; ++it)
                    acc += __popcll(va[r][it].x ^ vb[r][it].x) + __popcll(va[r][it].y ^ vb[r][it].y);
        }
    }
    if (acc == 0xffffffffu) atomicAdd(sink, acc);
}

template <int G, int PR, int U>
float run(const ulonglong2* X, uint32_t ncols, uint32_t w2, uint32_t npairs, uint32_t wc, uint32_t per_win,
          unsigned long long* sink, int grid) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        win<G, PR, U><<<grid, 256>>>(X, ncols, w2, npairs, wc, per_win, rep, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return best;
}

int main() {
    const uint32_t ncols = 1000000, words = 160, w2 = words / 2, npairs = 16000000;
    ulonglong2* X;
    cudaMalloc(&X, size_t(ncols) * words * 8);
    cudaMemset(X, 0x5a, size_t(ncols) * words * 8);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const double alg = double(npairs) * 2 * 1256;
    for (uint32_t wc : {4000u, 8000u, 16000u, 24000u, 32000u, 48000u, 64000u, 1000000u}) {
        const uint32_t per_win = 2000000;
        float t[8];
        t[0] = run<8, 1, 4>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 8);
        t[1] = run<8, 2, 4>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 8);
        t[2] = run<16, 1, 4>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 8);
        t[3] = run<16, 2, 2>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 8);
        t[4] = run<32, 1, 3>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 8);
        t[5] = run<8, 1, 4>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 16);
        t[6] = run<16, 1, 4>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 4);
        t[7] = run<32, 2, 3>(X, ncols, w2, npairs, wc, per_win, sink, 148 * 4);
        printf("window %7u cols (%7.1f MB):", wc, wc * 1280.0 / 1e6);
        for (float v : t) printf(" %6.0f", alg / (v * 1e-3) / 1e9);
        printf("  GB/s [8x1x4 8x2x4 16x1x4 16x2x2 32x1x3 | 8x1x4@16 16x1x4@4 32x2x3@4]\n");
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
