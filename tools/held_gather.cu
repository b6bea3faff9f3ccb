// Microbenchmark: column-pair XOR-popcount when a team keeps the held column
// in registers for R consecutive pairs (pairs sorted by held column) vs the
// fully random pair gather the verify does today. Rates in algorithmic GB/s
// (2 columns per pair, the verify roofline's count).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/held_gather tools/held_gather.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// team of G lanes, NIT 16-byte slices per lane and column (G*NIT >= w2)
template <int G, int NIT>
__global__ void __launch_bounds__(256) held(const ulonglong2* __restrict__ X, uint32_t ncols, uint32_t w2,
                                            uint32_t npairs, uint32_t R, uint32_t seed, unsigned long long* sink) {
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const uint32_t team = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t nteams = (gridDim.x * blockDim.x) / G;
    uint32_t acc = 0;
    const uint32_t ngroups = (npairs + R - 1) / R;
    for (uint32_t g = team; g < ngroups; g += nteams) {
        // held column: sorted order (group g -> column g * ncols / ngroups)
        const uint32_t j = uint32_t((uint64_t(g) * ncols) / ngroups);
        ulonglong2 a[NIT];
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const uint32_t wi = it * G + tl;
            a[it] = wi < w2 ? __ldg(X + size_t(j) * w2 + wi) : make_ulonglong2(0, 0);
        }
        for (uint32_t r = 0; r < R; ++r) {
            const uint32_t k = __umulhi(mix32(g * R + r + seed), ncols);
            ulonglong2 b[NIT];
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
                const uint32_t wi = it * G + tl;
                b[it] = wi < w2 ? __ldg(X + size_t(k) * w2 + wi) : make_ulonglong2(0, 0);
            }
            uint32_t s = 0;
#pragma unroll
            for (int it = 0; it < NIT; ++it) s += __popcll(a[it].x ^ b[it].x) + __popcll(a[it].y ^ b[it].y);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            acc += s;
        }
    }
    if (acc == 0xffffffffu) atomicAdd(sink, acc);
}

template <int G, int NIT>
float run(const ulonglong2* X, uint32_t ncols, uint32_t w2, uint32_t npairs, uint32_t R, int grid, unsigned long long* sink) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        held<G, NIT><<<grid, 256>>>(X, ncols, w2, npairs, R, rep, sink);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    return best;
}

int main() {
    struct Cfg { uint32_t ncols, words, npairs; const char* name; } cfgs[] = {
        {100000, 63, 15500000, "cfg2 p=1e5 W=63 (L2-resident)"},
        {1000000, 157, 31000000, "cfg4 p=1e6 W=157 (HBM)"}};
    unsigned long long* sink; cudaMalloc(&sink, 8);
    for (auto& c : cfgs) {
        const uint32_t wp = (c.words + 3) / 4 * 4, w2 = wp / 2;
        ulonglong2* X; cudaMalloc(&X, size_t(c.ncols) * wp * 8); cudaMemset(X, 0x5a, size_t(c.ncols) * wp * 8);
        for (uint32_t R : {1u, 2u, 4u, 8u, 16u, 32u}) {
            float best = 1e30f; int bg = 0; const char* bt = "";
            for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
                float t;
                if (w2 <= 32) {
                    t = run<8, 4>(X, c.ncols, w2, c.npairs, R, grid, sink); if (t < best) { best = t; bg = grid; bt = "8x4"; }
                    t = run<32, 1>(X, c.ncols, w2, c.npairs, R, grid, sink); if (t < best) { best = t; bg = grid; bt = "32x1"; }
                    t = run<16, 2>(X, c.ncols, w2, c.npairs, R, grid, sink); if (t < best) { best = t; bg = grid; bt = "16x2"; }
                } else {
                    t = run<32, 3>(X, c.ncols, w2, c.npairs, R, grid, sink); if (t < best) { best = t; bg = grid; bt = "32x3"; }
                    t = run<16, 5>(X, c.ncols, w2, c.npairs, R, grid, sink); if (t < best) { best = t; bg = grid; bt = "16x5"; }
                }
            }
            const double gbs = double(c.npairs) * 2.0 * 8.0 * c.words / (best * 1e-3) / 1e9;
            printf("%s R=%2u: %.3f ms  %.0f GB/s algorithmic (team %s grid %d)\n", c.name, R, best, gbs, bt, bg);
        }
        cudaFree(X);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
