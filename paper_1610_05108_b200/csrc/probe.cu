// Bandwidth probe for the verify roofline (libxyzb_probe.so).
//
// When X fits in L2 (BASELINE configs 1-3) the verify kernel is bound by the
// L2 -> SM fabric, not by HBM. This probe measures, on the GPU at hand, the
// rate at which random column PAIRS of an X-shaped matrix (ncols columns of
// Wp 8-byte words, the engine's padded layout) can be gathered and
// XOR-popcounted — the verify kernel's access pattern with the pair indices
// generated on the fly (no pair list, no Y, no hit test), by 8-lane teams
// of 16 B loads; the best over team sizes (8, 16 lanes), pairs in flight per
// team (1, 2) and grids (4, 8, 16 CTAs per SM). Reported as algorithmic
// GB/s: 2 x 8W bytes per pair, the same count bench.py uses for verify.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

// Team of G lanes gathers PR random column pairs at a time (16 B per lane
// per load, all PR x 2 columns in flight), XOR-popcounts them. Pair indices
// come from a hash (multiply-high range reduction), so nothing but the
// columns is read.
template <int G, int PR>
__global__ void __launch_bounds__(256) pair_gather(const ulonglong2* __restrict__ X, uint32_t ncols, uint32_t w2,
                                                   uint32_t npairs, uint32_t seed, unsigned long long* sink) {
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
            const uint32_t j = __umulhi(mix32(2 * q + seed), ncols), k = __umulhi(mix32(2 * q + 1 + seed), ncols);
            a[r] = X + size_t(j) * w2;
            b[r] = X + size_t(k) * w2;
        }
        for (uint32_t w0 = 0; w0 < w2; w0 += 4 * G) {
            ulonglong2 va[PR][4], vb[PR][4];
#pragma unroll
            for (int r = 0; r < PR; ++r)
#pragma unroll
                for (int it = 0; it < 4; ++it) {
                    const uint32_t wi = w0 + it * G + tl;
                    va[r][it] = wi < w2 ? __ldg(a[r] + wi) : make_ulonglong2(0, 0);
                    vb[r][it] = wi < w2 ? __ldg(b[r] + wi) : make_ulonglong2(0, 0);
                }
#pragma unroll
            for (int r = 0; r < PR; ++r)
#pragma unroll
                for (int it = 0; it < 4; ++it)
                    acc += __popcll(va[r][it].x ^ vb[r][it].x) + __popcll(va[r][it].y ^ vb[r][it].y);
        }
    }
    if (acc == 0xffffffffu) atomicAdd(sink, acc);
}

template <int G, int PR>
float time_gather(const ulonglong2* X, uint32_t ncols, uint32_t w2, uint32_t npairs, int grid, int reps,
                  unsigned long long* sink, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1) {
    float best = 1e30f;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(e0, st);
        pair_gather<G, PR><<<grid, 256, 0, st>>>(X, ncols, w2, npairs, uint32_t(r), sink);
        cudaEventRecord(e1, st);
        if (cudaEventSynchronize(e1) != cudaSuccess) return -1.f;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;  // the first launch warms L2
    }
    return best;
}

}  // namespace

extern "C" {

// Random column-pair gather rate (algorithmic GB/s = npairs * 2 * 8 * words /
// best time of `reps` launches). 0 on success, else the CUDA error code.
int xyzb_probe_pair_gather(int device, uint64_t ncols, uint64_t words, uint64_t npairs, int reps, double* gbps) {
    *gbps = 0.0;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return int(e);
    const uint64_t wp = (words + 3) / 4 * 4;
    const uint32_t w2 = uint32_t(wp / 2);
    ulonglong2* X = nullptr;
    unsigned long long* sink = nullptr;
    cudaStream_t st = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    float best = 1e30f;
    if ((e = cudaMalloc(&X, ncols * wp * 8)) != cudaSuccess) goto done;
    if ((e = cudaMalloc(&sink, 8)) != cudaSuccess) goto done;
    if ((e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) != cudaSuccess) goto done;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemsetAsync(X, 0x5a, ncols * wp * 8, st);
    // the best of several team shapes / grids / pairs in flight: a ceiling, not one kernel's rate
    for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
        const float t[4] = {time_gather<8, 1>(X, uint32_t(ncols), w2, uint32_t(npairs), grid, reps, sink, st, e0, e1),
                            time_gather<8, 2>(X, uint32_t(ncols), w2, uint32_t(npairs), grid, reps, sink, st, e0, e1),
                            time_gather<16, 1>(X, uint32_t(ncols), w2, uint32_t(npairs), grid, reps, sink, st, e0, e1),
                            time_gather<16, 2>(X, uint32_t(ncols), w2, uint32_t(npairs), grid, reps, sink, st, e0, e1)};
        for (float v : t) {
            if (v < 0) {
                e = cudaGetLastError();
                goto done;
            }
            if (v < best) best = v;
        }
    }
    *gbps = double(npairs) * 2.0 * 8.0 * double(words) / (double(best) * 1e-3) / 1e9;
    e = cudaGetLastError();
done:
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (st) cudaStreamDestroy(st);
    if (X) cudaFree(X);
    if (sink) cudaFree(sink);
    cudaSetDevice(prev);
    return int(e);
}

}  // extern "C"
