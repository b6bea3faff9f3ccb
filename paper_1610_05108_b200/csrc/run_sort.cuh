// Per-run LSD radix sort on thread-block clusters (sm_100a).
//
// One cluster of CL CTAs sorts one run's p keys (stable, 8-bit digits, all
// passes in one launch). Each CTA owns a contiguous segment of the run; per
// pass it histograms its segment into shared memory, the cluster exchanges
// the 256-bin histograms through distributed shared memory (DSMEM) to get
// every CTA's per-digit output base, and each CTA scatters its segment tile
// by tile with a stable in-tile ranking. Cluster barriers (release/acquire at
// cluster scope) order the global-memory ping-pong between passes. No global
// histogram/scan kernels and no host round trips: the whole sort is one
// launch, replacing upsweep/scan/downsweep per pass (radix_sort.cuh).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace xyzb {
namespace rsort {

constexpr int kRunThreads = 512;
constexpr int kRunWarps = kRunThreads / 32;
constexpr int kRunIpt = 8;                          // items per thread per tile
constexpr int kRunTile = kRunThreads * kRunIpt;     // 4096
constexpr int kRunPerWarp = kRunTile / kRunWarps;   // 256 = 8 chunks of 32

template <class K>
__global__ void __launch_bounds__(kRunThreads) sort_runs(K* __restrict__ ka, u32* __restrict__ va, K* __restrict__ kb,
                                                         u32* __restrict__ vb, u64 S, int passes) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const u32 CL = cl.num_blocks();
    const u32 cr = cl.block_rank();
    __shared__ u32 hist[256];
    __shared__ u32 base[256];
    __shared__ u32 wcount[kRunWarps][256];
    __shared__ u32 wsum[32];
    const u64 run = blockIdx.y;
    const u64 s0 = S * cr / CL, s1 = S * (cr + 1) / CL;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    K* kin = ka + run * S;
    u32* vin = va + run * S;
    K* kout = kb + run * S;
    u32* vout = vb + run * S;
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = pass * 8;
        // 1. histogram of this CTA's segment
        for (int i = threadIdx.x; i < 256; i += kRunThreads) hist[i] = 0;
        __syncthreads();
        for (u64 i0 = s0; i0 < s1; i0 += kRunThreads) {
            const u64 i = i0 + threadIdx.x;
            const bool valid = i < s1;
            const u32 active = __ballot_sync(0xffffffffu, valid);
            if (valid) {
                const u32 d = u32(kin[i] >> shift) & 255u;
                const u32 peers = __match_any_sync(active, d);
                if ((peers & lanemask_lt()) == 0) atomicAdd(&hist[d], __popc(peers));
            }
        }
        cl.sync();
        // 2. per-digit output base of this CTA from all histograms (DSMEM)
        u32 total = 0, below = 0;
        if (threadIdx.x < 256) {
            for (u32 c = 0; c < CL; ++c) {
                const u32 h = cl.map_shared_rank(hist, c)[threadIdx.x];
                total += h;
                if (c < cr) below += h;
            }
        }
        // exclusive scan of `total` over the 256 digits (threads 0..255 = warps 0..7)
        u32 incl = total;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31 && w < 8) wsum[w] = incl;
        cl.sync();  // every CTA has read all histograms; wsum visible
        if (threadIdx.x < 256) {
            u32 wb = 0;
            for (int q = 0; q < w; ++q) wb += wsum[q];
            base[threadIdx.x] = wb + incl - total + below;
        }
        __syncthreads();
        // 3. stable scatter, tile by tile
        for (u64 t0 = s0; t0 < s1; t0 += kRunTile) {
            for (int i = threadIdx.x; i < kRunWarps * 256; i += kRunThreads) (&wcount[0][0])[i] = 0;
            __syncthreads();
            K kk[kRunIpt];
            u32 vv[kRunIpt], rk[kRunIpt];
#pragma unroll
            for (int c = 0; c < kRunIpt; ++c) {
                const u64 i = t0 + u64(w) * kRunPerWarp + u64(c) * 32 + lane;
                const bool valid = i < s1;
                kk[c] = valid ? kin[i] : K(0);
                vv[c] = valid ? (pass == 0 ? u32(i) : vin[i]) : 0u;
            }
#pragma unroll
            for (int c = 0; c < kRunIpt; ++c) {
                const u64 i = t0 + u64(w) * kRunPerWarp + u64(c) * 32 + lane;
                const bool valid = i < s1;
                const u32 active = __ballot_sync(0xffffffffu, valid);
                u32 peers = 0, d = 0;
                if (valid) {
                    d = u32(kk[c] >> shift) & 255u;
                    peers = __match_any_sync(active, d);
                    rk[c] = wcount[w][d] + __popc(peers & lanemask_lt());
                }
                __syncwarp();
                if (valid && (peers & lanemask_lt()) == 0) wcount[w][d] += __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            // per digit: exclusive prefix over warps; tile total advances the base
            if (threadIdx.x < 256) {
                const int d = threadIdx.x;
                u32 run_sum = 0;
#pragma unroll
                for (int q = 0; q < kRunWarps; ++q) {
                    const u32 t = wcount[q][d];
                    wcount[q][d] = run_sum + base[d];
                    run_sum += t;
                }
                base[d] += run_sum;
            }
            __syncthreads();
#pragma unroll
            for (int c = 0; c < kRunIpt; ++c) {
                const u64 i = t0 + u64(w) * kRunPerWarp + u64(c) * 32 + lane;
                if (i < s1) {
                    const u32 d = u32(kk[c] >> shift) & 255u;
                    const u32 dst = wcount[w][d] + rk[c];
                    kout[dst] = kk[c];
                    vout[dst] = vv[c];
                }
            }
            __syncthreads();
        }
        // global writes of this pass visible to the whole cluster before the next
        __threadfence();
        cl.sync();
        K* tk = kin;
        kin = kout;
        kout = tk;
        u32* tv = vin;
        vin = vout;
        vout = tv;
    }
}

// Launch: sorts B runs of S keys in ka (values implicit = index) on key bits
// [0, bits); returns 0 if the result is in (ka, va), 1 if in (kb, vb).
template <class K>
int sort_runs_launch(K* ka, u32* va, K* kb, u32* vb, u64 B, u64 S, int bits, cudaStream_t st) {
    const int passes = (bits + 7) / 8;
    if (B == 0 || S == 0) return 0;
    // cluster size: enough CTAs to cover the SMs twice, segments >= one tile
    u64 cl = std::max<u64>(1, std::min<u64>(8, ceil_div(2 * kSMs, B)));
    while (cl > 1 && S / cl < u64(kRunTile)) --cl;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<u32>(cl), static_cast<u32>(B), 1);
    cfg.blockDim = dim3(kRunThreads, 1, 1);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<u32>(cl);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    XYZB_CUDA(cudaLaunchKernelEx(&cfg, sort_runs<K>, ka, va, kb, vb, S, passes));
    return passes & 1;
}

} // namespace rsort
} // namespace xyzb
