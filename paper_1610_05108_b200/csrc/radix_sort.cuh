// Segmented stable LSD radix sort (hand-written, no CUB): R segments of S
// (key, uint32 value) entries each, sorted independently on key bits
// [0, bits) in 8-bit digit passes. Used for the per-run key sort of the
// bucket join (replaces std::sort of KeyEntry, pair_search.cpp:26-32) and for
// the hit-list orderings of the merge (search.cpp:96-108).
//
// Per pass: upsweep (per-tile digit histograms in shared memory,
// warp-aggregated with match.any so skewed digits do not serialise on one
// bank), per-segment scan of the (digit, tile) table, downsweep (stable
// in-tile ranking with per-warp digit counters, then scatter). Stability
// comes from tile order, warp order inside a tile, and lane order inside a
// warp chunk, so equal keys keep their input (column-index) order — which is
// what reproduces the reference's (key, side, index) order without a side
// bit in the key.
#pragma once

#include "common.cuh"

namespace xyzb {
namespace rsort {

constexpr int kBlock = 256;
constexpr int kIpt = 16;
constexpr int kTile = kBlock * kIpt;  // 4096 entries per CTA
constexpr int kWarps = kBlock / 32;
constexpr int kPerWarp = kTile / kWarps;  // 512 = 16 chunks of 32
constexpr int kChunks = kPerWarp / 32;
constexpr int kRadix = 256;

template <class K>
__device__ __forceinline__ u32 digit_of(K k, int shift) {
    return static_cast<u32>(k >> shift) & (kRadix - 1);
}

template <class K>
__global__ void __launch_bounds__(kBlock) upsweep(const K* __restrict__ keys, u64 S, u32 tiles,
                                                  int shift, u32* __restrict__ hist) {
    __shared__ u32 h[kRadix];
    const u64 seg = blockIdx.y;
    const u32 tile = blockIdx.x;
    for (int i = threadIdx.x; i < kRadix; i += kBlock) h[i] = 0;
    __syncthreads();
    const u64 t0 = u64(tile) * kTile;
    const u32 cnt = static_cast<u32>(minu(kTile, S - t0));
    const K* base = keys + seg * S + t0;
    for (u32 r0 = 0; r0 < cnt; r0 += kBlock) {
        const u32 i = r0 + threadIdx.x;
        const bool valid = i < cnt;
        const u32 active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const u32 d = digit_of(base[i], shift);
            const u32 peers = __match_any_sync(active, d);
            if ((peers & lanemask_lt()) == 0) atomicAdd(&h[d], __popc(peers));
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kBlock) hist[(seg * kRadix + d) * tiles + tile] = h[d];
}

// In-place exclusive scan of each segment's (digit-major, tile-minor) table.
__global__ void __launch_bounds__(1024) scan_hist(u32* __restrict__ hist, u32 tiles) {
    __shared__ u32 warp_tot[32];
    const u64 seg = blockIdx.x;
    u32* h = hist + seg * kRadix * tiles;
    const u32 N = kRadix * tiles;
    const u32 per = (N + blockDim.x - 1) / blockDim.x;
    const u32 b = threadIdx.x * per;
    const u32 e = min(N, b + per);
    u32 local = 0;
    for (u32 i = b; i < e; ++i) local += h[i];
    // block exclusive scan of `local`
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        u32 v = lane < nw ? warp_tot[lane] : 0;
        u32 vi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, vi, o);
            if (lane >= o) vi += t;
        }
        if (lane < nw) warp_tot[lane] = vi - v;
    }
    __syncthreads();
    u32 run = warp_tot[wid] + incl - local;
    for (u32 i = b; i < e; ++i) {
        const u32 t = h[i];
        h[i] = run;
        run += t;
    }
}

template <class K>
__global__ void __launch_bounds__(kBlock) downsweep(const K* __restrict__ keys_in,
                                                    const u32* __restrict__ vals_in, K* __restrict__ keys_out,
                                                    u32* __restrict__ vals_out, u64 S, u32 tiles, int shift,
                                                    const u32* __restrict__ hist) {
    __shared__ u32 wcount[kWarps][kRadix];
    __shared__ u32 goff[kRadix];
    const u64 seg = blockIdx.y;
    const u32 tile = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kBlock) (&wcount[0][0])[i] = 0;
    for (int d = threadIdx.x; d < kRadix; d += kBlock) goff[d] = hist[(seg * kRadix + d) * tiles + tile];
    __syncthreads();
    const u64 t0 = u64(tile) * kTile;
    const u32 cnt = static_cast<u32>(minu(kTile, S - t0));
    const K* kb = keys_in + seg * S + t0;
    const u32* vb = vals_in ? vals_in + seg * S + t0 : nullptr;
    K kk[kChunks];
    u32 vv[kChunks];
    u32 rk[kChunks];
#pragma unroll
    for (int c = 0; c < kChunks; ++c) {
        const u32 i = w * kPerWarp + c * 32 + lane;
        const bool valid = i < cnt;
        kk[c] = valid ? kb[i] : K(0);
        vv[c] = valid ? (vb ? vb[i] : static_cast<u32>(t0 + i)) : 0u;
    }
#pragma unroll
    for (int c = 0; c < kChunks; ++c) {
        const u32 i = w * kPerWarp + c * 32 + lane;
        const bool valid = i < cnt;
        const u32 active = __ballot_sync(0xffffffffu, valid);
        u32 peers = 0, d = 0;
        if (valid) {
            d = digit_of(kk[c], shift);
            peers = __match_any_sync(active, d);
            rk[c] = wcount[w][d] + __popc(peers & lanemask_lt());
        }
        __syncwarp();
        if (valid && (peers & lanemask_lt()) == 0) wcount[w][d] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kBlock) {
        u32 run = 0;
#pragma unroll
        for (int w2 = 0; w2 < kWarps; ++w2) {
            const u32 t = wcount[w2][d];
            wcount[w2][d] = run;
            run += t;
        }
    }
    __syncthreads();
    K* ko = keys_out + seg * S;
    u32* vo = vals_out + seg * S;
#pragma unroll
    for (int c = 0; c < kChunks; ++c) {
        const u32 i = w * kPerWarp + c * 32 + lane;
        if (i < cnt) {
            const u32 d = digit_of(kk[c], shift);
            const u32 dst = goff[d] + wcount[w][d] + rk[c];
            ko[dst] = kk[c];
            vo[dst] = vv[c];
        }
    }
}

inline u32 tiles_for(u64 S) { return static_cast<u32>(ceil_div(S, kTile)); }
inline size_t hist_words(u64 R, u64 S) { return size_t(R) * kRadix * tiles_for(S); }

// Sort R segments of S entries on key bits [0, bits). Input keys in kbuf[0]
// (values implicit = index within segment when vals_in_implicit). Returns the
// index (0/1) of the ping-pong buffer pair holding the sorted result.
template <class K>
int sort_segments(K* kbuf[2], u32* vbuf[2], u64 R, u64 S, int bits, u32* hist, cudaStream_t st,
                  u64* launches = nullptr) {
    if (R == 0 || S == 0) return 0;
    const u32 tiles = tiles_for(S);
    const int passes = (bits + 7) / 8;
    int cur = 0;
    for (int pss = 0; pss < passes; ++pss) {
        const int shift = pss * 8;
        dim3 grid(tiles, static_cast<u32>(R));
        upsweep<K><<<grid, kBlock, 0, st>>>(kbuf[cur], S, tiles, shift, hist);
        XYZB_LAUNCH_CHECK();
        scan_hist<<<static_cast<u32>(R), 1024, 0, st>>>(hist, tiles);
        XYZB_LAUNCH_CHECK();
        downsweep<K><<<grid, kBlock, 0, st>>>(kbuf[cur], pss == 0 ? nullptr : vbuf[cur], kbuf[cur ^ 1],
                                              vbuf[cur ^ 1], S, tiles, shift, hist);
        XYZB_LAUNCH_CHECK();
        if (launches) *launches += 3;
        cur ^= 1;
    }
    return cur;
}

} // namespace rsort
} // namespace xyzb
