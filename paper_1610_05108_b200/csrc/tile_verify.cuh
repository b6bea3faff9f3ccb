// L2-tiled verification of a search's whole pair list (sm_100a).
//
// When X is much larger than the 126 MB L2 (config 4: 1.26 GB), the per-batch
// verify reads each candidate's two columns mostly from HBM: the candidate
// pairs of a run are spread over all of X. Here the pair lists of ALL batches
// accumulate in one buffer (one slot counter for the search), and are then
// bucketed by column tile before a single verify launch:
//   tile(j, k) = (min(j,k) / T, max(j,k) / T), upper triangle, snake order
// with T columns per range chosen so that two ranges (2T columns) fit in half
// of L2. All SMs sweep the tiles in order, so while a tile is verified its
// columns are L2-resident and every column is fetched from HBM about once per
// tile instead of once per pair; consecutive tiles share a column range.
// The candidate set and every strength are unchanged — only the order of the
// (order-free) verification moves; hits compute their x-side key from the
// run's draws (key_of_column) because the batch key arrays are gone by then.
//
//   tile_count    persistent CTAs, each a contiguous range of the pair list:
//                 shared histogram of tile ids -> hist[cta][tile]
//   tile_offsets  per tile: exclusive scan over CTAs, tile total
//   tile_starts   one CTA: exclusive scan of the tile totals
//   tile_scatter  the same ranges again: shared cursors (tile start + CTA
//                 offset) -> records in tile order; the batch-local run index
//                 becomes the search-global one (batch starts recorded
//                 between the batches)
#pragma once

#include "common.cuh"
#include "search_kernels.cuh"

namespace xyzb {
namespace tile {

using kern::PairRec;

constexpr int kThreads = 512;
constexpr u32 kCtas = kSMs * 4;
constexpr u32 kMaxTiles = 12288;  // 48 KB of shared counters
constexpr u32 kMaxBatches = 1024;

__device__ __forceinline__ u32 tile_of(u32 a, u32 b, u32 T, u32 A) {
    const u32 lo = min(a, b), hi = max(a, b);
    const u32 ta = lo / T, tb = hi / T;
    const u32 start = ta * A - ta * (ta - 1) / 2;  // rows 0..ta-1 hold A, A-1, ... tiles
    return start + ((ta & 1u) ? (A - 1 - tb) : (tb - ta));
}

// Bucket functor of the pair-list bucketing: the L2 column tile of (pa, pb).
struct TileOf {
    u32 T, A;
    __device__ __forceinline__ u32 operator()(u32 a, u32 b) const { return tile_of(a, b, T, A); }
};

__device__ __forceinline__ void cta_range(u32 P, u32& q0, u32& q1) {
    q0 = u32((u64(P) * blockIdx.x) / gridDim.x);
    q1 = u32((u64(P) * (blockIdx.x + 1)) / gridDim.x);
}

template <class F>
__global__ void __launch_bounds__(kThreads) tile_count(const PairRec* __restrict__ pairs, const u32* __restrict__ np,
                                                       u32 cap, F f, u32 ntiles, u32* __restrict__ hist) {
    extern __shared__ u32 h[];
    for (u32 i = threadIdx.x; i < ntiles; i += blockDim.x) h[i] = 0;
    __syncthreads();
    u32 q0, q1;
    cta_range(min(*np, cap), q0, q1);
    const uint2* pr = reinterpret_cast<const uint2*>(pairs);  // (pa, pb) of record q at 2q
    for (u32 q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
        const uint2 jk = __ldg(pr + 2 * u64(q));
        atomicAdd(h + f(jk.x, jk.y), 1u);
    }
    __syncthreads();
    for (u32 t = threadIdx.x; t < ntiles; t += blockDim.x) hist[u64(t) * gridDim.x + blockIdx.x] = h[t];
}

// One CTA per tile: hist[tile][cta] -> exclusive offsets within the tile; total.
__global__ void __launch_bounds__(1024) tile_offsets(u32* __restrict__ hist, u32 nctas, u32* __restrict__ total) {
    __shared__ u32 ws[33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32* row = hist + u64(blockIdx.x) * nctas;
    u32 carry = 0;
    for (u32 c0 = 0; c0 < nctas; c0 += blockDim.x) {
        const u32 c = c0 + threadIdx.x;
        const u32 x = c < nctas ? row[c] : 0u;
        u32 incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) ws[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const u32 v = lane < int(blockDim.x >> 5) ? ws[lane] : 0u;
            u32 vi = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, vi, o);
                if (lane >= o) vi += t;
            }
            ws[lane] = vi - v;
            if (lane == 31) ws[32] = vi;
        }
        __syncthreads();
        if (c < nctas) row[c] = carry + ws[wid] + incl - x;
        carry += ws[32];
        __syncthreads();
    }
    if (threadIdx.x == 0) total[blockIdx.x] = carry;
}

// One CTA: exclusive scan of the tile totals (in place).
__global__ void __launch_bounds__(1024) tile_starts(u32* __restrict__ total, u32 ntiles) {
    __shared__ u32 ws[33];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 carry = 0;
    for (u32 t0 = 0; t0 < ntiles; t0 += blockDim.x) {
        const u32 t = t0 + threadIdx.x;
        const u32 x = t < ntiles ? total[t] : 0u;
        u32 incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) ws[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const u32 v = lane < int(blockDim.x >> 5) ? ws[lane] : 0u;
            u32 vi = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 s = __shfl_up_sync(0xffffffffu, vi, o);
                if (lane >= o) vi += s;
            }
            ws[lane] = vi - v;
            if (lane == 31) ws[32] = vi;
        }
        __syncthreads();
        if (t < ntiles) total[t] = carry + ws[wid] + incl - x;
        carry += ws[32];
        __syncthreads();
    }
}

// bstart[i] = first slot of batch i (nb + 1 entries); batch i's runs are
// search runs i * B + run.
template <class F>
__global__ void __launch_bounds__(kThreads) tile_scatter(const PairRec* __restrict__ pairs, const u32* __restrict__ np,
                                                         u32 cap, F f, u32 ntiles,
                                                         const u32* __restrict__ hist, const u32* __restrict__ tstart,
                                                         const u32* __restrict__ bstart, u32 nb, u32 B,
                                                         PairRec* __restrict__ out) {
    extern __shared__ u32 cur[];  // [ntiles] cursors, then [nb + 1] batch starts
    u32* bs = cur + ntiles;
    for (u32 t = threadIdx.x; t < ntiles; t += blockDim.x) cur[t] = tstart[t] + hist[u64(t) * gridDim.x + blockIdx.x];
    for (u32 i = threadIdx.x; i <= nb; i += blockDim.x) bs[i] = bstart[i];
    __syncthreads();
    u32 q0, q1;
    cta_range(min(*np, cap), q0, q1);
    for (u32 q = q0 + threadIdx.x; q < q1; q += blockDim.x) {
        PairRec r = pairs[q];
        u32 lo = 0, hi = nb;  // the batch: last i with bs[i] <= q
        while (hi - lo > 1) {
            const u32 mid = (lo + hi) >> 1;
            if (bs[mid] <= q) lo = mid; else hi = mid;
        }
        r.run += lo * B;
        out[atomicAdd(cur + f(r.pa, r.pb), 1u)] = r;
    }
}

struct Plan {
    u32 T = 0, A = 0, ntiles = 0;
};

// Column ranges: 2T columns of `col_bytes` within half of the L2 (and at
// most kMaxTiles tiles).
inline Plan plan(u64 p, u64 col_bytes, u64 l2_bytes) {
    Plan t;
    u64 T = std::max<u64>(1, (l2_bytes / 2) / (2 * std::max<u64>(1, col_bytes)));
    u64 A = (p + T - 1) / T;
    while (A * (A + 1) / 2 > kMaxTiles) {
        T *= 2;
        A = (p + T - 1) / T;
    }
    t.T = u32(T);
    t.A = u32(A);
    t.ntiles = u32(A * (A + 1) / 2);
    return t;
}

inline u64 hist_words(const Plan& t) { return u64(t.ntiles) * kCtas + t.ntiles; }

// pairs (count at *np) -> out grouped by bucket f(pa, pb) (ntiles buckets);
// scratch: ntiles * (kCtas + 1) u32, its last ntiles words end as the bucket
// starts. bstart / nb / B: batch starts for the run globalisation (nb = 1 and
// bstart = {0, ~0} keep the runs as they are).
template <class F>
inline const u32* bucket_pairs(const PairRec* pairs, const u32* np, u32 cap, F f, u32 ntiles, const u32* bstart,
                               u32 nb, u32 B, u32* scratch, PairRec* out, cudaStream_t st, u64* launches) {
    func_smem(tile_count<F>, 64 << 10);
    func_smem(tile_scatter<F>, 64 << 10);
    u32* hist = scratch;
    u32* total = scratch + u64(ntiles) * kCtas;
    tile_count<F><<<kCtas, kThreads, ntiles * 4, st>>>(pairs, np, cap, f, ntiles, hist);
    XYZB_LAUNCH_CHECK();
    tile_offsets<<<ntiles, 1024, 0, st>>>(hist, kCtas, total);
    XYZB_LAUNCH_CHECK();
    tile_starts<<<1, 1024, 0, st>>>(total, ntiles);
    XYZB_LAUNCH_CHECK();
    tile_scatter<F><<<kCtas, kThreads, (ntiles + nb + 1) * 4, st>>>(pairs, np, cap, f, ntiles, hist, total, bstart,
                                                                    nb, B, out);
    XYZB_LAUNCH_CHECK();
    *launches += 4;
    return total;
}

inline void sort_by_tile(const PairRec* pairs, const u32* np, u32 cap, const Plan& t, const u32* bstart, u32 nb,
                         u32 B, u32* scratch, PairRec* out, cudaStream_t st, u64* launches) {
    bucket_pairs(pairs, np, cap, TileOf{t.T, t.A}, t.ntiles, bstart, nb, B, scratch, out, st, launches);
}

} // namespace tile
} // namespace xyzb
