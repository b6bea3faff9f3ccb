// Top-K over ALL verified candidates (BASELINE north_star "a top-K merge
// across runs"; the reference's A.8 hit list at any
// gamma low enough to hold K entries, ranked by the oracle.cpp:45-56
// comparator extended with the sign).
//
// The search keeps a running rank threshold `thr` (a lower bound of the
// strength of the K-th best DISTINCT candidate seen so far) and the hits of
// every occurrence at or above it. Per batch of runs:
//   pair-list path (binary):  the verify kernel writes each pair's integer
//     strength numerator to `sint` (no hit test); rank_hist bins those at or
//     above thr; emit_select picks the emission threshold E >= thr where the
//     batch holds >= `target` raw entries; emit_pairs appends the pairs at or
//     above E (warp-aggregated);
//   item path (continuous / long binary): the verify appends every pair whose
//     rank is at or above thr;
//   prune: dedup the buffer by (min(j,k), max(j,k), sign) in a hash table,
//     histogram the DISTINCT keys by rank, raise thr to the bin holding the
//     K-th distinct key, keep the occurrences at or above it.
// Pairs of a batch below E were never emitted; that is exact when the prune
// finds >= K distinct keys at or above E (then thr >= E). Otherwise the state
// records a failure and the host redoes the search with a larger target (the
// last attempt emits everything at or above thr, which cannot fail).
//
// Ranks: binary r = the strength numerator (exact, 0..n); continuous
// r = floor(s * 2^24) (s in [0, 1]). Bins are r >> shift (<= kBins bins), and
// every threshold is a bin's lower edge, so a threshold never exceeds the
// rank of the K-th distinct key. The final hits are those at or above the
// exact K-th strength (host, after the merge's A.10 ranking).
#pragma once

#include "common.cuh"
#include "merge_kernels.cuh"
#include "search_kernels.cuh"

namespace xyzb {
namespace topk {

using kern::DevHit;
using kern::PairRec;

constexpr int kBinsLog = 13;
constexpr u32 kBins = 1u << kBinsLog;

struct State {
    u32 thr;        // retained threshold (rank units, a bin edge)
    u32 emit;       // this batch's emission threshold
    u32 fail;       // bit 0: a dropped band may hold top-K keys; bit 1: hit buffer overflow; bit 2 (binned
                    // verify): a window without a phase of its own ran with thr still 0 (redo, phase per window)
    u32 max_hits;   // largest hit count seen (regrow)
    u32 distinct;   // distinct keys at or above thr after the last prune
    u32 pad[3];
};

inline int bin_shift(u64 max_rank) {
    int s = 0;
    while ((max_rank >> s) >= kBins) ++s;
    return s;
}

// rank of a hit record: binary = round(s n) (= the exact numerator), else floor(s 2^24)
__device__ __forceinline__ u32 rank_of(const DevHit& h, u32 n, int binary) {
    return kern::strength_rank(h.s, n, binary);
}

// Valid pair count of a batch, as the verify kernels compute it (an item
// overflow leaves unwritten slots; the host redoes the batch).
__device__ __forceinline__ u32 batch_pairs(const u32* npairs, u32 pair_cap, const u32* nitems, u32 item_cap) {
    return *nitems > item_cap ? 0u : min(*npairs, pair_cap);
}

// Histogram of the batch's pair ranks at or above thr (shared per CTA, then global).
__global__ void __launch_bounds__(512) rank_hist(const u32* __restrict__ sint, const u32* __restrict__ npairs,
                                                 u32 pair_cap, const u32* __restrict__ nitems, u32 item_cap,
                                                 const State* __restrict__ st, int shift, u32* __restrict__ hist) {
    __shared__ u32 h[kBins];
    for (u32 b = threadIdx.x; b < kBins; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const u32 thr = st->thr;
    if (thr > 0) return;  // the verify appended the pairs at or above thr itself (no ranks written)
    const u32 P = batch_pairs(npairs, pair_cap, nitems, item_cap);
    // four ranks per 16-byte load
    const u32 P4 = P / 4;
    const uint4* s4 = reinterpret_cast<const uint4*>(sint);
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < P4; i += u64(gridDim.x) * blockDim.x) {
        const uint4 r = s4[i];
        atomicAdd(&h[r.x >> shift], 1u);
        atomicAdd(&h[r.y >> shift], 1u);
        atomicAdd(&h[r.z >> shift], 1u);
        atomicAdd(&h[r.w >> shift], 1u);
    }
    for (u64 i = 4 * u64(P4) + u64(blockIdx.x) * blockDim.x + threadIdx.x; i < P; i += u64(gridDim.x) * blockDim.x)
        atomicAdd(&h[sint[i] >> shift], 1u);
    __syncthreads();
    for (u32 b = threadIdx.x; b < kBins; b += blockDim.x)
        if (h[b]) atomicAdd(&hist[b], h[b]);
}

// Largest bin b with sum_{b' >= b} hist[b'] >= target (0xffffffff if none),
// by one CTA of 1024 threads, 8 bins each.
__device__ __forceinline__ u32 suffix_bin(const u32* hist, u32 target, u32* total_out) {
    __shared__ u32 s_sum[1024];
    __shared__ u32 s_best;
    constexpr int kPer = kBins / 1024;
    const int t = threadIdx.x;
    u32 mine = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) mine += hist[t * kPer + q];
    s_sum[t] = mine;
    if (t == 0) s_best = 0;
    __syncthreads();
    // inclusive suffix sums over threads (Hillis-Steele, 10 steps)
    for (int o = 1; o < 1024; o <<= 1) {
        const u32 v = t + o < 1024 ? s_sum[t + o] : 0u;
        __syncthreads();
        s_sum[t] += v;
        __syncthreads();
    }
    // suffix at bin b = (suffix of threads after t) + bins of t from b upward
    u32 acc = t + 1 < 1024 ? s_sum[t + 1] : 0u;
    for (int q = kPer - 1; q >= 0; --q) {
        acc += hist[t * kPer + q];
        if (acc >= target) {
            atomicMax(&s_best, u32(t * kPer + q) + 1u);  // +1: 0 stays "none"
            break;
        }
    }
    __syncthreads();
    if (total_out) *total_out = s_sum[0];
    const u32 b = s_best;
    __syncthreads();
    return b == 0 ? 0xffffffffu : b - 1u;
}

// E = max(thr, lower edge of the bin where the batch's raw count from the top reaches target).
__global__ void __launch_bounds__(1024) emit_select(u32* __restrict__ hist, int shift, u32 target,
                                                    State* __restrict__ st, int conservative) {
    const u32 b = suffix_bin(hist, target, nullptr);
    if (threadIdx.x == 0) {
        const u32 thr = st->thr;
        u32 e = thr;  // thr > 0: the verify appended everything at or above thr
        if (thr == 0 && !conservative && b != 0xffffffffu) e = b << shift;
        st->emit = e;
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < kBins; i += blockDim.x) hist[i] = 0;  // next batch
}

// Append the batch's pairs with rank >= E (warp-aggregated slots).
__global__ void __launch_bounds__(256) emit_pairs(const PairRec* __restrict__ pairs, const u32* __restrict__ sint,
                                                  const u32* __restrict__ npairs, u32 pair_cap,
                                                  const u32* __restrict__ nitems, u32 item_cap,
                                                  const State* __restrict__ st, const void* __restrict__ xkeys,
                                                  int key64, u64 S, const u32* __restrict__ rid,
                                                  DevHit* __restrict__ hits, u32* __restrict__ hit_count, u32 hit_cap,
                                                  u32 n) {
    if (st->thr > 0) return;  // appended by the verify
    const u32 P = batch_pairs(npairs, pair_cap, nitems, item_cap);
    const u32 E = st->emit;
    const int lane = threadIdx.x & 31;
    for (u64 i0 = u64(blockIdx.x) * blockDim.x; i0 < P; i0 += u64(gridDim.x) * blockDim.x) {
        const u64 i = i0 + threadIdx.x;
        const u32 r = i < P ? sint[i] : 0u;
        const bool take = i < P && r >= E;
        const u32 bal = __ballot_sync(0xffffffffu, take);
        if (!bal) continue;
        u32 base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(hit_count, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
        if (take) {
            const u32 slot = base + __popc(bal & lanemask_lt());
            if (slot < hit_cap) {
                const PairRec pr = pairs[i];
                u32 j = pr.pa, k = pr.pb;
                if ((pr.pad & 2u) && j > k) {
                    const u32 t = j;
                    j = k;
                    k = t;
                }
                const u64 ki = u64(pr.run) * S + j;
                DevHit h;
                h.order = key64 ? static_cast<const u64*>(xkeys)[ki] : u64(static_cast<const u32*>(xkeys)[ki]);
                h.s = double(r) / double(n);
                h.j = j;
                h.k = k;
                h.rid = rid[pr.run];
                h.sint = int32_t(r);
                hits[slot] = h;
            }
        }
    }
}

// Quantised pair walks (sign transform, weighted): the pairs whose exact
// strength may reach E (rank lower bound at or above rank(E - 2 delta)) are
// re-verified exactly, one warp per pair, and appended at or above E.
template <class F>  // kern::SignStrength / kern::WeightedQ: delta + exact(j, k, pos_pass, lane, mask)
__global__ void __launch_bounds__(256) emit_pairs_requant(kern::VerifyArgs A, const PairRec* __restrict__ pairs,
                                                          const u32* __restrict__ npairs, u32 pair_cap, F f,
                                                          const State* __restrict__ st) {
    if (st->thr > 0) return;  // appended by the verify
    const u32 P = batch_pairs(npairs, pair_cap, A.nitems, A.item_cap);
    const u32 E = st->emit;
    const double lo_s = double(E) / double(1u << kern::kRealRankBits) - 2.0 * f.delta;
    const u32 lo = kern::strength_rank(lo_s > 0.0 ? lo_s : 0.0, 0u, 0);
    const int lane = threadIdx.x & 31;
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 c0 = warp * 32; c0 < P; c0 += nwarps * 32) {
        const u64 i = c0 + lane;
        u32 bal = __ballot_sync(0xffffffffu, i < P && A.sint_out[i] >= lo);
        while (bal) {
            const int t = __ffs(bal) - 1;
            bal &= bal - 1;
            const PairRec r = pairs[c0 + t];
            const bool pos_pass = A.run_sign[r.run] > 0;
            const double s = f.exact(r.pa, r.pb, pos_pass, lane, 0xffffffffu);
            if (lane == 0 && kern::strength_rank(s, 0u, 0) >= E) kern::append_pair_hit_real(A, r, s);
        }
    }
}

// ---- prune: distinct keys by rank, raise thr, keep occurrences >= thr ----

__global__ void prune_insert(const DevHit* __restrict__ hits, const u32* __restrict__ hit_count, u32 hit_cap,
                             const int8_t* __restrict__ sign_by_rid, u64* __restrict__ table, u64 mask, int shift,
                             u32 n, int binary, u32* __restrict__ dhist, State* __restrict__ st) {
    const u32 Hraw = *hit_count;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        atomicMax(&st->max_hits, Hraw);
        if (Hraw > hit_cap) st->fail |= 2u;
    }
    const u32 H = min(Hraw, hit_cap);
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += u64(gridDim.x) * blockDim.x) {
        const DevHit x = hits[i];
        const u64 t = merge::tag_of(x, sign_by_rid[x.rid]);
        u64 slot = merge::hash64(t) & mask;
        while (true) {
            const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(table + slot), merge::kEmpty, t);
            if (prev == merge::kEmpty) {
                atomicAdd(&dhist[rank_of(x, n, binary) >> shift], 1u);
                break;
            }
            if (prev == t) break;
            slot = (slot + 1) & mask;
        }
    }
}

__global__ void __launch_bounds__(1024) prune_select(u32* __restrict__ dhist, int shift, u32 K,
                                                     State* __restrict__ st) {
    u32 total = 0;
    const u32 b = suffix_bin(dhist, K, &total);
    // distinct keys at or above the emission threshold (a bin edge)
    __shared__ u32 s_above;
    if (threadIdx.x == 0) s_above = 0;
    __syncthreads();
    const u32 eb = st->emit >> shift;
    u32 mine = 0;
    for (u32 i = threadIdx.x; i < kBins; i += blockDim.x)
        if (i >= eb) mine += dhist[i];
    atomicAdd(&s_above, mine);
    __syncthreads();
    if (threadIdx.x == 0) {
        const u32 thr = st->thr;
        u32 nt = thr;
        if (b != 0xffffffffu) nt = max(thr, b << shift);
        if (st->emit > thr && s_above < K) st->fail |= 1u;  // pairs in [thr, emit) were dropped
        st->thr = nt;
        st->distinct = total;
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < kBins; i += blockDim.x) dhist[i] = 0;
}

__global__ void prune_compact(const DevHit* __restrict__ hits, const u32* __restrict__ hit_count, u32 hit_cap,
                              u32 n, int binary, const State* __restrict__ st, DevHit* __restrict__ out,
                              u32* __restrict__ out_count) {
    const u32 H = min(*hit_count, hit_cap);
    const u32 thr = st->thr;
    const int lane = threadIdx.x & 31;
    for (u64 i0 = u64(blockIdx.x) * blockDim.x; i0 < H; i0 += u64(gridDim.x) * blockDim.x) {
        const u64 i = i0 + threadIdx.x;
        DevHit x;
        bool keep = false;
        if (i < H) {
            x = hits[i];
            keep = rank_of(x, n, binary) >= thr;
        }
        const u32 bal = __ballot_sync(0xffffffffu, keep);
        if (!bal) continue;
        u32 base = 0;
        if (lane == __ffs(bal) - 1) base = atomicAdd(out_count, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
        if (keep) out[base + __popc(bal & lanemask_lt())] = x;
    }
}

// item path: the verify appended every pair at or above thr
__global__ void emit_all(State* st) { st->emit = st->thr; }

__global__ void copy_back(const DevHit* __restrict__ src, const u32* __restrict__ cnt, DevHit* __restrict__ dst,
                          u32* __restrict__ dst_count) {
    const u32 H = *cnt;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += u64(gridDim.x) * blockDim.x) dst[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) *dst_count = H;
}

} // namespace topk
} // namespace xyzb
