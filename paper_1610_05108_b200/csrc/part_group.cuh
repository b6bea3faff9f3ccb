// Partitioned grouping + join (sm_100a): one partition pass over the keys,
// then one small CTA per (run, partition) with its bucket table in shared
// memory.
//
// equal_pairs (pair_search.cpp:12-55) groups the x-keys v of a run and pairs
// group v with group v ^ c (c = x-key ^ z-key of every column, A.3). An
// invertible GF(2)-linear map w = T(v) with T(c) = e_0 makes the partner of
// w simply w ^ 1, so the top k bits of w name a partition that holds both
// sides of every block, and within it the partner bucket is the neighbour:
//   T(v) = swap_{0,t}(v ^ (v_t ? c ^ e_t : 0)),  t = lowest set bit of c
// (c ^ e_t has bit t clear, so v -> v ^ (v_t ? c ^ e_t : 0) is an involution
// mapping c to e_t; the bit swap moves e_t to e_0). c == 0 (diagonal blocks,
// every group paired with itself) keeps T = identity.
//
//   part_count    per tile of keys: per-warp shared histograms of the k-bit
//                 partition digit -> per-run partition sizes (global atomics)
//   part_scan     per run: exclusive scan of the 2^k sizes -> partition
//                 starts and cursors
//   part_scatter  per tile: one shared atomic per key (rank in its warp's
//                 digit counter), one global atomic per (tile, digit) ->
//                 (w, column) entries in partition order
//   part_join<0>  per (run, partition): bucket counts of the 2^lb local
//                 buckets in shared memory -> |E_r| incl. the diagonal and
//                 the canonical work (guard, pair_search.hpp:91-94)
//   part_join<2>  both in one pass (the binned verify, when the expected |E_r|
//                 is far below the guard): the pairs of a run that turns out
//                 aborted are dropped when they are binned (bin_window)
//   part_join<1>  per (run, partition) of a kept run: counts, scan, scatter of
//                 the columns into the run's grouped array, then the blocks
//                 (pairs of small blocks written warp-cooperatively, items for
//                 large ones) exactly as the fused kernels emit them.
// Under the binned verify nothing reads the keys afterwards, so the records
// come straight from the row planes (project_scatter: no key array), as 4
// bytes each — (local bucket << (32 - lb)) | column, the partition being the
// record's place — where both fit (part_packed_ok), and then without a count
// pass: every (run, partition) owns a fixed region of 2.5x the mean partition
// size, the scatter's cursors end as the partition sizes and part_scan runs
// after it. An overflowing region is flagged on the device and the host
// redoes the search with counted partitions (engine.cu).
// The order inside a bucket is not deterministic (atomics); nothing depends on
// it: pair-list hits carry columns and the merge orders hits by (rid, v, j, k).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "cta_group.cuh"
#include "search_kernels.cuh"

namespace xyzb {
namespace kern {

constexpr int kPgThreads = 512;
constexpr int kPgPerThread = 8;
constexpr int kPjThreads = 512;   // partition join CTA
constexpr int kPjPerThread = 8;   // entries per thread kept in registers
constexpr u32 kPgTile = kPgThreads * kPgPerThread;  // keys per tile of the partition passes
constexpr int kPgMaxK = 10;                          // partition digits: at most 1024 partitions per run

// Local bucket bits: 2^lb u32 counters per partition CTA (16 KB at lb = 12).
// Partition digits k: the fewest that bring the mean partition (p / 2^k
// entries) to kPjTarget, at least M - 14 (a 2^14-bucket table is 64 KB), at
// most kPgMaxK and M - 1 (a key and its partner share a partition).
constexpr u64 kPjTarget = 4096;
inline int part_digits(int M, u64 p) {
    int k = 1;
    while (k < kPgMaxK && k < M - 1 && (p >> k) > kPjTarget) ++k;
    return std::min(std::max(k, M - 14), M - 1);
}
inline int part_local_bits(int M, u64 p) { return M - part_digits(M, p); }

struct PartMap {
    u32 c, cm, t;
    __device__ __forceinline__ PartMap(u32 c_) : c(c_), cm(0), t(0) {
        if (c) {
            t = u32(__ffs(int(c)) - 1);
            cm = c ^ (1u << t);
        }
    }
    __device__ __forceinline__ u32 fwd(u32 v) const {
        if (!c) return v;
        u32 x = v ^ (((v >> t) & 1u) ? cm : 0u);
        const u32 d = (x ^ (x >> t)) & 1u;
        return x ^ (d | (d << t));
    }
    __device__ __forceinline__ u32 inv(u32 w) const {
        if (!c) return w;
        const u32 d = (w ^ (w >> t)) & 1u;
        const u32 x = w ^ (d | (d << t));
        return x ^ (((x >> t) & 1u) ? cm : 0u);
    }
};

// ---------------------------------------------------------- partition pass --

// Partition digit of w: its top k bits (dense path: the local bucket is the
// low lb bits), or, for the hashed path, the top k bits of a multiplicative
// hash of w >> 1 — w and its partner w ^ 1 still share it, and the partitions
// stay balanced when key bits are correlated (a row drawn twice makes two key
// bits equal for every column).
__device__ __forceinline__ u32 part_digit(u32 w, int lb, int k, bool hashed) {
    return hashed ? (k ? ((w >> 1) * 0x9E3779B1u) >> (32 - k) : 0u) : (w >> lb);
}

// Entries of the partitioned keys: (w, column) as one 8-byte record.
template <bool SCATTER>
__device__ __forceinline__ void part_tile(const u32* __restrict__ keys, u64 p, int M, int lb, bool hashed,
                                          const u32* __restrict__ xorc, u32* __restrict__ pcnt,
                                          u32* __restrict__ cursor, uint2* __restrict__ pe) {
    extern __shared__ u32 hist[];  // [nwarps][2^k]
    const int k = M - lb;
    const u32 D = 1u << k;
    const u32 b = blockIdx.y;
    const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const u32 mask = M >= 32 ? 0xffffffffu : (1u << M) - 1u;
    const PartMap pm(xorc[b] & mask);
    for (u32 i = threadIdx.x; i < D * nw; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const u64 t0 = u64(blockIdx.x) * kPgTile;
    const u32* kb = keys + u64(b) * p;
    u32 w[kPgPerThread], rk[kPgPerThread];
    u32* hw = hist + wid * D;
#pragma unroll
    for (int q = 0; q < kPgPerThread; ++q) {
        const u64 i = t0 + u64(q) * blockDim.x + threadIdx.x;
        w[q] = i < p ? pm.fwd(__ldg(kb + i) & mask) : 0u;
    }
#pragma unroll
    for (int q = 0; q < kPgPerThread; ++q) {
        const u64 i = t0 + u64(q) * blockDim.x + threadIdx.x;
        if (i < p) rk[q] = atomicAdd(hw + part_digit(w[q], lb, k, hashed), 1u);
    }
    __syncthreads();
    if constexpr (!SCATTER) {
        for (u32 d = threadIdx.x; d < D; d += blockDim.x) {
            u32 s = 0;
            for (int v = 0; v < nw; ++v) s += hist[v * D + d];
            if (s) atomicAdd(pcnt + u64(b) * D + d, s);
        }
    } else {
        // per digit: reserve the tile's range, then per-warp exclusive offsets
        for (u32 d = threadIdx.x; d < D; d += blockDim.x) {
            u32 s = 0;
            for (int v = 0; v < nw; ++v) s += hist[v * D + d];
            u32 base = s ? atomicAdd(cursor + u64(b) * D + d, s) : 0u;
            for (int v = 0; v < nw; ++v) {
                const u32 x = hist[v * D + d];
                hist[v * D + d] = base;
                base += x;
            }
        }
        __syncthreads();
        uint2* out = pe + u64(b) * p;
#pragma unroll
        for (int q = 0; q < kPgPerThread; ++q) {
            const u64 i = t0 + u64(q) * blockDim.x + threadIdx.x;
            if (i < p) out[hw[part_digit(w[q], lb, k, hashed)] + rk[q]] = make_uint2(w[q], u32(i));
        }
    }
}

// The projection (project_bits_t's u32 form) with the partition count fused:
// each thread's 32 keys are counted into a shared histogram of partition
// digits right after the transpose, so part_count's re-read of the keys is
// not needed (xorc must be computed before: ykey_xorc runs first).
template <bool STORE_KEYS>
__global__ void __launch_bounds__(128) project_count(const u32* __restrict__ Xr, u64 P32, u64 p,
                                                     const u32* __restrict__ rows, int M, u32* __restrict__ keys,
                                                     const u32* __restrict__ xorc, int lb, int hashed,
                                                     u32* __restrict__ pcnt) {
    __shared__ u32 srow[64];
    __shared__ u32 h[1u << kPgMaxK];
    const u64 b = blockIdx.y;
    const int k = M - lb;
    const u32 D = 1u << k;
    const u32 mask = M >= 32 ? 0xffffffffu : (1u << M) - 1u;
    if (threadIdx.x < M) srow[threadIdx.x] = rows[b * M + threadIdx.x];
    for (u32 d = threadIdx.x; d < D; d += blockDim.x) h[d] = 0;
    __syncthreads();
    const u64 word = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (word < P32) {
        const u64 col0 = word * 32;
        const u32 ncol = u32(minu(32, p - col0));
        u32 a[32];
#pragma unroll
        for (int s = 0; s < 32; ++s) a[s] = s < M ? __ldg(Xr + u64(srow[s]) * P32 + word) : 0u;
        transpose32(a);
        if (STORE_KEYS) {
            u32* out = keys + b * p + col0;
            if (ncol == 32 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
                uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
                for (int c = 0; c < 8; ++c) o4[c] = make_uint4(a[4 * c], a[4 * c + 1], a[4 * c + 2], a[4 * c + 3]);
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (u32(c) < ncol) out[c] = a[c];
            }
        }
        const PartMap pm(xorc[b] & mask);
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (u32(c) < ncol) atomicAdd(&h[part_digit(pm.fwd(a[c] & mask), lb, k, hashed != 0)], 1u);
    }
    __syncthreads();
    for (u32 d = threadIdx.x; d < D; d += blockDim.x)
        if (h[d]) atomicAdd(pcnt + b * D + d, h[d]);
}

// The partition scatter from the row planes directly (binned verify: nothing
// reads the keys afterwards): each thread projects its 32 columns again, the
// CTA counts its keys per partition in shared memory (the atomic's return is
// the key's rank; order inside a partition is immaterial), reserves one range
// per (CTA, partition) at the run's cursors (part_scan) and writes the
// (w, column) records there.
// fixed_cap != 0 (PACKED only): no count pass ran — partition d of run b owns
// the fixed region [(b D + d) fixed_cap, +fixed_cap) of the record array, the
// cursors start at 0 and end as the partition sizes (part_scan turns them into
// the compact positions of the grouped columns afterwards); a record beyond its
// region is dropped and *fixed_ovf raised (the host redoes the search counted).
template <bool PACKED>
__global__ void __launch_bounds__(128, 6) project_scatter(const u32* __restrict__ Xr, u64 P32, u64 p,
                                                       const u32* __restrict__ rows, int M,
                                                       const u32* __restrict__ xorc, int lb, int hashed,
                                                       u32* __restrict__ cursor, uint2* __restrict__ pe,
                                                       u32 fixed_cap = 0, u32* __restrict__ fixed_ovf = nullptr) {
    __shared__ u32 srow[64];
    extern __shared__ u32 ps_dyn[];  // h, lstart, gbase: 2^k words each (project_scatter_smem)
    const u64 b = blockIdx.y;
    const int k = M - lb;
    const u32 D = 1u << k;
    u32* h = ps_dyn;
    u32* lstart = ps_dyn + D;
    u32* gbase = ps_dyn + 2 * D;
    const u32 mask = M >= 32 ? 0xffffffffu : (1u << M) - 1u;
    if (threadIdx.x < M) srow[threadIdx.x] = rows[b * M + threadIdx.x];
    for (u32 d = threadIdx.x; d < D; d += blockDim.x) h[d] = 0;
    __syncthreads();
    const u64 word = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    const u64 col0 = word * 32;
    const u32 ncol = word < P32 ? u32(minu(32, p - col0)) : 0u;
    const PartMap pm(xorc[b] & mask);
    u32 a[32], dr[32];  // key, then (digit << 16 | rank within the CTA's digit)
    if (word < P32) {
#pragma unroll
        for (int s2 = 0; s2 < 32; ++s2) a[s2] = s2 < M ? __ldg(Xr + u64(srow[s2]) * P32 + word) : 0u;
        transpose32(a);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            a[c] = pm.fwd(a[c] & mask);
            if (u32(c) < ncol) {
                const u32 d = part_digit(a[c], lb, k, hashed != 0);
                dr[c] = (d << 16) | atomicAdd(&h[d], 1u);
            }
        }
    }
    __syncthreads();
    // the CTA's keys grouped by partition in shared memory (lstart: exclusive scan of the counts), then every
    // partition's run written contiguously at its reserved global range
    __shared__ uint2 buf[128 * 32];
    __shared__ u32 ws[33];
    {
        const u32 per = (D + blockDim.x - 1) / blockDim.x;
        const u32 d0 = threadIdx.x * per, d1 = min(D, d0 + per);
        u32 loc = 0;
        for (u32 d = d0; d < d1; ++d) {
            gbase[d] = h[d] ? atomicAdd(cursor + b * D + d, h[d]) : 0u;
            loc += h[d];
        }
        u32 tot;
        u32 run = block_exclusive(loc, ws, &tot);
        for (u32 d = d0; d < d1; ++d) {
            lstart[d] = run;
            run += h[d];
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 32; ++c)
        if (u32(c) < ncol) buf[lstart[dr[c] >> 16] + (dr[c] & 0xffffu)] = make_uint2(a[c], u32(col0) + c);
    __syncthreads();
    const u32 nk = u32(minu(u64(blockDim.x) * 32, p - u64(blockIdx.x) * blockDim.x * 32));
    if (PACKED) {  // 4-byte records: (local bucket << (32 - lb)) | column (the partition is the record's place)
        const int cb = 32 - lb;
        const u32 lmask = (1u << lb) - 1u;
        if (fixed_cap) {
            u32* out = reinterpret_cast<u32*>(pe) + b * D * fixed_cap;
            bool over = false;
            for (u32 e = threadIdx.x; e < nk; e += blockDim.x) {
                const uint2 r = buf[e];
                const u32 d = r.x >> lb;
                const u32 pos = gbase[d] + (e - lstart[d]);
                if (pos < fixed_cap) out[u64(d) * fixed_cap + pos] = ((r.x & lmask) << cb) | r.y;
                else over = true;
            }
            if (over) *fixed_ovf = 1u;
            return;
        }
        u32* out = reinterpret_cast<u32*>(pe) + b * p;
        for (u32 e = threadIdx.x; e < nk; e += blockDim.x) {
            const uint2 r = buf[e];
            const u32 d = r.x >> lb;
            out[gbase[d] + (e - lstart[d])] = ((r.x & lmask) << cb) | r.y;
        }
        return;
    }
    uint2* out = pe + b * p;
    for (u32 e = threadIdx.x; e < nk; e += blockDim.x) {
        const uint2 r = buf[e];
        const u32 d = part_digit(r.x, lb, k, hashed != 0);
        out[gbase[d] + (e - lstart[d])] = r;
    }
}

inline size_t project_scatter_smem(int k) { return (size_t(3) << k) * 4; }

// 4-byte partition records fit when the local bucket (lb bits) and the column share 32 bits (dense partitions).
inline bool part_packed_ok(int lb, u64 p, bool hashed) {
    return !hashed && lb >= 1 && lb <= 16 && p <= (u64(1) << (32 - lb));
}

__global__ void __launch_bounds__(kPgThreads) part_count(const u32* __restrict__ keys, u64 p, int M, int lb,
                                                         int hashed, const u32* __restrict__ xorc,
                                                         u32* __restrict__ pcnt) {
    part_tile<false>(keys, p, M, lb, hashed != 0, xorc, pcnt, nullptr, nullptr);
}

__global__ void __launch_bounds__(kPgThreads) part_scatter(const u32* __restrict__ keys, u64 p, int M, int lb,
                                                           int hashed, const u32* __restrict__ xorc,
                                                           u32* __restrict__ cursor, uint2* __restrict__ pe) {
    part_tile<true>(keys, p, M, lb, hashed != 0, xorc, nullptr, cursor, pe);
}

// One CTA per run: pbeg[b][d] = run-local start of partition d (pbeg[b][D] = p);
// cursor[b][d] = pbeg[b][d]; tot / work_run of the run cleared.
__global__ void __launch_bounds__(1024) part_scan(const u32* __restrict__ pcnt, int k, u64 p, u32* __restrict__ pbeg,
                                                  u32* __restrict__ cursor, u64* __restrict__ tot,
                                                  u64* __restrict__ work_run) {
    __shared__ u32 ws[33];
    const u32 D = 1u << k, b = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 x = threadIdx.x < D ? pcnt[u64(b) * D + threadIdx.x] : 0u;
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
    }
    __syncthreads();
    const u32 ex = ws[wid] + incl - x;
    if (threadIdx.x < D) {
        pbeg[u64(b) * (D + 1) + threadIdx.x] = ex;
        cursor[u64(b) * D + threadIdx.x] = ex;
    }
    if (threadIdx.x == 0) {
        pbeg[u64(b) * (D + 1) + D] = u32(p);
        tot[b] = 0;
        work_run[b] = 0;
    }
}

// --------------------------------------------------------- partition join --

// Exclusive scan of the n counters in place (each warp owns a contiguous
// segment walked in conflict-free 32-word steps): counters -> bucket starts.
__device__ __forceinline__ void part_table_scan(u32* T, u32 n, u32* ws) {
    if (n >= 4 * blockDim.x && n % (4 * blockDim.x) == 0) {
        // large tables (2^12 buckets on 512 threads): every thread scans its own run of n / blockDim
        // consecutive counters with 16-byte accesses, one block scan of the thread sums in between
        const u32 per4 = n / (4 * blockDim.x);
        uint4* T4 = reinterpret_cast<uint4*>(T) + threadIdx.x * per4;
        u32 loc = 0;
        for (u32 q = 0; q < per4; ++q) {
            const uint4 v = T4[q];
            loc += v.x + v.y + v.z + v.w;
        }
        u32 total;
        u32 run = block_exclusive(loc, ws, &total);
        for (u32 q = 0; q < per4; ++q) {
            const uint4 v = T4[q];
            uint4 o;
            o.x = run;
            o.y = o.x + v.x;
            o.z = o.y + v.y;
            o.w = o.z + v.z;
            run = o.w + v.w;
            T4[q] = o;
        }
        __syncthreads();
        return;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 nw = blockDim.x >> 5;
    const u32 seg = max(32u, (n + nw - 1) / nw);
    const u32 s0 = min(n, u32(wid) * seg), s1 = min(n, s0 + seg);
    u32 loc = 0;
    for (u32 i = s0 + lane; i < s1; i += 32) loc += T[i];
    loc = warp_sum(loc);
    if (lane == 0) ws[wid] = loc;
    __syncthreads();
    if (wid == 0) {
        const u32 t = u32(lane) < nw ? ws[lane] : 0u;
        u32 incl = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        ws[lane] = incl - t;
    }
    __syncthreads();
    u32 carry = ws[wid];
    for (u32 i0 = s0; i0 < s1; i0 += 32) {
        const u32 i = i0 + lane;
        const u32 x = i < s1 ? T[i] : 0u;
        u32 incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (i < s1) T[i] = carry + incl - x;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncthreads();
}

template <int EMIT, bool PACKED = false>
__global__ void __launch_bounds__(kPjThreads, 3) part_join(const uint2* __restrict__ pe, const u32* __restrict__ pbeg,
                                                        u64 p, int M, int lb, const u32* __restrict__ xorc, u64 guard,
                                                        u32 hmax, u32* __restrict__ grouped, u64* __restrict__ tot,
                                                        u64* __restrict__ work_run, Item* __restrict__ items,
                                                        u32* __restrict__ nitems, u32 item_cap,
                                                        u32* __restrict__ npairs, PairRec* __restrict__ pairs,
                                                        u32 pair_cap, u32 fixed_cap) {
    extern __shared__ __align__(16) u32 T[];  // 2^lb local buckets
    __shared__ u32 ws[68];
    __shared__ u64 red[2][kPjThreads / 32];
    const u32 b = blockIdx.y, d = blockIdx.x;
    const int k = M - lb;
    const u32 D = 1u << k, L = 1u << lb, lmask = L - 1u;
    const u32 mask = M >= 32 ? 0xffffffffu : (1u << M) - 1u;
    const u32 c = xorc[b] & mask;
    if (EMIT == 1 && tot[b] > guard) return;  // aborted run: nothing to emit (uniform per CTA)
    const u32 beg = pbeg[u64(b) * (D + 1) + d], end = pbeg[u64(b) * (D + 1) + d + 1];
    // records: (w, column), or packed (local bucket << (32 - lb)) | column (project_scatter<true>), then
    // either in partition order at the run's positions or in the partition's fixed region (fixed_cap;
    // an overflowing partition keeps its first fixed_cap records and the search is redone)
    using Rec = typename std::conditional<PACKED, u32, uint2>::type;
    const u32 cnt = fixed_cap ? min(end - beg, fixed_cap) : end - beg;
    const Rec* e = reinterpret_cast<const Rec*>(pe) +
                   (fixed_cap ? (u64(b) * D + d) * fixed_cap : u64(b) * p + beg);
    const int cb = 32 - lb;
    auto bucket_of = [&](const Rec& r) -> u32 {
        if constexpr (PACKED) return r >> cb; else return r.x & lmask;
    };
    auto column_of = [&](const Rec& r) -> u32 {
        if constexpr (PACKED) return r & ((1u << cb) - 1u); else return r.y;
    };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (cnt < 2) {
        // no block with work; a lone column of a c == 0 run still counts its
        // diagonal pair in |E_r| (pair_search.cpp:48-49)
        if (EMIT != 1 && c == 0 && threadIdx.x == 0 && cnt == 1)
            atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), 1ull);
        return;
    }
    if (L >= 4) {
        for (u32 i = threadIdx.x; i < L / 4; i += blockDim.x) reinterpret_cast<uint4*>(T)[i] = make_uint4(0, 0, 0, 0);
    } else {
        for (u32 i = threadIdx.x; i < L; i += blockDim.x) T[i] = 0;
    }
    __syncthreads();
    // entries of the partition: in registers when they fit (the count's atomic
    // returns each entry's rank in its bucket, so the scatter needs no second
    // pass), else two streaming passes
    const bool inreg = cnt <= kPjPerThread * blockDim.x;
    Rec v[kPjPerThread];
    u32 rk[kPjPerThread];
    if (inreg) {
#pragma unroll
        for (int q = 0; q < kPjPerThread; ++q) {
            const u32 i = q * blockDim.x + threadIdx.x;
            v[q] = i < cnt ? __ldg(e + i) : Rec{};
        }
#pragma unroll
        for (int q = 0; q < kPjPerThread; ++q) {
            const u32 i = q * blockDim.x + threadIdx.x;
            if (i < cnt) rk[q] = atomicAdd(T + bucket_of(v[q]), 1u);
        }
    } else {
        for (u32 i0 = 0; i0 < cnt; i0 += kPjPerThread * blockDim.x) {
#pragma unroll
            for (int q = 0; q < kPjPerThread; ++q) {
                const u32 i = i0 + q * blockDim.x + threadIdx.x;
                if constexpr (PACKED) v[q] = i < cnt ? __ldg(e + i) : 0u;
                else v[q].x = i < cnt ? __ldg(&e[i].x) : 0u;
            }
#pragma unroll
            for (int q = 0; q < kPjPerThread; ++q) {
                const u32 i = i0 + q * blockDim.x + threadIdx.x;
                if (i < cnt) atomicAdd(T + bucket_of(v[q]), 1u);
            }
        }
    }
    __syncthreads();
    // c != 0: buckets u (even) and u | 1 form one block; c == 0: every bucket
    // is a diagonal block. li walks the block heads.
    const u32 NL = c ? L / 2 : L;
    if (EMIT == 0) {  // |E_r| incl. the diagonal and the canonical work (EMIT = 2: summed in the emission count walk)
        u64 pa = 0, wa = 0;
        for (u32 li = threadIdx.x; li < NL; li += blockDim.x) {
            if (c == 0) {
                const u64 cx = T[li];
                pa += cx * cx;
                wa += cx ? cx * (cx - 1) / 2 : 0;
            } else {
                const uint2 t2 = reinterpret_cast<const uint2*>(T)[li];
                pa += 2ull * t2.x * t2.y;
                wa += u64(t2.x) * t2.y;
            }
        }
        pa = warp_sum(pa);
        wa = warp_sum(wa);
        if (lane == 0) {
            red[0][wid] = pa;
            red[1][wid] = wa;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            u64 a = 0, w = 0;
            for (int q = 0; q < nw; ++q) {
                a += red[0][q];
                w += red[1][q];
            }
            if (a) atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), static_cast<unsigned long long>(a));
            if (w) atomicAdd(reinterpret_cast<unsigned long long*>(work_run + b), static_cast<unsigned long long>(w));
        }
        return;
    }
    // bucket starts, scatter (T ends as bucket ends), then the blocks
    part_table_scan(T, L, ws);
    const u64 off = u64(b) * p;
    u32* sg = T + L;  // the partition's grouped columns (in-register case)
    if (inreg) {
#pragma unroll
        for (int q = 0; q < kPjPerThread; ++q) {
            const u32 i = q * blockDim.x + threadIdx.x;
            if (i < cnt) sg[T[bucket_of(v[q])] + rk[q]] = column_of(v[q]);
        }
        __syncthreads();
    } else {
        for (u32 i0 = 0; i0 < cnt; i0 += kPjPerThread * blockDim.x) {
#pragma unroll
            for (int q = 0; q < kPjPerThread; ++q) {
                const u32 i = i0 + q * blockDim.x + threadIdx.x;
                v[q] = i < cnt ? __ldg(e + i) : Rec{};
            }
#pragma unroll
            for (int q = 0; q < kPjPerThread; ++q) {
                const u32 i = i0 + q * blockDim.x + threadIdx.x;
                if (i < cnt) grouped[off + beg + atomicAdd(T + bucket_of(v[q]), 1u)] = column_of(v[q]);
            }
        }
        __syncthreads();
    }
    // inreg: T holds bucket starts (end of u = start of u + 1, the last ends at cnt);
    // streaming: T holds bucket ends (start of u = end of u - 1)
    const PartMap pm(c);
    const u32 hi = d << lb;
    auto group = [&](u32 u, u32& gb, u32& gc) {
        u32 s0, s1;
        if (inreg) {
            s0 = T[u];
            s1 = u + 1 < L ? T[u + 1] : cnt;
        } else {
            s1 = T[u];
            s0 = u ? T[u - 1] : 0u;
        }
        gb = beg + s0;
        gc = s1 - s0;
    };
    auto block_of = [&](u32 li) {
        HeadBlock hb;
        if (c == 0) {
            u32 bx, cx;
            group(li, bx, cx);
            if (cx >= 2) {
                hb.pairs = u64(cx) * cx;
                hb.work = u64(cx) * (cx - 1) / 2;
                hb.hs = bx; hb.hc = cx; hb.ss = bx; hb.sc = cx; hb.flags = 3u;
            }
            return hb;
        }
        const u32 u = 2 * li;
        // buckets u and u | 1 hold keys v and v ^ c; the block belongs to the
        // smaller key, whose group is the x side (pair_search.cpp:35-53)
        const u32 ve = pm.inv(hi | u);
        const bool even_x = ve < (ve ^ c);
        u32 bx, cx, bz, cz;
        group(even_x ? u : (u | 1u), bx, cx);
        group(even_x ? (u | 1u) : u, bz, cz);
        if (cx && cz) {
            hb.pairs = 2ull * cx * cz;
            hb.work = u64(cx) * cz;
            if (cx <= cz) {
                hb.hs = bx; hb.hc = cx; hb.ss = bz; hb.sc = cz; hb.flags = 1u;
            } else {
                hb.hs = bz; hb.hc = cz; hb.ss = bx; hb.sc = cx; hb.flags = 0u;
            }
        }
        return hb;
    };
    const bool pair_list = npairs != nullptr;
    u32 my_items = 0, my_pairs = 0;
    u64 pa = 0, wa = 0;
    for (u32 li = threadIdx.x; li < NL; li += blockDim.x) {
        const HeadBlock hb = block_of(li);
        u32 ne, np, nsc;
        emit_count(hb, hmax, pair_list, ne, np, nsc);
        my_items += ne;
        my_pairs += np;
        if (EMIT == 2) {
            pa += hb.pairs;
            wa += hb.work;
        }
    }
    if (EMIT == 2) {  // the run's |E_r| incl. the diagonal and canonical work (the guard is applied when binned)
        if (c == 0)  // diagonal blocks: a lone column still counts its j == k pair (block_of leaves it out)
            for (u32 li = threadIdx.x; li < NL; li += blockDim.x) {
                u32 bx, cx;
                group(li, bx, cx);
                if (cx == 1) pa += 1;
            }
        pa = warp_sum(pa);
        wa = warp_sum(wa);
        if (lane == 0) {
            red[0][wid] = pa;
            red[1][wid] = wa;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            u64 a = 0, w = 0;
            for (int q = 0; q < nw; ++q) {
                a += red[0][q];
                w += red[1][q];
            }
            if (a) atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), static_cast<unsigned long long>(a));
            if (w) atomicAdd(reinterpret_cast<unsigned long long*>(work_run + b), static_cast<unsigned long long>(w));
        }
    }
    u32 ti, tp, ibase, pbase;
    block_exclusive2(my_items, my_pairs, ws, ibase, pbase, &ti, &tp);
    if (ti == 0 && tp == 0) return;
    // only items (large blocks, expanded later) read the global grouped array:
    // inline pairs carry their columns, taken from shared memory here
    if (inreg && ti)
        for (u32 i = threadIdx.x; i < cnt; i += blockDim.x) grouped[off + beg + i] = sg[i];  // coalesced
    if (threadIdx.x == 0) {
        ws[66] = ti ? atomicAdd(nitems, ti) : 0u;
        ws[67] = (pair_list && tp) ? atomicAdd(npairs, tp) : 0u;
    }
    __syncthreads();
    ibase += ws[66];
    pbase += ws[67];
    if (inreg)
        emit_blocks_warp(block_of, NL, b, hmax, p, pair_list, ibase, pbase, items, item_cap, pairs, pair_cap, grouped,
                         sg, beg);
    else
        emit_blocks_warp(block_of, NL, b, hmax, p, pair_list, ibase, pbase, items, item_cap, pairs, pair_cap, grouped,
                         grouped + off, 0u);
}

inline size_t part_tile_smem(int k) { return size_t(kPgThreads / 32) * (size_t(1) << k) * 4; }
inline size_t part_join_smem(int lb) { return ((size_t(1) << lb) + kPjThreads * kPjPerThread) * 4; }

// ------------------------------------------------ hashed partition join --
//
// Sparse bucket spaces (2^M >> p, e.g. config 3: M = 20, p = 5e4): a dense
// 2^lb table per partition would be mostly empty, so the partition's local
// keys go into an open-addressing hash table in shared memory instead
// (kHsSlots slots for at most kHsCap records, load <= 1/2). A slot holds a
// key PAIR g = w >> 1 — a key w and its partner w ^ 1 (the T map, PartMap)
// share the slot — with both counts in one word (even key low 16 bits, odd
// key high 16 bits): the insertion's count atomic returns each record's rank,
// and a block's partner count sits in the same slot, so no partner probe is
// needed. The occupied slots are listed as they are claimed, and the table
// passes walk that list only. A partition above kHsCap records (a skewed key
// distribution) is not processed: the kernel raises *ovf and the host redoes
// the search on the sorted path.
constexpr int kHsThreads = 512;
constexpr int kHsPer = 4;
constexpr u32 kHsCap = kHsThreads * kHsPer;  // 2048 records per partition
constexpr u32 kHsSlots = 2 * kHsCap;
constexpr u32 kHsEmpty = 0xffffffffu;

// Slot hash (12 bits: kHsSlots = 4096): a full avalanche finalizer, so the
// slot bits are independent of the partition digit (a multiplicative hash of
// w >> 1 that every key of the partition shares in its top bits).
__device__ __forceinline__ u32 hs_hash(u32 u) {
    u ^= u >> 16;
    u *= 0x85EBCA6Bu;
    u ^= u >> 13;
    u *= 0xC2B2AE35u;
    u ^= u >> 16;
    return u >> 20;
}

template <int EMIT>
__global__ void __launch_bounds__(kHsThreads) part_join_hash(const uint2* __restrict__ pe, const u32* __restrict__ pbeg,
                                                             u64 p, int M, int lb, const u32* __restrict__ xorc,
                                                             u64 guard, u32 hmax, u32* __restrict__ grouped,
                                                             u64* __restrict__ tot, u64* __restrict__ work_run,
                                                             Item* __restrict__ items, u32* __restrict__ nitems,
                                                             u32 item_cap, u32* __restrict__ npairs,
                                                             PairRec* __restrict__ pairs, u32 pair_cap,
                                                             u32* __restrict__ ovf) {
    extern __shared__ __align__(16) u32 hsm[];
    u32* tk = hsm;                  // [kHsSlots] key pairs g = w >> 1
    u32* tc = tk + kHsSlots;        // [kHsSlots] counts: even key (low 16 bits), odd key (high 16 bits)
    u32* occ = tc + kHsSlots;       // [kHsCap] occupied slots
    u32* ts = occ + kHsCap;         // [kHsSlots] grouped start of the slot's records that are in a block
    u32* sg = ts + kHsSlots;        // [kHsCap] grouped columns
    u32* heads = sg + kHsCap;       // [kHsCap] block heads: slot * 2 + key parity
    __shared__ u32 ws[68];
    __shared__ u32 s_nheads, s_cursor, s_nocc;
    __shared__ u64 red[2][kHsThreads / 32];
    const u32 b = blockIdx.y, d = blockIdx.x;
    const int k = M - lb;
    const u32 D = 1u << k;
    const u32 mask = M >= 32 ? 0xffffffffu : (1u << M) - 1u;
    const u32 c = xorc[b] & mask;
    if (EMIT && tot[b] > guard) return;
    const u32 beg = pbeg[u64(b) * (D + 1) + d], end = pbeg[u64(b) * (D + 1) + d + 1];
    const u32 cnt = end - beg;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (cnt > kHsCap) {  // uniform: redo the search on the sorted path
        if (threadIdx.x == 0) atomicExch(ovf, 1u);
        return;
    }
    if (cnt < 2) {
        if (EMIT != 1 && c == 0 && threadIdx.x == 0 && cnt == 1)
            atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), 1ull);
        return;
    }
    for (u32 i = threadIdx.x; i < kHsSlots; i += blockDim.x) {
        tk[i] = kHsEmpty;
        tc[i] = 0;
    }
    if (threadIdx.x == 0) {
        s_nheads = 0;
        s_cursor = 0;
        s_nocc = 0;
    }
    __syncthreads();
    const uint2* e = pe + u64(b) * p + beg;
    uint2 v[kHsPer];
    u32 slot[kHsPer], rk[kHsPer];
#pragma unroll
    for (int q = 0; q < kHsPer; ++q) {
        const u32 i = q * blockDim.x + threadIdx.x;
        v[q] = i < cnt ? __ldg(e + i) : make_uint2(0, 0);
    }
#pragma unroll
    for (int q = 0; q < kHsPer; ++q) {
        const u32 i = q * blockDim.x + threadIdx.x;
        if (i < cnt) {
            const u32 u = v[q].x;  // the whole key w (partitions are hashed, M <= 31)
            const u32 g = u >> 1;
            u32 h = hs_hash(g);
            for (;;) {
                const u32 old = atomicCAS(tk + h, kHsEmpty, g);
                if (old == kHsEmpty) {
                    occ[atomicAdd(&s_nocc, 1u)] = h;
                    break;
                }
                if (old == g) break;
                h = (h + 1) & (kHsSlots - 1);
            }
            slot[q] = h;
            const u32 sh = (u & 1u) << 4;
            rk[q] = (atomicAdd(tc + h, 1u << sh) >> sh) & 0xffffu;
        }
    }
    __syncthreads();
    const u32 nocc = s_nocc;
    if (!EMIT) {
        u64 pa = 0, wa = 0;
        for (u32 o = threadIdx.x; o < nocc; o += blockDim.x) {
            const u32 t2 = tc[occ[o]];
            const u64 ce = t2 & 0xffffu, co = t2 >> 16;
            if (c == 0) {
                pa += ce * ce + co * co;
                wa += (ce ? ce * (ce - 1) / 2 : 0) + (co ? co * (co - 1) / 2 : 0);
            } else {
                pa += 2 * ce * co;
                wa += ce * co;
            }
        }
        pa = warp_sum(pa);
        wa = warp_sum(wa);
        if (lane == 0) {
            red[0][wid] = pa;
            red[1][wid] = wa;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            u64 a = 0, w = 0;
            for (int q = 0; q < nw; ++q) {
                a += red[0][q];
                w += red[1][q];
            }
            if (a) atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), static_cast<unsigned long long>(a));
            if (w) atomicAdd(reinterpret_cast<unsigned long long*>(work_run + b), static_cast<unsigned long long>(w));
        }
        return;
    }
    // Only keys that are in a block are grouped: c == 0, a key with >= 2
    // records (a diagonal block); else a slot holding both keys of the pair.
    // A slot reserves one grouped range (order is irrelevant): its even key's
    // records first, then the odd key's; records of keys in no block are
    // dropped — no pair references them.
    for (u32 o = threadIdx.x; o < nocc; o += blockDim.x) {
        const u32 h = occ[o];
        const u32 t2 = tc[h];
        const u32 ce = t2 & 0xffffu, co = t2 >> 16;
        u32 ne = 0, no = 0;
        if (c == 0) {
            ne = ce >= 2 ? ce : 0u;
            no = co >= 2 ? co : 0u;
            if (ne) heads[atomicAdd(&s_nheads, 1u)] = 2 * h;
            if (no) heads[atomicAdd(&s_nheads, 1u)] = 2 * h + 1;
        } else if (ce && co) {
            ne = ce;
            no = co;
            heads[atomicAdd(&s_nheads, 1u)] = 2 * h;
        }
        ts[h] = (ne + no) ? atomicAdd(&s_cursor, ne + no) : kHsEmpty;
    }
    __syncthreads();
    const u32 nheads = s_nheads, used = s_cursor;
    if (nheads == 0) return;
#pragma unroll
    for (int q = 0; q < kHsPer; ++q) {
        const u32 i = q * blockDim.x + threadIdx.x;
        if (i < cnt) {
            const u32 h = slot[q], base = ts[h];
            if (base == kHsEmpty) continue;
            const u32 t2 = tc[h];
            const u32 ce = t2 & 0xffffu, co = t2 >> 16;
            const bool odd = v[q].x & 1u;
            if (c == 0 && (odd ? co : ce) < 2) continue;  // a lone key of a c == 0 run
            const u32 odd_off = c == 0 ? (ce >= 2 ? ce : 0u) : ce;
            sg[base + (odd ? odd_off : 0u) + rk[q]] = v[q].y;
        }
    }
    __syncthreads();
    const u64 off = u64(b) * p;
    for (u32 i = threadIdx.x; i < used; i += blockDim.x) grouped[off + beg + i] = sg[i];
    const PartMap pm(c);
    auto block_of = [&](u32 t) {
        HeadBlock hb;
        const u32 hh = heads[t], h = hh >> 1;
        const u32 t2 = tc[h];
        const u32 ce = t2 & 0xffffu, co = t2 >> 16;
        const u32 base = beg + ts[h];
        if (c == 0) {
            const bool odd = hh & 1u;
            const u32 cx = odd ? co : ce;
            const u32 bx = base + (odd ? (ce >= 2 ? ce : 0u) : 0u);
            hb.pairs = u64(cx) * cx;
            hb.work = u64(cx) * (cx - 1) / 2;
            hb.hs = bx; hb.hc = cx; hb.ss = bx; hb.sc = cx; hb.flags = 3u;
            return hb;
        }
        const u32 ue = tk[h] << 1;  // the even key of the pair
        const u32 ve = pm.inv(ue);
        const bool even_x = ve < (ve ^ c);
        const u32 bx = even_x ? base : base + ce, cx = even_x ? ce : co;
        const u32 bz = even_x ? base + ce : base, cz = even_x ? co : ce;
        hb.pairs = 2ull * cx * cz;
        hb.work = u64(cx) * cz;
        if (cx <= cz) {
            hb.hs = bx; hb.hc = cx; hb.ss = bz; hb.sc = cz; hb.flags = 1u;
        } else {
            hb.hs = bz; hb.hc = cz; hb.ss = bx; hb.sc = cx; hb.flags = 0u;
        }
        return hb;
    };
    const bool pair_list = npairs != nullptr;
    u32 my_items = 0, my_pairs = 0;
    for (u32 h = threadIdx.x; h < nheads; h += blockDim.x) {
        const HeadBlock hb = block_of(h);
        u32 ne, np, nsc;
        emit_count(hb, hmax, pair_list, ne, np, nsc);
        my_items += ne;
        my_pairs += np;
    }
    u32 ti, tp;
    u32 ibase = block_exclusive(my_items, ws, &ti);
    u32 pbase = block_exclusive(my_pairs, ws + 33, &tp);
    if (ti == 0 && tp == 0) return;
    if (threadIdx.x == 0) {
        ws[66] = ti ? atomicAdd(nitems, ti) : 0u;
        ws[67] = (pair_list && tp) ? atomicAdd(npairs, tp) : 0u;
    }
    __syncthreads();
    ibase += ws[66];
    pbase += ws[67];
    emit_blocks_coop(block_of, nheads, b, hmax, p, pair_list, ibase, pbase, items, item_cap, pairs, pair_cap,
                     grouped, sg, beg);
}

// Dynamic shared memory of the hashed join: keys + counts + occupied slots
// (+ starts, grouped columns and block heads for the emitting kernel).
inline size_t part_hash_smem(bool emit) {
    return size_t(2 * kHsSlots + kHsCap + (emit ? kHsSlots + 2 * kHsCap : 0)) * 4;
}

// Partition digits of the hashed path: mean partition <= 0.85 kHsCap (a
// balanced partition stays below kHsCap by > 6 standard deviations).
inline int part_digits_hash(int M, u64 p) {
    int k = 1;
    while (k < kPgMaxK && k < M - 1 && (p >> k) > u64(kHsCap) * 85 / 100) ++k;
    return std::min(k, M - 1);
}

// The partitioned path (u32 keys, M <= 31). k partition digits; scratch:
// pcnt / cursor B * 2^k u32, pbeg B * (2^k + 1) u32; pe: B * p (w, column).
inline u64 part_scratch_words(int k, u64 B) { return B * ((u64(1) << k) * 3 + 1); }

// counted: the partition sizes are already in scratch[0, B * 2^k) (project_count)
inline void part_partition_launch(const u32* keys, u64 B, u64 p, int M, int k, bool hashed, const u32* xorc,
                                  u64* tot, u64* work_run, u32* scratch, uint2* pe, cudaStream_t st,
                                  bool counted = false, bool scatter = true) {
    const int lb = M - k;
    const u64 D = u64(1) << k;
    u32* pcnt = scratch;
    u32* cursor = scratch + B * D;
    u32* pbeg = scratch + 2 * B * D;
    func_smem(part_count, 64 << 10);
    func_smem(part_scatter, 64 << 10);
    dim3 gt(static_cast<u32>(ceil_div(p, kPgTile)), static_cast<u32>(B));
    if (!counted) {
        XYZB_CUDA(cudaMemsetAsync(pcnt, 0, B * D * 4, st));
        part_count<<<gt, kPgThreads, part_tile_smem(k), st>>>(keys, p, M, lb, hashed ? 1 : 0, xorc, pcnt);
        XYZB_LAUNCH_CHECK();
    }
    part_scan<<<static_cast<u32>(B), 1024, 0, st>>>(pcnt, k, p, pbeg, cursor, tot, work_run);
    XYZB_LAUNCH_CHECK();
    if (!scatter) return;  // project_scatter writes the records
    part_scatter<<<gt, kPgThreads, part_tile_smem(k), st>>>(keys, p, M, lb, hashed ? 1 : 0, xorc, cursor, pe);
    XYZB_LAUNCH_CHECK();
}

// hash: the hashed join (ovf raised when a partition exceeds kHsCap records).
inline void part_join_launch(u64 B, u64 p, int M, int k, bool hash, const u32* xorc, u64 guard, u32 hmax,
                             u32* grouped, u64* tot, u64* work_run, Item* items, u32* nitems, u32 item_cap,
                             u32* npairs, PairRec* pairs, u32 pair_cap, const u32* scratch, const uint2* pe,
                             u32* ovf, cudaStream_t st, bool one_pass = false, bool packed = false,
                             u32 fixed_cap = 0) {
    const int lb = M - k;
    const u64 D = u64(1) << k;
    const u32* pbeg = scratch + 2 * B * D;
    dim3 gj(static_cast<u32>(D), static_cast<u32>(B));
    if (hash) {
        func_smem(part_join_hash<0>, part_hash_smem(true));
        func_smem(part_join_hash<1>, part_hash_smem(true));
        part_join_hash<0><<<gj, kHsThreads, part_hash_smem(false), st>>>(pe, pbeg, p, M, lb, xorc, guard, hmax, grouped, tot, work_run,
                                                     items, nitems, item_cap, npairs, pairs, pair_cap, ovf);
        XYZB_LAUNCH_CHECK();
        part_join_hash<1><<<gj, kHsThreads, part_hash_smem(true), st>>>(pe, pbeg, p, M, lb, xorc, guard, hmax, grouped, tot, work_run,
                                                     items, nitems, item_cap, npairs, pairs, pair_cap, ovf);
        XYZB_LAUNCH_CHECK();
        return;
    }
    auto launch = [&](auto kernel, size_t smem) {
        func_smem(kernel, 64 << 10);
        kernel<<<gj, kPjThreads, smem, st>>>(pe, pbeg, p, M, lb, xorc, guard, hmax, grouped, tot, work_run, items, nitems,
                                             item_cap, npairs, pairs, pair_cap, fixed_cap);
        XYZB_LAUNCH_CHECK();
    };
    if (one_pass) {
        if (packed) launch(part_join<2, true>, part_join_smem(lb));
        else launch(part_join<2, false>, part_join_smem(lb));
        return;
    }
    if (packed) {
        launch(part_join<0, true>, (size_t(1) << lb) * 4);
        launch(part_join<1, true>, part_join_smem(lb));
    } else {
        launch(part_join<0, false>, (size_t(1) << lb) * 4);
        launch(part_join<1, false>, part_join_smem(lb));
    }
}

} // namespace kern
} // namespace xyzb
