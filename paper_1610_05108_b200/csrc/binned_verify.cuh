// Binned verification for X far larger than L2 (BASELINE config 4: 1e6
// columns x 1280 B = 1.26 GB, 10x L2) — the pair strengths of
// pair_search.hpp:104-106 / transforms.cpp:33-40 (popc(X_j ^ X_k ^ Y)), the
// same numbers verify_pairs_simple computes, in an order that reuses columns.
//
// The per-batch verify reads both columns of a candidate from DRAM (~1.29
// columns per pair, the in-block reuse limit). Here the
// search's canonical pairs are instead collected over ALL batches and
// bucketed by (kt, jt): kt = the z-side column's window of 2^wshift columns
// (sized to stay L2-resident, ~84 MB), jt = the x-side column's tile of
// kBinJT columns. The verify walks the bins kt-major with one persistent
// 1024-thread CTA per SM: the bin's x-side tile sits in shared memory
// (cp.async, double-buffered, pre-XORed with Y), the z-side columns come
// from the current window in L2 (evict_last). Per pair: one column from L2,
// one from shared memory; DRAM reads ~ one window pass + one tile pass per
// window (tools/tile_probe.cu: 3.9e8 random pairs in 50 ms against 85-98 ms
// for DRAM gathers).
//
// Pair records (u64): x-side column (24 bits) | z-side column (24) | diagonal
// flag (1, at bit 48) | the run's pass is negative (1, bit 49) | global run
// index in execution order (14, at bit 50).
//   bin_scatter1  (per batch)  the batch's pair list -> per-window regions
//   bin_hist2 / bin_scan2 / bin_scatter2 (end of the search)  each window's
//                 region -> bins by x-side tile (counting sort, shared
//                 histograms, one global reservation per (chunk, bin))
//   verify_binned (per window) strengths; hits (or, top-K first phase, the
//                 rank of every pair) exactly as verify_pairs_simple
//   emit_binned   top-K first phase: append the pairs at or above E
#pragma once

#include "common.cuh"
#include "search_kernels.cuh"
#include "topk_kernels.cuh"

namespace xyzb {
namespace bins {

using kern::DevHit;
using kern::PairRec;

constexpr int kBinJT = 64;           // x-side columns per tile (shared memory: 64 x 1280 B at n = 1e4)
constexpr int kBinJTShift = 6;
constexpr int kVerifyThreads = 1024;  // one CTA per SM
constexpr int kScatterThreads = 1024;
constexpr u32 kChunk2 = 131072;       // records per level-2 chunk (8 per bin at p = 1e6)
constexpr int kColBits = 24;          // columns < 2^24
constexpr int kRunBits = 14;          // runs < 2^14 per search

__host__ __device__ __forceinline__ u64 rec_make(u32 a, u32 b, u32 diag, u32 neg, u32 run) {
    return u64(a) | (u64(b) << 24) | (u64(diag & 1u) << 48) | (u64(neg & 1u) << 49) | (u64(run) << 50);
}
__device__ __forceinline__ u32 rec_a(u64 r) { return u32(r) & 0xffffffu; }
__device__ __forceinline__ u32 rec_b(u64 r) { return u32(r >> 24) & 0xffffffu; }
__device__ __forceinline__ u32 rec_diag(u64 r) { return u32(r >> 48) & 1u; }
__device__ __forceinline__ u32 rec_neg(u64 r) { return u32(r >> 49) & 1u; }
__device__ __forceinline__ u32 rec_run(u64 r) { return u32(r >> 50); }

// ---- level 1: a batch's pair list -> per-window regions (kt = z column >> wshift) ----
// CTA chunks of 8 records per thread; shared counts per window, one global
// reservation per (chunk, window); a region past its capacity raises the
// cursor beyond cap (the host regrows and redoes the search).
constexpr int kS1Threads = 256, kS1PerThread = 8;
__global__ void __launch_bounds__(kS1Threads) bin_scatter1(const PairRec* __restrict__ pairs,
                                                           const u32* __restrict__ npairs, u32 pair_cap,
                                                           const u32* __restrict__ nitems, u32 item_cap, u32 run0,
                                                           const int8_t* __restrict__ run_sign, int wshift, int nkt, u64* __restrict__ S1, u64 cap_kt,
                                                           u32* __restrict__ cur1) {
    __shared__ u32 h[256];
    __shared__ u32 base[256];
    const u32 P = topk::batch_pairs(npairs, pair_cap, nitems, item_cap);
    constexpr u32 CH = kS1Threads * kS1PerThread;
    for (u32 i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (u64 c0 = u64(blockIdx.x) * CH; c0 < P; c0 += u64(gridDim.x) * CH) {
        u64 rec[kS1PerThread];
        u32 kt[kS1PerThread], rk[kS1PerThread];
#pragma unroll
        for (int u = 0; u < kS1PerThread; ++u) {
            const u64 i = c0 + u64(u) * kS1Threads + threadIdx.x;
            kt[u] = 0xffffffffu;
            if (i < P) {
                const PairRec pr = pairs[i];
                rec[u] = rec_make(pr.pa, pr.pb, (pr.pad >> 1) & 1u, run_sign[pr.run] < 0 ? 1u : 0u, run0 + pr.run);
                kt[u] = pr.pb >> wshift;
                rk[u] = atomicAdd(&h[kt[u]], 1u);
            }
        }
        __syncthreads();
        for (int t = threadIdx.x; t < nkt; t += blockDim.x) {
            const u32 cnt = h[t];
            base[t] = cnt ? atomicAdd(cur1 + t, cnt) : 0u;
            h[t] = 0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < kS1PerThread; ++u) {
            if (kt[u] == 0xffffffffu) continue;
            const u64 pos = u64(base[kt[u]]) + rk[u];
            if (pos < cap_kt) S1[u64(kt[u]) * cap_kt + pos] = rec[u];
        }
    }
}

// ---- level 2: each window's region -> bins by x-side tile ----
// Work items (window, chunk) flattened window-major; chunks past the region's
// count are skipped. hist: per-chunk shared counts added to gh[kt][jt].
__global__ void __launch_bounds__(kScatterThreads) bin_hist2(const u64* __restrict__ S1, u64 cap_kt,
                                                             const u32* __restrict__ cur1, int nkt, u32 chunks_per_kt,
                                                             u32 nbj, u32* __restrict__ gh) {
    extern __shared__ u32 h2[];
    for (u32 w = blockIdx.x; w < u32(nkt) * chunks_per_kt; w += gridDim.x) {
        const u32 kt = w / chunks_per_kt, ch = w % chunks_per_kt;
        const u64 cnt = minu(cur1[kt], cap_kt);
        const u64 r0 = u64(ch) * kChunk2;
        if (r0 >= cnt) continue;  // uniform over the CTA
        const u64 r1 = minu(cnt, r0 + kChunk2);
        for (u32 i = threadIdx.x; i < nbj; i += blockDim.x) h2[i] = 0;
        __syncthreads();
        const u64* src = S1 + u64(kt) * cap_kt;
        for (u64 i = r0 + threadIdx.x; i < r1; i += blockDim.x) atomicAdd(&h2[rec_a(src[i]) >> kBinJTShift], 1u);
        __syncthreads();
        u32* g = gh + u64(kt) * nbj;
        for (u32 i = threadIdx.x; i < nbj; i += blockDim.x)
            if (h2[i]) atomicAdd(g + i, h2[i]);
        __syncthreads();
    }
}

// One CTA per window: exclusive scan of its bin counts -> boff[kt][0..nbj]
// (boff[kt][nbj] = the window's total) and the scatter cursors.
__global__ void __launch_bounds__(1024) bin_scan2(const u32* __restrict__ gh, u32 nbj, u32* __restrict__ boff,
                                                  u32* __restrict__ cur2) {
    __shared__ u32 ws[33];
    const u32 kt = blockIdx.x;
    const u32* g = gh + u64(kt) * nbj;
    u32* bo = boff + u64(kt) * (nbj + 1);
    u32* cu = cur2 + u64(kt) * nbj;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const u32 per = (nbj + blockDim.x - 1) / blockDim.x;
    const u32 s0 = threadIdx.x * per, s1 = min(nbj, s0 + per);
    u32 loc = 0;
    for (u32 i = s0; i < s1; ++i) loc += g[i];
    u32 incl = loc;
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
    u32 run = ws[wid] + incl - loc;
    for (u32 i = s0; i < s1; ++i) {
        bo[i] = run;
        cu[i] = run;
        run += g[i];
    }
    if (threadIdx.x == 0) bo[nbj] = ws[32];
}

// Scatter: per chunk, shared counts -> one reservation per nonzero bin ->
// second pass over the (L2-resident) chunk writes each record at its bin's
// reserved base + a shared rank. Order within a bin is immaterial.
__global__ void __launch_bounds__(kScatterThreads) bin_scatter2(const u64* __restrict__ S1, u64 cap_kt,
                                                                const u32* __restrict__ cur1, int nkt,
                                                                u32 chunks_per_kt, u32 nbj, u32* __restrict__ cur2,
                                                                u64* __restrict__ F) {
    extern __shared__ u32 h2[];  // [nbj] counts, then bases; [nbj] ranks
    u32* rk = h2 + nbj;
    for (u32 w = blockIdx.x; w < u32(nkt) * chunks_per_kt; w += gridDim.x) {
        const u32 kt = w / chunks_per_kt, ch = w % chunks_per_kt;
        const u64 cnt = minu(cur1[kt], cap_kt);
        const u64 r0 = u64(ch) * kChunk2;
        if (r0 >= cnt) continue;
        const u64 r1 = minu(cnt, r0 + kChunk2);
        for (u32 i = threadIdx.x; i < nbj; i += blockDim.x) {
            h2[i] = 0;
            rk[i] = 0;
        }
        __syncthreads();
        const u64* src = S1 + u64(kt) * cap_kt;
        for (u64 i = r0 + threadIdx.x; i < r1; i += blockDim.x) atomicAdd(&h2[rec_a(src[i]) >> kBinJTShift], 1u);
        __syncthreads();
        u32* cu = cur2 + u64(kt) * nbj;
        for (u32 i = threadIdx.x; i < nbj; i += blockDim.x)
            if (h2[i]) h2[i] = atomicAdd(cu + i, h2[i]);
        __syncthreads();
        u64* dst = F + u64(kt) * cap_kt;
        for (u64 i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
            const u64 r = src[i];
            const u32 jt = rec_a(r) >> kBinJTShift;
            dst[h2[jt] + atomicAdd(&rk[jt], 1u)] = r;
        }
        __syncthreads();
    }
}

// ---- verify one window's bins ----
struct BinVerifyArgs {
    const u64* Xc;
    u32 Wp;
    const u64* Yw;
    u32 n, astar;
    u64 p;
    const u64* F;       // the window's region (bins by x-side tile)
    const u32* boff;    // the window's bin offsets [nbj + 1]
    u32 nbj;
    const u32* rid;          // global run ids by run index
    DevHit* hits;
    u32* hit_count;
    u32 hit_cap;
    const u32* krows;  // the runs' draws [R][M]: x-side keys of hits
    int kM;
    u32* sint_out;        // top-K first phase: rank of every pair of this window (thr == 0)
    const u32* rank_thr;  // top-K running threshold (nullptr: hits mode)
};

__device__ __forceinline__ u32 smem_u32(const void* p) { return u32(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ ulonglong2 ld_keep(const ulonglong2* p, u64 pol) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                 : "=l"(v.x), "=l"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// Team of 16 lanes per pair, NS 16-byte slices per lane (W2 = Wp/2 <= 16 NS),
// two pairs in flight per team; the loops are warp-uniform (full-warp shuffles).
template <int NS, bool FULL>
__global__ void __launch_bounds__(kVerifyThreads, 1) verify_binned(BinVerifyArgs A) {
    constexpr int G = 16, PR = 2, TPW = 32 / G, NWARPS = kVerifyThreads / 32;
    extern __shared__ __align__(128) ulonglong2 tiles[];  // [2][kBinJT][W2]
    const u32 W2 = A.Wp / 2;
    const u32 tile_elems = u32(kBinJT) * W2;
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const u32 warp = threadIdx.x >> 5, tw = (threadIdx.x / G) % TPW;
    const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(A.Xc);
    const ulonglong2* Y2 = reinterpret_cast<const ulonglong2*>(A.Yw);
    u64 pol = 0, tpol = 0;  // the window stays (evict_last), the tiles stream through (evict_first)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(tpol));
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    const bool ranks = A.sint_out != nullptr && rthr == 0;
    const u32 astar = max(A.astar, rthr);
    auto load_tile = [&](u32 jt, int s) {
        const u32 c0 = jt << kBinJTShift;
        const u32 ncol = u32(minu(A.p - c0, kBinJT));
        const bool any = A.boff[jt + 1] > A.boff[jt];
        if (any) {
            const ulonglong2* src = X2 + u64(c0) * W2;
            ulonglong2* dst = tiles + u32(s) * tile_elems;
            for (u32 e = threadIdx.x; e < ncol * W2; e += blockDim.x)
                asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst + e)),
                             "l"(src + e), "l"(tpol)
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (blockIdx.x < A.nbj) load_tile(blockIdx.x, 0);
    u32 i = 0;
    for (u32 jt = blockIdx.x; jt < A.nbj; jt += gridDim.x, ++i) {
        const int s = i & 1;
        if (jt + gridDim.x < A.nbj) {
            load_tile(jt + gridDim.x, s ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        const u32 r0 = A.boff[jt], r1 = A.boff[jt + 1];
        ulonglong2* tile = tiles + u32(s) * tile_elems;
        if (r1 > r0) {
            // pre-XOR the response into the x-side tile: popc(a ^ y ^ b) per pair
            const u32 ncol = u32(minu(A.p - (u64(jt) << kBinJTShift), kBinJT));
            for (u32 e = threadIdx.x; e < ncol * W2; e += blockDim.x) {
                const ulonglong2 y = __ldg(Y2 + e % W2);
                ulonglong2 v = tile[e];
                v.x ^= y.x;
                v.y ^= y.y;
                tile[e] = v;
            }
            __syncthreads();
            const u32 c0 = jt << kBinJTShift;
            constexpr u32 STRIDE = NWARPS * TPW * PR;
            // the next iteration's records are loaded one iteration ahead (record -> column is a dependent chain)
            u64 nrec[PR];
#pragma unroll
            for (int r = 0; r < PR; ++r) {
                const u32 q = r0 + warp * TPW * PR + tw * PR + r;
                nrec[r] = q < r1 ? __ldg(A.F + q) : 0ull;
            }
            for (u32 q0 = r0 + warp * TPW * PR; q0 < r1; q0 += STRIDE) {  // warp-uniform
                const u32 qb = q0 + tw * PR;
                ulonglong2 kv[PR][NS];
                u64 rec[PR];
#pragma unroll
                for (int r = 0; r < PR; ++r) {
                    const u32 q = qb + r;
                    rec[r] = nrec[r];
                    const ulonglong2* kc = X2 + u64(rec_b(rec[r])) * W2;
#pragma unroll
                    for (int it = 0; it < NS; ++it) {
                        const u32 wi = it * G + tl;
                        kv[r][it] = (q < r1 && (FULL || wi < W2)) ? ld_keep(kc + wi, pol) : make_ulonglong2(0, 0);
                    }
                }
#pragma unroll
                for (int r = 0; r < PR; ++r) {
                    const u32 q = qb + STRIDE + r;
                    nrec[r] = q < r1 ? __ldg(A.F + q) : 0ull;
                }
#pragma unroll
                for (int r = 0; r < PR; ++r) {
                    const u32 q = qb + r;
                    const u32 jl = q < r1 ? rec_a(rec[r]) - c0 : 0u;
                    const ulonglong2* a = tile + jl * W2 + tl;
                    u32 acc = 0;
#pragma unroll
                    for (int it = 0; it < NS; ++it) {
                        if (FULL || it * G + tl < W2) {
                            const ulonglong2 av = a[it * G];
                            acc += __popcll(av.x ^ kv[r][it].x) + __popcll(av.y ^ kv[r][it].y);
                        }
                    }
#pragma unroll
                    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                    if (tl == 0 && q < r1) {
                        const u32 si = rec_neg(rec[r]) ? A.n - acc : acc;  // the run's sign (search.cpp:25-36)
                        if (ranks) {
                            A.sint_out[q] = si;
                        } else if (si >= astar) {
                            PairRec pr{rec_a(rec[r]), rec_b(rec[r]), rec_run(rec[r]), rec_diag(rec[r]) << 1};
                            kern::append_pair_hit(nullptr, 0, 0, A.rid, A.hits, A.hit_count, A.hit_cap, pr, si, A.n,
                                                  A.krows, A.kM, A.Xc, A.Wp);
                        }
                    }
                }
            }
        }
        __syncthreads();  // the tile buffer is refilled next iteration
    }
}

// Top-K first phase over a window: append its pairs with rank >= E (as topk::emit_pairs).
__global__ void __launch_bounds__(256) emit_binned(const u64* __restrict__ F, const u32* __restrict__ sint,
                                                   const u32* __restrict__ count, const topk::State* __restrict__ st,
                                                   const u32* __restrict__ rid, const u32* __restrict__ krows, int kM,
                                                   const u64* __restrict__ Xc, u32 Wp, DevHit* __restrict__ hits,
                                                   u32* __restrict__ hit_count, u32 hit_cap, u32 n) {
    if (st->thr > 0) return;
    const u32 P = *count;
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
                const u64 rc = F[i];
                u32 j = rec_a(rc), k = rec_b(rc);
                if (rec_diag(rc) && j > k) {
                    const u32 t = j;
                    j = k;
                    k = t;
                }
                const u32 run = rec_run(rc);
                DevHit h;
                h.order = kern::key_of_column(krows + u64(run) * kM, kM, Xc, Wp, j);
                h.s = double(r) / double(n);
                h.j = j;
                h.k = k;
                h.rid = rid[run];
                h.sint = int32_t(r);
                hits[slot] = h;
            }
        }
    }
}

inline size_t verify_smem(u32 Wp) { return size_t(2) * kBinJT * (Wp / 2) * 16; }

} // namespace bins
} // namespace xyzb
