// Binned verification for X far larger than L2 (BASELINE config 4: 1e6
// columns x 1280 B = 1.26 GB, 10x L2) — the pair strengths of
// pair_search.hpp:104-106 / transforms.cpp:33-40 (popc(X_j ^ X_k ^ Y)), the
// same numbers verify_pairs_simple computes, in an order that reuses columns.
//
// The per-batch verify reads both columns of a candidate from DRAM (~1.29
// columns per pair, the in-block reuse limit). Here the
// search's canonical pairs are instead collected over ALL batches into bins
// (kt, jt): kt = the z-side column's window of 2^wshift columns (sized to
// stay L2-resident, ~84 MB), jt = the x-side column's tile of kBinJT
// columns. The verify walks the bins of one window per launch with one
// persistent 1024-thread CTA per SM: the bin's x-side tile (from X ^ Y) sits
// in shared memory (TMA bulk copies into a two-deep mbarrier ring, no CTA
// barrier), the z-side columns come from the current window in L2
// (evict_last). Per pair: one column from L2, one from shared memory; DRAM
// ~ one window pass + one tile pass per window (tools/tile_probe.cu; ncu: 244
// DRAM bytes per pair against 1619).
//
// Three partition passes put the pairs in bins, each a small fan-out so the
// writes stay long runs: per batch, each pair goes to its z-side window (16
// regions at config 4); after the last batch, each window is split by the
// x-side tile >> 7 (128 buckets), and one CTA per bucket splits it by the
// tile's low 7 bits (every tile a fixed 1/128 of the bucket's region);
// tile_sort then orders every tile by x column. Regions have fixed
// capacities from the previous search's mean fills; a pair whose region is
// full goes to an overflow list, verified afterwards by a plain gather; an
// overflowing list makes the host redo the search with a larger one.
//
// Pair records (u64): x-side column (24 bits) | z-side column (24) | diagonal
// flag (1, at bit 48) | the run's pass is negative (1, bit 49) | global run
// index in execution order (14, at bit 50).
//   bin_window   (per batch)  the batch's pair list -> windows (or the overflow list)
//   bin_split    (end)        each window -> buckets by x-side tile >> 7
//   bin_sort     (end)        each bucket -> its 128 tiles' runs
//   tile_sort    (end)        each tile ordered by x column, in place
//   bin_scan     (end)        per window, exclusive offsets of the tile fills
//                             (compact rank indices for the top-K first phase)
//   xor_response (end)        X ^ Y, the source of the x tiles
//   verify_binned (per window) strengths; hits (or, top-K first phase, the
//                 rank of every pair) exactly as verify_pairs_simple
//   verify_list  the overflow list (warp per pair)
//   emit_bins / emit_list  top-K first phase: append the pairs at or above E
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

__device__ __forceinline__ u32 smem_u32(const void* p) { return u32(__cvta_generic_to_shared(p)); }

// ---- partition passes: records -> fixed-capacity regions ----
// Every pass is one sweep over steps of kPartThreads x R records (R loads in
// flight per thread; bin_window and bin_split prefetch the next step by
// cp.async): a step is grouped by region in shared memory (an unstable local
// counting sort: order inside a region is immaterial), reserves its runs with
// one global atomic per non-empty region and writes every region's run
// contiguously, so the stores are whole sectors instead of one scattered
// 8-byte store per record (ncu: the scattered form was bound on L2 store
// transactions). A record whose region is full goes to the overflow list.
constexpr int kHiBits = 7;                  // x-side tiles per bucket: 128
constexpr u32 kMaxRegions = 256;            // regions per partition pass (shared counters)
constexpr int kPartThreads = 512, kPartPerThread = 8;
constexpr u32 kPartStep = kPartThreads * kPartPerThread;
constexpr u32 kMaxRunsPerBatch = 4096;      // a batch's run signs in shared memory

struct PartSmem {
    u64 buf[kPartStep];
    u32 lcnt[kMaxRegions], lstart[kMaxRegions], runo[kMaxRegions];
    u32 total;
};

// One step: rec[u] (valid when rg[u] < nreg) -> dst regions of `cap` records;
// the step reserves its runs in the global region counters gcnt (one atomic
// per non-empty region).
template <int THREADS, int R, class RegionOf>
__device__ __forceinline__ void scatter_step(PartSmem& sm, const u64 (&rec)[R], const u32 (&rg)[R], u32 nreg,
                                             RegionOf region_of, u64* __restrict__ dst, u64 stride, u32 cap,
                                             u64* __restrict__ ovf, u32 ovf_cap, u32* __restrict__ ovf_n,
                                             u32* __restrict__ gcnt) {
    u32 rk[R];
#pragma unroll
    for (int u = 0; u < R; ++u)
        if (rg[u] < nreg) rk[u] = atomicAdd(&sm.lcnt[rg[u]], 1u);
    __syncthreads();
    for (u32 g = threadIdx.x; g < nreg; g += THREADS) sm.runo[g] = sm.lcnt[g] ? atomicAdd(gcnt + g, sm.lcnt[g]) : 0u;
    if (threadIdx.x < 32) {  // exclusive scan of the step's region counts (<= 256, 8 per lane)
        const int lane = threadIdx.x;
        constexpr int PER = kMaxRegions / 32;
        u32 c[PER], tot = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const u32 g = lane * PER + q;
            c[q] = g < nreg ? sm.lcnt[g] : 0u;
            tot += c[q];
        }
        u32 incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        u32 ex = incl - tot;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const u32 g = lane * PER + q;
            if (g < nreg) sm.lstart[g] = ex;
            ex += c[q];
        }
        if (lane == 31) sm.total = incl;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < R; ++u)
        if (rg[u] < nreg) sm.buf[sm.lstart[rg[u]] + rk[u]] = rec[u];
    __syncthreads();
    const u32 total = sm.total;
    for (u32 e = threadIdx.x; e < total; e += THREADS) {
        const u64 r = sm.buf[e];
        const u32 g = region_of(r);
        const u32 pos = sm.runo[g] + (e - sm.lstart[g]);
        if (pos < cap) {
            dst[u64(g) * stride + pos] = r;
        } else {
            const u32 o = atomicAdd(ovf_n, 1u);
            if (o < ovf_cap) ovf[o] = r;
        }
    }
    __syncthreads();
    for (u32 g = threadIdx.x; g < nreg; g += THREADS) sm.lcnt[g] = 0;
    __syncthreads();
}

// Sweep 2's loads one step ahead: the next step's records travel (cp.async)
// into thread-private slots of dynamic shared memory (kPartStep x 8 B) while
// the current step is grouped and written; a thread reads back only what it
// fetched itself, so no barrier is involved.
__device__ __forceinline__ void step_fetch(u64* stage, const u64* __restrict__ src, u64 s0, u64 end) {
#pragma unroll
    for (int u = 0; u < kPartPerThread; ++u) {
        const u64 i = s0 + u64(u) * kPartThreads + threadIdx.x;
        if (i < end)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(stage + u * kPartThreads + threadIdx.x)),
                         "l"(src + i)
                         : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void step_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
inline size_t step_stage_smem() { return size_t(kPartStep) * 8; }

// Per batch: the batch's pair list -> z-side windows (region = kt). With a
// small fan-out (16 windows at config 4) one sweep suffices: each step of
// kPartStep records (held in registers) is counted per window in shared
// memory, reserved with one global atomic per window and written at base +
// shared rank (runs of ~256 records).
__global__ void __launch_bounds__(kPartThreads) bin_window(const PairRec* __restrict__ pairs,
                                                           const u32* __restrict__ npairs, u32 pair_cap,
                                                           const u32* __restrict__ nitems, u32 item_cap, u32 run0,
                                                           const int8_t* __restrict__ run_sign, u32 nruns,
                                                           const u64* __restrict__ tot, u64 guard,
                                                           int wshift, u32 nkt, u64* __restrict__ S, u32 cap_kt,
                                                           u32* __restrict__ wcnt, u64* __restrict__ ovf, u32 ovf_cap,
                                                           u32* __restrict__ ovf_n) {
    constexpr int R = kPartPerThread;
    __shared__ u32 cnt[kMaxRegions], base[kMaxRegions];
    __shared__ int8_t neg[kMaxRunsPerBatch];
    const u32 P = topk::batch_pairs(npairs, pair_cap, nitems, item_cap);
    for (u32 t = threadIdx.x; t < nkt; t += blockDim.x) cnt[t] = 0;
    // bit 0: the run's pass is negative; bit 1: the run is over the guard (a one-pass join emitted it anyway)
    for (u32 t = threadIdx.x; t < nruns; t += blockDim.x)
        neg[t] = int8_t((run_sign[t] < 0 ? 1 : 0) | (tot[t] > guard ? 2 : 0));
    __syncthreads();
    const uint4* P4 = reinterpret_cast<const uint4*>(pairs);
    // the next step's records travel (cp.async) into thread-private slots of shared memory while the
    // current step is counted, reserved and written: a thread reads back only what it fetched itself
    extern __shared__ __align__(16) uint4 stage[];  // [kPartStep]
    auto fetch = [&](u64 s0) {
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const u64 i = s0 + u64(u) * kPartThreads + threadIdx.x;
            if (i < P)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(stage + u * kPartThreads + threadIdx.x)),
                             "l"(P4 + i)
                             : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (u64(blockIdx.x) * kPartStep < P) fetch(u64(blockIdx.x) * kPartStep);
    for (u64 s0 = u64(blockIdx.x) * kPartStep; s0 < P; s0 += u64(gridDim.x) * kPartStep) {
        u64 rec[R];
        u32 kt[R], rk[R];
        asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const u64 i = s0 + u64(u) * kPartThreads + threadIdx.x;
            const uint4 pr = i < P ? stage[u * kPartThreads + threadIdx.x] : make_uint4(0, 0, 0, 0);
            rec[u] = rec_make(pr.x, pr.y, (pr.w >> 1) & 1u, neg[pr.z] & 1, run0 + pr.z);
            kt[u] = i < P && !(neg[pr.z] & 2) ? pr.y >> wshift : 0xffffffffu;
        }
        if (s0 + u64(gridDim.x) * kPartStep < P) fetch(s0 + u64(gridDim.x) * kPartStep);
#pragma unroll
        for (int u = 0; u < R; ++u)
            if (kt[u] != 0xffffffffu) rk[u] = atomicAdd(&cnt[kt[u]], 1u);
        __syncthreads();
        for (u32 t = threadIdx.x; t < nkt; t += blockDim.x) {
            base[t] = cnt[t] ? atomicAdd(wcnt + t, cnt[t]) : 0u;
            cnt[t] = 0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < R; ++u) {
            if (kt[u] == 0xffffffffu) continue;
            const u32 pos = base[kt[u]] + rk[u];
            if (pos < cap_kt) {
                S[u64(kt[u]) * cap_kt + pos] = rec[u];
            } else {
                const u32 o = atomicAdd(ovf_n, 1u);
                if (o < ovf_cap) ovf[o] = rec[u];
            }
        }
    }
}

// End of the search: each window -> buckets by x-side tile >> 7 (region =
// kt * nbh + hi). ctas_per_kt CTAs per window, one contiguous range each.
__global__ void __launch_bounds__(kPartThreads) bin_split(const u64* __restrict__ S, u32 cap_kt,
                                                          const u32* __restrict__ wcnt, u32 ctas_per_kt, u32 nbh,
                                                          u64* __restrict__ B, u32 cap_bucket,
                                                          u32* __restrict__ bcnt, u64* __restrict__ ovf, u32 ovf_cap,
                                                          u32* __restrict__ ovf_n) {
    constexpr int R = kPartPerThread;
    constexpr int SH = kBinJTShift + kHiBits;
    __shared__ PartSmem sm;
    const u32 kt = blockIdx.x / ctas_per_kt, part = blockIdx.x % ctas_per_kt;
    const u32 n = min(wcnt[kt], cap_kt);
    const u64 chunk = ceil_div(ceil_div(n, ctas_per_kt), kPartStep) * kPartStep;
    const u64 c0 = u64(part) * chunk, c1 = minu(n, c0 + chunk);
    if (c0 >= c1) return;
    const u64* src = S + u64(kt) * cap_kt;
    for (u32 t = threadIdx.x; t < nbh; t += blockDim.x) sm.lcnt[t] = 0;
    __syncthreads();
    // one sweep: every step of kPartStep records reserves its runs in the buckets itself
    auto region_of = [](u64 r) { return rec_a(r) >> SH; };
    u64* dst = B + u64(kt) * nbh * cap_bucket;
    extern __shared__ __align__(16) u64 stage8[];  // [kPartStep]
    step_fetch(stage8, src, c0, c1);
    for (u64 s0 = c0; s0 < c1; s0 += kPartStep) {
        u64 rec[R];
        u32 rg[R];
        step_wait();
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const u64 i = s0 + u64(u) * kPartThreads + threadIdx.x;
            rec[u] = i < c1 ? stage8[u * kPartThreads + threadIdx.x] : 0ull;
            rg[u] = i < c1 ? rec_a(rec[u]) >> SH : 0xffffffffu;
        }
        if (s0 + kPartStep < c1) step_fetch(stage8, src, s0 + kPartStep, c1);
        scatter_step<kPartThreads, R>(sm, rec, rg, nbh, region_of, dst, cap_bucket, cap_bucket, ovf, ovf_cap,
                                      ovf_n, bcnt + u64(kt) * nbh);
    }
}

// ---- end of the search: each bucket split by the low 7 bits of its x-side tile ----
// One CTA per bucket, one sweep: every tile owns a fixed region of
// cap_bucket / 128 records inside the bucket (bstart, relative to the window's
// first bucket); each step of kPartStep records is grouped by tile in shared
// memory, reserves its runs in the tiles' fill counters (bfill, zeroed by the
// host; one atomic per non-empty tile and step) and writes them contiguously.
// A record beyond its tile's region goes to the overflow list.
__global__ void __launch_bounds__(kPartThreads, 2) bin_sort(const u64* __restrict__ B, u32 cap_bucket,
                                                         const u32* __restrict__ bcnt, u32 nbh, u32 nbj,
                                                         u64* __restrict__ D, u32* __restrict__ bstart,
                                                         u32* __restrict__ bfill, u64* __restrict__ ovf, u32 ovf_cap,
                                                         u32* __restrict__ ovf_n) {
    constexpr u32 T = 1u << kHiBits;
    constexpr int R = kPartPerThread;
    __shared__ PartSmem sm;
    const u32 bk = blockIdx.x;
    const u32 kt = bk / nbh, hi = bk % nbh;
    const u32 cnt = min(bcnt[bk], cap_bucket);
    const u64* src = B + u64(bk) * cap_bucket;
    const u32 cap_tile = cap_bucket / T;
    if (threadIdx.x < T) {
        sm.lcnt[threadIdx.x] = 0;
        const u32 jt = hi * T + threadIdx.x;
        if (jt < nbj) bstart[u64(kt) * nbj + jt] = hi * cap_bucket + threadIdx.x * cap_tile;
    }
    __syncthreads();
    auto region_of = [](u64 r) { return (rec_a(r) >> kBinJTShift) & (T - 1); };
    u64* dst = D + u64(bk) * cap_bucket;
    u32* gfill = bfill + u64(kt) * nbj + u64(hi) * T;  // tiles past nbj hold no records: never touched
    extern __shared__ __align__(16) u64 stage8[];  // [kPartStep]: the next step's records (step_fetch)
    step_fetch(stage8, src, 0, cnt);
    for (u32 s0 = 0; s0 < cnt; s0 += kPartStep) {
        u64 rec[R];
        u32 rg[R];
        step_wait();
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const u32 i = s0 + u * kPartThreads + threadIdx.x;
            rec[u] = i < cnt ? stage8[u * kPartThreads + threadIdx.x] : 0ull;
            rg[u] = i < cnt ? (rec_a(rec[u]) >> kBinJTShift) & (T - 1) : 0xffffffffu;
        }
        if (s0 + kPartStep < cnt) step_fetch(stage8, src, s0 + kPartStep, cnt);
        scatter_step<kPartThreads, R>(sm, rec, rg, T, region_of, dst, cap_tile, cap_tile, ovf, ovf_cap, ovf_n, gfill);
    }
    // the counters ran past the regions of overflowing tiles: the fills the later passes read are clamped
    if (threadIdx.x < T && hi * T + threadIdx.x < nbj) atomicMin(&gfill[threadIdx.x], cap_tile);
}

// Each tile's records ordered by their x column (6 bits), in place: one CTA
// per tile, the records in registers, shared counts and ranks, written back
// through shared memory. A tile above kTileSortMax records stays unordered
// (the verify is exact either way; the order only lets consecutive pairs
// share the x column's shared-memory reads).
constexpr int kTileSortThreads = 256;
constexpr u32 kTileSortMax = 2048;
__global__ void __launch_bounds__(kTileSortThreads, 8) tile_sort(u64* __restrict__ D, u32 cap_bucket, u32 nbh, u32 nbj,
                                                              const u32* __restrict__ bstart,
                                                              const u32* __restrict__ bfill) {
    constexpr int R = kTileSortMax / kTileSortThreads;
    constexpr u32 C = 1u << kBinJTShift;
    __shared__ u64 buf[kTileSortMax];
    __shared__ u32 cnt[C], st[C];
    const u32 t = blockIdx.x;
    const u32 kt = t / nbj;
    const u32 fill = bfill[t];
    if (fill < 3 || fill > kTileSortMax) return;
    u64* rp = D + u64(kt) * nbh * cap_bucket + bstart[t];
    if (threadIdx.x < C) cnt[threadIdx.x] = 0;
    __syncthreads();
    u64 r[R];
    u32 rk[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
        const u32 i = u * kTileSortThreads + threadIdx.x;
        r[u] = i < fill ? rp[i] : 0ull;
        if (i < fill) rk[u] = atomicAdd(&cnt[rec_a(r[u]) & (C - 1)], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const u32 c0 = cnt[2 * lane], c1 = cnt[2 * lane + 1];
        u32 incl = c0 + c1;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        st[2 * lane] = incl - c0 - c1;
        st[2 * lane + 1] = incl - c1;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < R; ++u) {
        const u32 i = u * kTileSortThreads + threadIdx.x;
        if (i < fill) buf[st[rec_a(r[u]) & (C - 1)] + rk[u]] = r[u];
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < fill; i += kTileSortThreads) rp[i] = buf[i];
}

// One CTA per window: exclusive scan of the tiles' fills -> boff[kt][0..nbj]
// (compact rank indices; boff[kt][nbj] = the window's pairs held in buckets).
__global__ void __launch_bounds__(1024) bin_scan(const u32* __restrict__ fill, u32 nbj, u32* __restrict__ boff) {
    __shared__ u32 ws[33];
    const u32 kt = blockIdx.x;
    const u32* g = fill + u64(kt) * nbj;
    u32* bo = boff + u64(kt) * (nbj + 1);
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
        run += g[i];
    }
    if (threadIdx.x == 0) bo[nbj] = ws[32];
}

// ---- verify ----
struct BinVerifyArgs {
    const u64* Xc;
    u32 Wp;
    const u64* Yw;
    u32 n, astar;
    u64 p;
    const u64* F;       // the window's first bucket (sorted by tile)
    const u32* bstart;  // the window's tiles: first record, relative to F
    const u32* boff;    // the window's compact tile offsets [nbj + 1] (fill = boff[jt + 1] - boff[jt])
    u32 nbj;
    const u32* rid;          // global run ids by run index
    DevHit* hits;
    u32* hit_count;
    u32 hit_cap;
    const u32* krows;  // the runs' draws [R][M]: x-side keys of hits
    int kM;
    u32* sint_out;        // top-K first phase: rank of every pair of this window at its compact index (thr == 0)
    const u32* rank_thr;  // top-K running threshold (nullptr: hits mode)
    u32* rank_fail;       // top-K state's failure bits (topk::State::fail)
    u32 phase_follows;    // top-K: this window's ranks are consumed by a phase right after it (else bit 2 of
                          // *rank_fail is raised when the window still runs in the rank-writing first phase)
};

__device__ __forceinline__ u64 ld_stream(const u64* p, u64 pol) {
    u64 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ ulonglong2 ld_keep(const ulonglong2* p, u64 pol) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                 : "=l"(v.x), "=l"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// The x tiles come from X ^ Y (xor_response, once per search) by TMA bulk
// copies (cp.async.bulk, L2 evict_first) into a two-deep ring with mbarrier
// "full" phases, so there is no shared-memory XOR pass and no CTA barrier: a
// warp done with a tile moves on to the next one while slower warps finish
// (47.0 -> 41.0 ms at config 4 against a cp.async + __syncthreads form), and
// the last warp done with a buffer refills it. Teams of 16 lanes per pair,
// NS 16-byte slices per lane (W2 = Wp/2 <= 16 NS), two pairs in flight per
// team, the next records loaded one iteration ahead; the loops are
// warp-uniform (full-warp shuffles). Tiles are ordered by x column
// (tile_sort), so a team's second pair usually reuses the first's x slices.
__global__ void __launch_bounds__(256) xor_response(const ulonglong2* __restrict__ X, const ulonglong2* __restrict__ Y,
                                                    u32 W2, u64 total, ulonglong2* __restrict__ Xy) {
    for (u64 e = u64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += u64(gridDim.x) * blockDim.x) {
        const ulonglong2 x = __ldg(X + e), y = __ldg(Y + e % W2);
        Xy[e] = make_ulonglong2(x.x ^ y.x, x.y ^ y.y);
    }
}

template <int NS, bool FULL>
__global__ void __launch_bounds__(kVerifyThreads, 1) verify_binned(BinVerifyArgs A, const u64* __restrict__ Xy) {
    constexpr int G = 16, PR = 2, TPW = 32 / G, NWARPS = kVerifyThreads / 32;
    extern __shared__ __align__(128) ulonglong2 tiles[];  // [2][kBinJT][W2]
    __shared__ __align__(8) u64 full[2];
    __shared__ u32 done[2];
    const u32 W2 = A.Wp / 2;
    const u32 tile_elems = u32(kBinJT) * W2;
    const int lane = threadIdx.x & 31, tl = lane & (G - 1);
    const u32 warp = threadIdx.x >> 5, tw = (threadIdx.x / G) % TPW;
    const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(A.Xc);
    const ulonglong2* XY2 = reinterpret_cast<const ulonglong2*>(Xy);
    u64 pol = 0, tpol = 0;  // the window stays (evict_last), the tiles stream through (evict_first)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(tpol));
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    const bool ranks = A.sint_out != nullptr && rthr == 0;
    const u32 astar = max(A.astar, rthr);
    if (ranks && !A.phase_follows && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(A.rank_fail, 4u);
    if (threadIdx.x == 0) {
        for (int bb = 0; bb < 2; ++bb) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[bb])));
            done[bb] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const u32 nmine = blockIdx.x < A.nbj ? (A.nbj - 1 - blockIdx.x) / gridDim.x + 1 : 0u;
    auto issue = [&](u32 i) {  // one thread: the tile of this CTA's i-th bin into buffer i & 1
        const u32 jt = blockIdx.x + i * gridDim.x;
        const int bb = i & 1;
        const u32 c0 = jt << kBinJTShift;
        const u32 ncol = u32(minu(A.p - c0, kBinJT));
        const u32 bytes = A.boff[jt + 1] > A.boff[jt] ? ncol * W2 * 16 : 0u;
        const u32 bar = smem_u32(&full[bb]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        if (bytes)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                "[%3], %4;" ::"r"(smem_u32(tiles + bb * tile_elems)),
                "l"(XY2 + u64(c0) * W2), "r"(bytes), "r"(bar), "l"(tpol)
                : "memory");
    };
    if (threadIdx.x == 0) {
        if (nmine > 0) issue(0);
        if (nmine > 1) issue(1);
    }
    for (u32 i = 0; i < nmine; ++i) {
        const u32 jt = blockIdx.x + i * gridDim.x;
        const int bb = i & 1;
        const u32 rbase = A.boff[jt], r1 = A.boff[jt + 1] - rbase;  // the bin's fill
        const u64* Fb = A.F + A.bstart[jt];
        {
            u32 ok = 0;
            while (!ok)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(ok) : "r"(smem_u32(&full[bb])), "r"((i >> 1) & 1u) : "memory");
        }
        const ulonglong2* tile = tiles + bb * tile_elems;
        const u32 c0 = jt << kBinJTShift;
        constexpr u32 STRIDE = NWARPS * TPW * PR;
        u64 nrec[PR];
#pragma unroll
        for (int r = 0; r < PR; ++r) {
            const u32 q = warp * TPW * PR + tw * PR + r;
            nrec[r] = q < r1 ? ld_stream(Fb + q, tpol) : 0ull;
        }
        for (u32 q0 = warp * TPW * PR; q0 < r1; q0 += STRIDE) {  // warp-uniform
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
                nrec[r] = q < r1 ? ld_stream(Fb + q, tpol) : 0ull;
            }
            u32 jl[PR], acc[PR];
#pragma unroll
            for (int r = 0; r < PR; ++r) {
                jl[r] = qb + r < r1 ? rec_a(rec[r]) - c0 : 0u;
                acc[r] = 0;
            }
#pragma unroll
            for (int it = 0; it < NS; ++it) {
                if (FULL || it * G + tl < W2) {
                    ulonglong2 av = tile[jl[0] * W2 + it * G + tl];
                    acc[0] += __popcll(av.x ^ kv[0][it].x) + __popcll(av.y ^ kv[0][it].y);
#pragma unroll
                    for (int r = 1; r < PR; ++r) {
                        if (jl[r] != jl[r - 1]) av = tile[jl[r] * W2 + it * G + tl];
                        acc[r] += __popcll(av.x ^ kv[r][it].x) + __popcll(av.y ^ kv[r][it].y);
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < PR; ++r) {
                const u32 q = qb + r;
                u32 a = acc[r];
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (tl == 0 && q < r1) {
                    const u32 si = rec_neg(rec[r]) ? A.n - a : a;
                    if (ranks) {
                        A.sint_out[rbase + q] = si;
                    } else if (si >= astar) {
                        PairRec pr{rec_a(rec[r]), rec_b(rec[r]), rec_run(rec[r]), rec_diag(rec[r]) << 1};
                        kern::append_pair_hit(nullptr, 0, 0, A.rid, A.hits, A.hit_count, A.hit_cap, pr, si, A.n,
                                              A.krows, A.kM, A.Xc, A.Wp);
                    }
                }
            }
        }
        // this warp is done with buffer bb: the last warp refills it with the tile of bin i + 2
        __syncwarp();
        if (lane == 0) {
            const u32 d = atomicAdd(&done[bb], 1u);
            if (d == NWARPS - 1) {
                done[bb] = 0;
                if (i + 2 < nmine) issue(i + 2);
            }
        }
    }
}

__device__ __forceinline__ void emit_rec(u64 rc, u32 r, const u32* __restrict__ rid, const u32* __restrict__ krows,
                                         int kM, const u64* __restrict__ Xc, u32 Wp, DevHit* __restrict__ hits,
                                         u32 slot, u32 n) {
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

// Top-K first phase over a window: append its pairs with rank >= E (as
// topk::emit_pairs); warp per bin, warp-aggregated slots.
__global__ void __launch_bounds__(256) emit_bins(const u64* __restrict__ F, const u32* __restrict__ bstart,
                                                 const u32* __restrict__ boff,
                                                 u32 nbj, const u32* __restrict__ sint,
                                                 const topk::State* __restrict__ st, const u32* __restrict__ rid,
                                                 const u32* __restrict__ krows, int kM, const u64* __restrict__ Xc,
                                                 u32 Wp, DevHit* __restrict__ hits, u32* __restrict__ hit_count,
                                                 u32 hit_cap, u32 n) {
    if (st->thr > 0) return;
    const u32 E = st->emit;
    const int lane = threadIdx.x & 31;
    const u32 gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (u32 jt = gw; jt < nbj; jt += nw) {
        const u32 b0 = boff[jt], fill = boff[jt + 1] - b0;
        for (u32 i0 = 0; i0 < fill; i0 += 32) {
            const u32 i = i0 + lane;
            const u32 r = i < fill ? sint[b0 + i] : 0u;
            const bool take = i < fill && r >= E;
            const u32 bal = __ballot_sync(0xffffffffu, take);
            if (!bal) continue;
            u32 base = 0;
            if (lane == __ffs(bal) - 1) base = atomicAdd(hit_count, __popc(bal));
            base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
            const u32 slot = base + __popc(bal & lanemask_lt());
            if (take && slot < hit_cap) emit_rec(F[bstart[jt] + i], r, rid, krows, kM, Xc, Wp, hits, slot, n);
        }
    }
}

// The overflow list: warp per pair, both columns gathered (lane w: slices w, w + 32, w + 64).
__global__ void __launch_bounds__(256) verify_list(BinVerifyArgs A, const u64* __restrict__ list,
                                                   const u32* __restrict__ count, u32 cap) {
    const int lane = threadIdx.x & 31;
    const u32 W2 = A.Wp / 2;
    const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(A.Xc);
    const ulonglong2* Y2 = reinterpret_cast<const ulonglong2*>(A.Yw);
    const u32 P = min(*count, cap);
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    const bool ranks = A.sint_out != nullptr && rthr == 0;
    const u32 astar = max(A.astar, rthr);
    const u32 gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (u32 q = gw; q < P; q += nw) {
        const u64 rc = list[q];
        const ulonglong2* a = X2 + u64(rec_a(rc)) * W2;
        const ulonglong2* b = X2 + u64(rec_b(rc)) * W2;
        u32 acc = 0;
        for (u32 w = lane; w < W2; w += 32) {
            const ulonglong2 x = __ldg(a + w), z = __ldg(b + w), y = __ldg(Y2 + w);
            acc += __popcll(x.x ^ z.x ^ y.x) + __popcll(x.y ^ z.y ^ y.y);
        }
        acc = warp_sum(acc);
        if (lane == 0) {
            const u32 si = rec_neg(rc) ? A.n - acc : acc;
            if (ranks) {
                A.sint_out[q] = si;
            } else if (si >= astar) {
                PairRec pr{rec_a(rc), rec_b(rc), rec_run(rc), rec_diag(rc) << 1};
                kern::append_pair_hit(nullptr, 0, 0, A.rid, A.hits, A.hit_count, A.hit_cap, pr, si, A.n, A.krows,
                                      A.kM, A.Xc, A.Wp);
            }
        }
    }
}

__global__ void __launch_bounds__(256) emit_list(const u64* __restrict__ list, const u32* __restrict__ sint,
                                                 const u32* __restrict__ count, u32 cap,
                                                 const topk::State* __restrict__ st, const u32* __restrict__ rid,
                                                 const u32* __restrict__ krows, int kM, const u64* __restrict__ Xc,
                                                 u32 Wp, DevHit* __restrict__ hits, u32* __restrict__ hit_count,
                                                 u32 hit_cap, u32 n) {
    if (st->thr > 0) return;
    const u32 P = min(*count, cap);
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
        const u32 slot = base + __popc(bal & lanemask_lt());
        if (take && slot < hit_cap) emit_rec(list[i], r, rid, krows, kM, Xc, Wp, hits, slot, n);
    }
}

inline size_t bin_window_smem() { return size_t(kPartStep) * 16; }
inline size_t verify_smem(u32 Wp) { return size_t(2) * kBinJT * (Wp / 2) * 16; }

} // namespace bins
} // namespace xyzb
