// Fused per-run grouping + join on a thread-block cluster (sm_100a, DSMEM).
//
// For M <= 17 the 2^M bucket table of one run fits in the distributed shared
// memory of a cluster (CL CTAs x 2^M/CL u32 counters, 64 KB per CTA). One
// cluster per run then does, without touching global memory except to read
// the keys and write the grouped column indices and the candidate list:
//   1. count: warp-aggregated atomics into the owning CTA's table (DSMEM);
//   2. scan: per-CTA exclusive scan + cross-CTA base through DSMEM;
//   3. scatter: atomic cursors (DSMEM) -> grouped[b*p + pos] = column;
//   4. join: per key v, its group [begin, end) and the partner group of
//      v ^ c are read straight from the tables; |E_r| (incl. the diagonal)
//      and the canonical work are reduced across the cluster, so the guard
//      (pair_search.hpp:91-94) is decided on-chip;
//   5. emit: candidate pairs / work items of the kept runs (emit_items).
// It replaces bucket_count + scan + bucket_scatter + bucket_join_count +
// bucket_join_emit (five launches and four global passes over 2^M tables).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "search_kernels.cuh"

namespace xyzb {
namespace kern {

constexpr int kCgThreads = 1024;
constexpr u32 kCgPerCta = 16384;  // table entries per CTA (64 KB)

template <class K>
__global__ void __launch_bounds__(kCgThreads) cluster_group_join(
    const K* __restrict__ keys, u64 p, int M, const K* __restrict__ xorc, u64 guard, u32 hmax,
    u32* __restrict__ grouped, u64* __restrict__ tot, u64* __restrict__ work_run, Item* __restrict__ items,
    u32* __restrict__ nitems, u32 item_cap, u32* __restrict__ npairs, PairRec* __restrict__ pairs, u32 pair_cap) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) u32 tab[];
    __shared__ u32 warp_tot[33];
    __shared__ u32 s_total;
    __shared__ u64 s_red[2][32];
    __shared__ u64 s_pairs, s_work;
    const u32 CL = cl.num_blocks(), cr = cl.block_rank();
    const u32 per = u32((u64(1) << M) / CL);  // power of two
    const int lshift = __ffs(per) - 1;
    const u64 b = blockIdx.y;
    const K* kb = keys + b * p;
    const u64 s0 = p * cr / CL, s1 = p * (cr + 1) / CL;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const K c = xorc[b];

    for (u32 i = threadIdx.x; i < per; i += kCgThreads) tab[i] = 0;
    cl.sync();
    // 1. count
    for (u64 i0 = s0; i0 < s1; i0 += kCgThreads) {
        const u64 i = i0 + threadIdx.x;
        const bool valid = i < s1;
        const u32 active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const u32 v = u32(kb[i]);
            const u32 peers = __match_any_sync(active, v);
            if ((peers & lanemask_lt()) == 0)
                atomicAdd(cl.map_shared_rank(tab, v >> lshift) + (v & (per - 1)), __popc(peers));
        }
    }
    cl.sync();
    // 2. exclusive scan (run-local positions)
    {
        const u32 chunk = (per + kCgThreads - 1) / kCgThreads;
        const u32 a0 = min(per, threadIdx.x * chunk), a1 = min(per, a0 + chunk);
        u32 loc = 0;
        for (u32 i = a0; i < a1; ++i) loc += tab[i];
        u32 incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const u32 x = warp_tot[lane];
            u32 xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += t;
            }
            warp_tot[lane] = xi - x;
            if (lane == 31) s_total = xi;
        }
        cl.sync();  // s_total of every CTA visible
        u32 base = 0;
        for (u32 q = 0; q < cr; ++q) base += *cl.map_shared_rank(&s_total, q);
        u32 run = base + warp_tot[wid] + incl - loc;
        for (u32 i = a0; i < a1; ++i) {
            const u32 t = tab[i];
            tab[i] = run;
            run += t;
        }
    }
    cl.sync();
    // 3. scatter (non-stable inside a bucket: hits recover (key, j, k) order)
    for (u64 i0 = s0; i0 < s1; i0 += kCgThreads) {
        const u64 i = i0 + threadIdx.x;
        const bool valid = i < s1;
        const u32 active = __ballot_sync(0xffffffffu, valid);
        if (valid) {
            const u32 v = u32(kb[i]);
            const u32 peers = __match_any_sync(active, v);
            const int leader = __ffs(peers) - 1;
            u32 pos = 0;
            if (lane == leader) pos = atomicAdd(cl.map_shared_rank(tab, v >> lshift) + (v & (per - 1)), __popc(peers));
            pos = __shfl_sync(peers, pos, leader) + __popc(peers & lanemask_lt());
            grouped[b * p + pos] = u32(i);
        }
    }
    cl.sync();  // tab now holds each bucket's end
    auto group = [&](u32 v, u32& beg, u32& cnt) {
        const u32 own = v >> lshift, loc = v & (per - 1);
        const u32 end = cl.map_shared_rank(tab, own)[loc];
        u32 start;
        if (loc > 0) start = cl.map_shared_rank(tab, own)[loc - 1];
        else start = own > 0 ? cl.map_shared_rank(tab, own - 1)[per - 1] : 0u;
        beg = start;
        cnt = end - start;
    };
    auto block_of = [&](u32 v) {
        HeadBlock hb;
        u32 bx, cx;
        group(v, bx, cx);
        if (cx == 0) return hb;
        const u32 v2 = v ^ u32(c);
        if (v2 == v) {
            hb.pairs = u64(cx) * cx;  // the diagonal j == k counts (pair_search.cpp:48-49)
            if (cx >= 2) {
                hb.work = u64(cx) * (cx - 1) / 2;
                hb.hs = bx;
                hb.hc = cx;
                hb.ss = bx;
                hb.sc = cx;
                hb.flags = 3u;
            }
        } else if (v2 > v) {
            u32 bz, cz;
            group(v2, bz, cz);
            if (cz) {
                hb.pairs = 2ull * cx * cz;
                hb.work = u64(cx) * cz;
                if (cx <= cz) {
                    hb.hs = bx; hb.hc = cx; hb.ss = bz; hb.sc = cz; hb.flags = 1u;
                } else {
                    hb.hs = bz; hb.hc = cz; hb.ss = bx; hb.sc = cx; hb.flags = 0u;
                }
            }
        }
        return hb;
    };
    // 4. |E_r| and canonical work across the cluster
    u64 pairs_acc = 0, work_acc = 0;
    for (u32 l = threadIdx.x; l < per; l += kCgThreads) {
        const HeadBlock hb = block_of(cr * per + l);
        pairs_acc += hb.pairs;
        work_acc += hb.work;
    }
    pairs_acc = warp_sum(pairs_acc);
    work_acc = warp_sum(work_acc);
    if (lane == 0) {
        s_red[0][wid] = pairs_acc;
        s_red[1][wid] = work_acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 a = 0, w = 0;
        for (int q = 0; q < kCgThreads / 32; ++q) {
            a += s_red[0][q];
            w += s_red[1][q];
        }
        s_pairs = a;
        s_work = w;
    }
    cl.sync();
    u64 run_pairs = 0, run_work = 0;
    for (u32 q = 0; q < CL; ++q) {
        run_pairs += *cl.map_shared_rank(&s_pairs, q);
        run_work += *cl.map_shared_rank(&s_work, q);
    }
    if (cr == 0 && threadIdx.x == 0) {
        tot[b] = run_pairs;
        work_run[b] = run_work;
    }
    // 5. emit candidates of a run the guard keeps
    if (run_pairs <= guard) {
        for (u32 l0 = 0; l0 < per; l0 += kCgThreads) {
            const u32 l = l0 + threadIdx.x;
            HeadBlock hb;
            if (l < per) hb = block_of(cr * per + l);
            emit_items(hb, u32(b), hmax, items, nitems, item_cap, npairs, pairs, pair_cap, p, grouped);
        }
    }
    cl.sync();  // peers may still read this CTA's table
}

// Launch one cluster per run; returns false if the table does not fit (M too
// large for kCgPerCta entries x 8 CTAs).
template <class K>
bool cluster_group_join_launch(const K* keys, u64 B, u64 p, int M, const K* xorc, u64 guard, u32 hmax, u32* grouped,
                               u64* tot, u64* work_run, Item* items, u32* nitems, u32 item_cap, u32* npairs,
                               PairRec* pairs, u32 pair_cap, cudaStream_t st) {
    const u64 T = u64(1) << M;
    u64 cl = 1;
    while (T / cl > kCgPerCta) cl <<= 1;
    if (cl > 8) return false;
    const size_t smem = size_t(T / cl) * 4;
    func_smem(cluster_group_join<K>, kCgPerCta * 4);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<u32>(cl), static_cast<u32>(B), 1);
    cfg.blockDim = dim3(kCgThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = static_cast<u32>(cl);
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    XYZB_CUDA(cudaLaunchKernelEx(&cfg, cluster_group_join<K>, keys, p, M, xorc, guard, hmax, grouped, tot, work_run,
                                 items, nitems, item_cap, npairs, pairs, pair_cap));
    return true;
}

} // namespace kern
} // namespace xyzb
