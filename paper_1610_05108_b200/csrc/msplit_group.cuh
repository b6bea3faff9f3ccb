// Per-run grouping + join on a cluster of 2^s CTAs, for 17 <= M <= 20
// (configs 3 and 4), generalising split_group_join (cta_group.cuh).
//
// The 2^M buckets of a run are split over CS = 2^s CTAs (s = M - 16, one
// 2^16-bucket 16-bit table per CTA, 128 KB; 16 CTAs at M = 20 with the
// non-portable cluster size). CTA r owns the keys v with owner(v) = r, where
// owner bit i = parity(v & S_i) for s disjoint bit sets S_i. The S_i are
// built per run from the zero bits of c = x-key ^ z-key (round robin), so a
// key and its partner v ^ c agree on every S_i and live in the same CTA;
// parities of several biased bits balance the CTAs. When c has fewer than s
// zero bits the remaining S_i are single bits where c is 1: the partner then
// lives in CTA r ^ owner(c) and the join reads its table through DSMEM.
// Each S_i has a pivot bit (its lowest) that the local index drops; the
// pivot is recovered from r and the parity of the rest of S_i.
// Per run: count (every CTA streams all keys, keeps its own), scan, an
// all-to-all exchange of the CTA key counts (positions: CTA r's follow the
// counts of CTAs < r), scatter, join pass 1 (|E_r| share, work, emit counts),
// cluster reduction of |E_r| (the guard), emission. Overflow of the 16-bit
// counters (p > 65535 only) redoes the run exactly on CTA 0 with 32-bit
// counters in a global scratch slot.
#pragma once

#include <cooperative_groups.h>

#include "cta_group.cuh"

namespace xyzb {
namespace kern {

constexpr int kMsThreads = 1024;
constexpr int kMsMaxS = 4;
constexpr u32 kMsSlots = 16;  // global fallback tables (2^M u32 each)

struct MSplit {
    int s = 0;
    u32 set[kMsMaxS];      // S_i
    int piv[kMsMaxS];      // pivot bit of S_i
    int sorted[kMsMaxS];   // pivots ascending
    u32 oc = 0;            // owner(c): the partner's CTA is r ^ oc

    __device__ void build(u32 c, int M, int s_) {
        s = s_;
        const u32 mask = M >= 32 ? ~0u : ((1u << M) - 1u);
        const u32 Z = ~c & mask;
        const int nz = __popc(Z);
        for (int i = 0; i < kMsMaxS; ++i) {
            set[i] = 0;
            piv[i] = -1;
        }
        // zero bits round robin over the sets (the lowest one of each set is its pivot)
        int idx = 0;
        for (int b = 0; b < M; ++b)
            if ((Z >> b) & 1u) {
                const int i = idx % s;
                if (piv[i] < 0) piv[i] = b;
                set[i] |= 1u << b;
                ++idx;
            }
        // fewer zero bits than sets: single bits where c is 1, from the top
        int b = M - 1;
        for (int i = nz; i < s; ++i) {
            while ((Z >> b) & 1u) --b;
            piv[i] = b;
            set[i] = 1u << b;
            --b;
        }
        for (int i = 0; i < s; ++i) sorted[i] = piv[i];
        for (int i = 1; i < s; ++i)  // insertion sort, s <= 4
            for (int j = i; j > 0 && sorted[j - 1] > sorted[j]; --j) {
                const int t = sorted[j];
                sorted[j] = sorted[j - 1];
                sorted[j - 1] = t;
            }
        oc = owner(c);
    }
    __device__ __forceinline__ u32 owner(u32 v) const {
        u32 o = 0;
#pragma unroll
        for (int i = 0; i < kMsMaxS; ++i)
            if (i < s) o |= (u32(__popc(v & set[i])) & 1u) << i;
        return o;
    }
    __device__ __forceinline__ u32 local(u32 v) const {  // drop the pivots (highest first)
#pragma unroll
        for (int i = kMsMaxS - 1; i >= 0; --i)
            if (i < s) {
                const int t = sorted[i];
                v = ((v >> (t + 1)) << t) | (v & ((1u << t) - 1u));
            }
        return v;
    }
    __device__ __forceinline__ u32 key(u32 li, u32 r) const {  // inverse of local for owner r
        u32 u = li;
#pragma unroll
        for (int i = 0; i < kMsMaxS; ++i)
            if (i < s) {
                const int t = sorted[i];
                u = ((u >> t) << (t + 1)) | (u & ((1u << t) - 1u));
            }
#pragma unroll
        for (int i = 0; i < kMsMaxS; ++i)
            if (i < s) u |= (((r >> i) & 1u) ^ (u32(__popc(u & set[i])) & 1u)) << piv[i];
        return u;
    }
};

template <bool CHECK, bool SCATTER>
__device__ __forceinline__ void msplit_pass(SmemTab16& tab, const u32* __restrict__ kb, u32 p, const MSplit& ms,
                                            u32 r, u32 base, u32* __restrict__ out) {
    auto one = [&](u32 v, u32 i, bool valid) {
        if (valid && ms.owner(v) == r) {
            const u32 li = ms.local(v);
            const u32 pos = tab.template add<CHECK>(li, 1u);
            if (SCATTER) out[base + tab.chunk_base(li) + pos] = i;
        }
    };
    const u32 mis = u32(reinterpret_cast<uintptr_t>(kb) >> 2) & 3u;
    const u32 head = min(p, (4u - mis) & 3u);
    const u32 n4 = (p - head) >> 2;
    const u32 tail0 = head + 4 * n4;
    if (threadIdx.x < head) one(kb[threadIdx.x], threadIdx.x, true);
    if (tail0 + threadIdx.x < p && threadIdx.x < 4) one(kb[tail0 + threadIdx.x], tail0 + threadIdx.x, true);
    const uint4* k4 = reinterpret_cast<const uint4*>(kb + head);
    for (u32 q0 = 0; q0 < n4; q0 += 2 * blockDim.x) {
        const u32 qa = q0 + threadIdx.x, qb = qa + blockDim.x;
        const bool va = qa < n4, vb = qb < n4;
        const uint4 a = va ? __ldg(k4 + qa) : make_uint4(0, 0, 0, 0);
        const uint4 b = vb ? __ldg(k4 + qb) : make_uint4(0, 0, 0, 0);
        const u32 ia = head + 4 * qa, ib = head + 4 * qb;
        one(a.x, ia, va);
        one(a.y, ia + 1, va);
        one(a.z, ia + 2, va);
        one(a.w, ia + 3, va);
        one(b.x, ib, vb);
        one(b.y, ib + 1, vb);
        one(b.z, ib + 2, vb);
        one(b.w, ib + 3, vb);
    }
}

template <bool CHECK>
__global__ void __launch_bounds__(kMsThreads, 1) msplit_group_join(
    const u32* __restrict__ keys, u64 p, int M, int s, const u32* __restrict__ xorc, u64 guard, u32 hmax,
    u32* __restrict__ grouped, u64* __restrict__ tot, u64* __restrict__ work_run, Item* __restrict__ items,
    u32* __restrict__ nitems, u32 item_cap, u32* __restrict__ npairs, PairRec* __restrict__ pairs, u32 pair_cap,
    u32* __restrict__ gtab, u32* __restrict__ slots) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) u32 smem[];
    __shared__ u32 ws[68];
    __shared__ u32 s_ovf, s_n, s_slot;
    __shared__ u32 s_base[1 << kMsMaxS];
    __shared__ u64 red[2][33];
    __shared__ u64 s_part[2];
    const u32 r = cl.block_rank(), CS = cl.num_blocks();
    const u32 b = blockIdx.y;
    const u32* kb = keys + u64(b) * p;
    u32* out = grouped + u64(b) * p;
    const int Ml = M - s;
    const u32 Tl = u32(1) << Ml;
    const int cbits = min(Ml, kCtChunkBits);
    const u32 nbase = max(1u, Tl >> cbits);
    SmemTab16 tab{smem + nbase, smem, Ml, cbits, &s_ovf};
    const u32 mask = (u32(1) << M) - 1;
    const u32 c = xorc[b] & mask;
    MSplit ms;
    ms.build(c, M, s);

    if (threadIdx.x == 0) s_ovf = 0;
    tab.clear();
    __syncthreads();
    msplit_pass<CHECK, false>(tab, kb, u32(p), ms, r, 0u, static_cast<u32*>(nullptr));
    __syncthreads();
    const u32 n_mine = tab.scan(ws);
    if (threadIdx.x == 0) s_n = n_mine;
    __syncthreads();
    cl.sync();  // #1: every CTA's count and overflow flag
    bool ovf = false;
    if (threadIdx.x == 0) {
        u32 acc = 0;
        for (u32 q = 0; q < CS; ++q) {
            s_base[q] = acc;
            acc += *cl.map_shared_rank(&s_n, q);
        }
    }
    if (CHECK)
        for (u32 q = 0; q < CS; ++q) ovf |= *cl.map_shared_rank(&s_ovf, q) != 0;
    __syncthreads();
    if (ovf) {
        if (r == 0) {
            if (threadIdx.x == 0) {
                u32 sl = b % kMsSlots;
                while (atomicCAS(slots + sl, 0u, 1u) != 0u) sl = (sl + 1) % kMsSlots;
                s_slot = sl;
            }
            __syncthreads();
            GlobalTab32 g{gtab + (u64(s_slot) << M), M};
            g.clear();
            __syncthreads();
            tab_pass<false, false, false>(g, kb, p, static_cast<u32*>(nullptr));
            __syncthreads();
            g.scan(ws);
            __syncthreads();
            tab_pass<false, false, false>(g, kb, p, out);
            __syncthreads();
            tab_join<u32>(g, M, b, c, p, guard, hmax, tot, work_run, items, nitems, item_cap, npairs, pairs, pair_cap,
                          red, ws, grouped);
            __threadfence();
            if (threadIdx.x == 0) atomicExch(slots + s_slot, 0u);
        }
        cl.sync();
        return;
    }
    msplit_pass<false, true>(tab, kb, u32(p), ms, r, s_base[r], out);
    __syncthreads();
    if (ms.oc) cl.sync();  // #2: partner tables final before remote reads
    auto group = [&](u32 v, u32& beg, u32& cnt) {
        const u32 o = ms.owner(v);
        const u32 li = ms.local(v);
        if (o == r) {
            tab.group(li, beg, cnt);
        } else {
            SmemTab16 rt = tab;
            rt.w = cl.map_shared_rank(tab.w, o);
            rt.base = cl.map_shared_rank(tab.base, o);
            rt.group(li, beg, cnt);
        }
        beg += s_base[o];
    };
    auto block_of = [&](u32 li) {
        HeadBlock hb;
        const u32 v = ms.key(li, r);
        u32 bx, cx;
        group(v, bx, cx);
        if (cx == 0) return hb;
        const u32 v2 = v ^ c;
        if (v2 == v) {
            hb.pairs = u64(cx) * cx;  // the diagonal j == k counts (pair_search.cpp:48-49)
            if (cx >= 2) {
                hb.work = u64(cx) * (cx - 1) / 2;
                hb.hs = bx; hb.hc = cx; hb.ss = bx; hb.sc = cx; hb.flags = 3u;
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
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool pair_list = npairs != nullptr;
    u64 pa = 0, wa = 0;
    u32 my_items = 0, my_pairs = 0;
    for (u32 li = threadIdx.x; li < Tl; li += blockDim.x) {
        const HeadBlock hb = block_of(li);
        pa += hb.pairs;
        wa += hb.work;
        u32 ne, np, nsc;
        emit_count(hb, hmax, pair_list, ne, np, nsc);
        my_items += ne;
        my_pairs += np;
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
        s_part[0] = a;
        s_part[1] = w;
    }
    cl.sync();  // #3: every CTA's share of |E_r|
    u64 run_pairs = 0, run_work = 0;
    for (u32 q = 0; q < CS; ++q) {
        const u64* op = cl.map_shared_rank(s_part, q);
        run_pairs += op[0];
        run_work += op[1];
    }
    if (r == 0 && threadIdx.x == 0) {
        tot[b] = run_pairs;
        work_run[b] = run_work;
    }
    if (run_pairs <= guard) {
        u32 ti, tp;
        u32 ibase = block_exclusive(my_items, ws, &ti);
        u32 pbase = block_exclusive(my_pairs, ws + 33, &tp);
        if (threadIdx.x == 0) {
            ws[66] = ti ? atomicAdd(nitems, ti) : 0u;
            ws[67] = (pair_list && tp) ? atomicAdd(npairs, tp) : 0u;
        }
        __syncthreads();
        ibase += ws[66];
        pbase += ws[67];
        for (u32 li = threadIdx.x; li < Tl; li += blockDim.x) {
            const HeadBlock hb = block_of(li);
            if (hb.work == 0) continue;
            u32 ne, np, nsc;
            emit_count(hb, hmax, pair_list, ne, np, nsc);
            emit_write(hb, b, hmax, pair_list, ne, nsc, ibase, pbase, items, item_cap, pairs, pair_cap, p, grouped);
            ibase += ne;
            pbase += np;
        }
    }
    cl.sync();  // #4: peers may still read this CTA's table and shares
}

inline size_t msplit_group_smem(int Ml) {
    const u64 Tl = u64(1) << Ml;
    const int cbits = Ml < kCtChunkBits ? Ml : kCtChunkBits;
    return size_t(Tl / 2) * 4 + size_t(std::max<u64>(1, Tl >> cbits)) * 4;
}

// Scratch (u32 entries) of the overflow fallback.
inline u64 msplit_group_scratch(int M, u64 p) { return p > 0xffffu ? (u64(kMsSlots) << M) : 0; }

// Whether a 2^(M-16)-CTA cluster of this kernel fits on the GPU.
inline bool msplit_schedulable(int M) {
    const int s = M - 16;
    if (s < 1 || s > kMsMaxS) return false;
    // per (device, s), under a lock (datasets on several devices / host threads)
    static std::mutex mu;
    static std::map<std::pair<int, int>, bool> cached;
    int dev = 0;
    XYZB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(dev, s);
    if (!cached.count(key)) {
        auto kernel = msplit_group_join<false>;
        func_smem(kernel, msplit_group_smem(16));
        func_attr(reinterpret_cast<const void*>(kernel), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1u << s, 1, 1);
        cfg.blockDim = dim3(kMsThreads, 1, 1);
        cfg.dynamicSmemBytes = msplit_group_smem(16);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1u << s;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        const bool ok = cudaOccupancyMaxActiveClusters(&ncl, kernel, &cfg) == cudaSuccess && ncl >= 1;
        cudaGetLastError();
        cached[key] = ok;
    }
    return cached[key];
}

// Launch one 2^s-CTA cluster per run (s = M - 16); false when the cluster
// cannot be scheduled on this GPU (the caller keeps another grouping path).
inline bool msplit_group_join_launch(const u32* keys, u64 B, u64 p, int M, const u32* xorc, u64 guard, u32 hmax,
                                     u32* grouped, u64* tot, u64* work_run, Item* items, u32* nitems, u32 item_cap,
                                     u32* npairs, PairRec* pairs, u32 pair_cap, u32* gtab, u32* slots,
                                     cudaStream_t st) {
    const int s = M - 16;
    if (s < 1 || s > kMsMaxS) return false;
    const u32 CS = 1u << s;
    const size_t smem = msplit_group_smem(M - s);
    const bool check = p > 0xffffu;
    auto kernel = check ? msplit_group_join<true> : msplit_group_join<false>;
    func_smem(kernel, msplit_group_smem(16));
    func_attr(reinterpret_cast<const void*>(kernel), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, static_cast<u32>(B), 1);
    cfg.blockDim = dim3(kMsThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kernel, &cfg) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        return false;
    }
    XYZB_CUDA(cudaLaunchKernelEx(&cfg, kernel, keys, p, M, s, xorc, guard, hmax, grouped, tot, work_run, items,
                                 nitems, item_cap, npairs, pairs, pair_cap, gtab, slots));
    return true;
}

} // namespace kern
} // namespace xyzb
