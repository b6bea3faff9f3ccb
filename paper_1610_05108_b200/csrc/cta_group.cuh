// Per-run grouping + join with 16-bit bucket tables in shared memory (sm_100a).
//
// For M <= 16 the 2^M bucket counters of one run fit in shared memory as
// 16-bit halves of u32 words. Positions above 16 bits come from per-chunk
// u32 bases (a chunk = 256 buckets): start(v) = base[v >> 8] + off16[v].
// Per run, all on chip (split_group_join below, two CTAs of a cluster; the
// table helpers are shared with msplit_group.cuh):
//   1. count: one shared atomic per key (warp-aggregated with match.any only
//      when 2^M is small enough for lanes to collide);
//   2. scan: per-thread bucket ranges, block scan, chunk bases;
//   3. scatter: atomic cursors -> grouped[b*p + pos] = column;
//   4. join: |E_r| (incl. the diagonal, pair_search.cpp:48-49) and the
//      canonical work, reduced in the cluster: the guard
//      (pair_search.hpp:91-94) is decided on-chip;
//   5. emit: candidate pairs / work items of a kept run (emit_items).
// A run whose bucket or chunk exceeds 65535 columns (possible only when
// p > 65535, e.g. many monomorphic columns) is redone exactly with 32-bit
// counters in a global table slot.
#pragma once

#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"
#include "search_kernels.cuh"

namespace xyzb {
namespace kern {

constexpr int kCtThreads = 1024;
constexpr int kCtChunkBits = 8;  // 256 buckets share one u32 base

// Block-wide exclusive scan of one u32 per thread; returns the exclusive
// prefix, *total gets the block total. Uses `ws` (>= 33 u32) as scratch.
__device__ __forceinline__ u32 block_exclusive(u32 x, u32* ws, u32* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    u32 incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) ws[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const u32 w = lane < nw ? ws[lane] : 0u;
        u32 wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        ws[lane] = wi - w;
        if (lane == 31) ws[32] = wi;
    }
    __syncthreads();
    const u32 r = ws[wid] + incl - x;
    *total = ws[32];
    __syncthreads();  // ws reusable
    return r;
}

// Two scans behind the same three barriers (items and pairs of a join's emission): ws >= 66 u32.
__device__ __forceinline__ void block_exclusive2(u32 x, u32 y, u32* ws, u32& ex, u32& ey, u32* tx, u32* ty) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    u32 ix = x, iy = y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 a = __shfl_up_sync(0xffffffffu, ix, o), b = __shfl_up_sync(0xffffffffu, iy, o);
        if (lane >= o) {
            ix += a;
            iy += b;
        }
    }
    if (lane == 31) {
        ws[wid] = ix;
        ws[33 + wid] = iy;
    }
    __syncthreads();
    if (wid == 0) {
        const u32 wx = lane < nw ? ws[lane] : 0u, wy = lane < nw ? ws[33 + lane] : 0u;
        u32 jx = wx, jy = wy;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 a = __shfl_up_sync(0xffffffffu, jx, o), b = __shfl_up_sync(0xffffffffu, jy, o);
            if (lane >= o) {
                jx += a;
                jy += b;
            }
        }
        ws[lane] = jx - wx;
        ws[33 + lane] = jy - wy;
        if (lane == 31) {
            ws[32] = jx;
            ws[65] = jy;
        }
    }
    __syncthreads();
    ex = ws[wid] + ix - x;
    ey = ws[33 + wid] + iy - y;
    *tx = ws[32];
    *ty = ws[65];
    __syncthreads();  // ws reusable
}

// 16-bit counters in shared memory + chunk bases.
struct SmemTab16 {
    u32* w;      // 2^(M-1) words (two buckets each)
    u32* base;   // 2^M >> kCtChunkBits chunk bases (>= 1)
    int M;
    int cbits;   // log2 buckets per chunk
    u32* ovf;    // shared overflow flag

    __device__ void clear() {
        const u32 nw = (u32(1) << M) >> 1;
        for (u32 i = threadIdx.x; i < nw; i += blockDim.x) w[i] = 0;
    }
    template <bool CHECK>
    __device__ __forceinline__ u32 add(u32 v, u32 n) {
        const u32 sh = (v & 1u) << 4;
        const u32 old = atomicAdd(w + (v >> 1), n << sh);
        const u32 h = (old >> sh) & 0xffffu;
        if (CHECK && h + n > 0xffffu) *ovf = 1u;
        return h;
    }
    __device__ __forceinline__ u32 chunk_base(u32 v) const { return base[v >> cbits]; }
    __device__ __forceinline__ u32 half(u32 v) const { return (w[v >> 1] >> ((v & 1u) << 4)) & 0xffffu; }
    // counts -> exclusive in-chunk offsets; chunk bases; flags chunks > 65535.
    // Each warp owns a contiguous segment of whole chunks: pass A sums it,
    // one warp scans the segment totals, pass B walks the segment in 32-word
    // steps (conflict-free, warp shuffles) writing offsets and chunk bases.
    // Two block barriers in all.
    __device__ u32 scan(u32* ws) {
        const u32 NW = (u32(1) << M) >> 1;
        const u32 cw = u32(1) << (cbits - 1);  // words per chunk (cbits >= 1)
        const u32 nwarps = blockDim.x >> 5;
        u32 seg = (NW + nwarps - 1) / nwarps;
        seg = (seg + cw - 1) / cw * cw;
        if (seg < 32) seg = 32;  // whole steps (a segment may then hold several chunks)
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        const u32 s0 = u32(wid) * seg, s1 = min(NW, s0 + seg);
        u32 loc = 0;
        for (u32 wi = s0 + lane; wi < s1; wi += 32) {
            const u32 x = w[wi];
            loc += (x & 0xffffu) + (x >> 16);
        }
        loc = warp_sum(loc);
        if (lane == 0) ws[wid] = loc;
        __syncthreads();
        if (wid == 0) {
            const u32 t = u32(lane) < nwarps ? ws[lane] : 0u;
            u32 incl = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            ws[lane] = incl - t;
            if (lane == 31) ws[32] = incl;
        }
        __syncthreads();
        u32 carry = ws[wid], cb = 0;
        for (u32 w0 = s0; w0 < s1; w0 += 32) {
            const u32 wi = w0 + u32(lane);
            const bool act = wi < s1;
            const u32 x = act ? w[wi] : 0u;
            const u32 lo = x & 0xffffu, hi = x >> 16;
            u32 incl = lo + hi;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const u32 pos = carry + incl - (lo + hi);
            if (cw >= 32) {  // chunk starts are step starts
                if ((w0 & (cw - 1)) == 0) cb = __shfl_sync(0xffffffffu, pos, 0);
            } else {  // several chunks per step: the base is the chunk's first lane
                cb = __shfl_sync(0xffffffffu, pos, lane & ~int(cw - 1));
            }
            if (act) {
                if ((wi & (cw - 1)) == 0) base[wi / cw] = pos;
                const u32 o = pos - cb;
                if (o + lo + hi > 0xffffu) *ovf = 1u;
                w[wi] = (o & 0xffffu) | (((o + lo) & 0xffffu) << 16);
            }
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
        const u32 total = ws[32];
        __syncthreads();  // ws reusable
        return total;
    }
    // after the scatter: bucket v occupies [beg, beg + cnt)
    __device__ __forceinline__ void group(u32 v, u32& beg, u32& cnt) const {
        const u32 cb = base[v >> cbits];
        const u32 end = cb + half(v);
        const u32 st = (v & ((u32(1) << cbits) - 1)) ? cb + half(v - 1) : cb;
        beg = st;
        cnt = end - st;
    }
};

// 32-bit counters in global memory (overflow fallback).
struct GlobalTab32 {
    u32* t;  // 2^M
    int M;

    __device__ void clear() {
        const u32 T = u32(1) << M;
        for (u32 i = threadIdx.x; i < T; i += blockDim.x) t[i] = 0;
    }
    template <bool CHECK>
    __device__ __forceinline__ u32 add(u32 v, u32 n) { return atomicAdd(t + v, n); }
    __device__ void scan(u32* ws) {
        const u32 T = u32(1) << M;
        const u32 bpt = max(1u, T / blockDim.x);
        const u32 a0 = threadIdx.x * bpt;
        const bool act = a0 < T;
        u32 loc = 0;
        if (act)
            for (u32 i = a0; i < a0 + bpt; ++i) loc += t[i];
        u32 total;
        u32 run = block_exclusive(loc, ws, &total);
        if (act)
            for (u32 i = a0; i < a0 + bpt; ++i) {
                const u32 x = t[i];
                t[i] = run;
                run += x;
            }
    }
    __device__ __forceinline__ void group(u32 v, u32& beg, u32& cnt) const {
        const u32 end = t[v];
        const u32 st = v ? t[v - 1] : 0u;
        beg = st;
        cnt = end - st;
    }
};

constexpr int kCtUnroll = 8;  // keys in flight per thread

// One pass over a run's keys: count (out == nullptr) or scatter positions.
// POS16: positions are chunk base + 16-bit in-chunk offset (SmemTab16).
template <bool AGG, bool CHECK, bool POS16, class K, class Tab>
__device__ __forceinline__ void tab_pass(Tab& tab, const K* __restrict__ kb, u64 p, u32* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const u64 step = u64(blockDim.x) * kCtUnroll;
    for (u64 i0 = 0; i0 < p; i0 += step) {
        u32 v[kCtUnroll];
#pragma unroll
        for (int u = 0; u < kCtUnroll; ++u) {
            const u64 i = i0 + u64(u) * blockDim.x + threadIdx.x;
            v[u] = i < p ? u32(__ldg(kb + i)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kCtUnroll; ++u) {
            const u64 i = i0 + u64(u) * blockDim.x + threadIdx.x;
            const bool valid = i < p;
            if (AGG) {
                const u32 active = __ballot_sync(0xffffffffu, valid);
                if (valid) {
                    const u32 peers = __match_any_sync(active, v[u]);
                    const int leader = __ffs(peers) - 1;
                    u32 pos = 0;
                    if (lane == leader) {
                        pos = tab.template add<CHECK>(v[u], __popc(peers));
                        if constexpr (POS16) pos += tab.chunk_base(v[u]);
                    }
                    if (out) {
                        pos = __shfl_sync(peers, pos, leader) + __popc(peers & lanemask_lt());
                        out[pos] = u32(i);
                    }
                }
            } else if (valid) {
                u32 pos = tab.template add<CHECK>(v[u], 1u);
                if (out) {
                    if constexpr (POS16) pos += tab.chunk_base(v[u]);
                    out[pos] = u32(i);
                }
            }
        }
    }
}

template <class K, class Tab>
__device__ __forceinline__ HeadBlock tab_block(const Tab& tab, u32 v, K c) {
    HeadBlock hb;
    u32 bx, cx;
    tab.group(v, bx, cx);
    if (cx == 0) return hb;
    const u32 v2 = v ^ u32(c);
    if (v2 == v) {
        hb.pairs = u64(cx) * cx;  // the diagonal j == k counts (pair_search.cpp:48-49)
        if (cx >= 2) {
            hb.work = u64(cx) * (cx - 1) / 2;
            hb.hs = bx; hb.hc = cx; hb.ss = bx; hb.sc = cx; hb.flags = 3u;
        }
    } else if (v2 > v) {
        u32 bz, cz;
        tab.group(v2, bz, cz);
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
}

// Steps 4-5 on a filled table. Pass 1 sums |E_r|, the canonical work and
// this thread's item / pair counts; a kept run reserves its slots with ONE
// atomic per counter, and pass 2 writes at per-thread offsets (no barriers).
template <class K, class Tab>
__device__ void tab_join(const Tab& tab, int M, u32 b, K c, u64 p, u64 guard, u32 hmax, u64* __restrict__ tot,
                         u64* __restrict__ work_run, Item* __restrict__ items, u32* __restrict__ nitems, u32 item_cap,
                         u32* __restrict__ npairs, PairRec* __restrict__ pairs, u32 pair_cap, u64 (*red)[33],
                         u32* ws, const u32* __restrict__ grouped) {
    const u32 T = u32(1) << M;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool pair_list = npairs != nullptr;
    u64 pa = 0, wa = 0;
    u32 my_items = 0, my_pairs = 0;
    for (u32 v = threadIdx.x; v < T; v += blockDim.x) {
        const HeadBlock hb = tab_block<K>(tab, v, c);
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
        red[0][32] = a;
        red[1][32] = w;
        tot[b] = a;
        work_run[b] = w;
    }
    __syncthreads();
    const u64 run_pairs = red[0][32];
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
        for (u32 v = threadIdx.x; v < T; v += blockDim.x) {
            const HeadBlock hb = tab_block<K>(tab, v, c);
            if (hb.work == 0) continue;
            u32 ne, np, nsc;
            emit_count(hb, hmax, pair_list, ne, np, nsc);
            emit_write(hb, b, hmax, pair_list, ne, nsc, ibase, pbase, items, item_cap, pairs, pair_cap, p, grouped);
            ibase += ne;
            pbase += np;
        }
    }
    __syncthreads();  // red / ws / tables reusable
}

// ------------------------------------------------ two-CTA split per run --
//
// The bucket space of a run is split between the two CTAs of a cluster
// (2^(M-1) 16-bit counters each, 64 KB at M = 16, so three CTAs share an SM
// and every run of a 200-run batch is resident at once instead of two rounds
// of one CTA per SM). CTA r owns the keys v with parity(v & Z) == r, Z = the
// zero bits of c = x-key ^ z-key: a key and its partner v ^ c agree on Z, so
// they always live in the same CTA, and the parity of several biased bits
// splits the keys evenly. The local index drops bit t = lowest bit of Z
// (recovered from r and the parity of the other Z bits). Only when c has no
// zero bit (c = all ones, partner = ~v) is the split on bit t = M - 1 and the
// join reads the partner CTA's table through distributed shared memory. The cluster exchanges three things: the
// key count of CTA 0 (CTA 1's positions follow it), the overflow flags, and
// the run's |E_r| for the guard.
constexpr int kSpThreads = 512;

__device__ __forceinline__ u32 split_local(u32 v, int t) {
    return ((v >> (t + 1)) << t) | (v & ((u32(1) << t) - 1));
}
// Owner CTA of key v: parity of v & om (om = Z, or bit t when c has no zero bit).
__device__ __forceinline__ u32 split_owner(u32 v, u32 om) { return u32(__popc(v & om)) & 1u; }
__device__ __forceinline__ u32 split_key(u32 li, u32 r, int t, u32 om) {
    const u32 u = ((li >> t) << (t + 1)) | (li & ((u32(1) << t) - 1));  // bit t clear
    return u | ((r ^ split_owner(u, om)) << t);
}

// Leaner pass over a run's u32 keys (the split path always has M <= 16):
// 16-byte vector loads (8 keys in flight per thread), 32-bit indices, and
// ownership / local index by masks. A scalar head and tail cover a run
// whose keys are not 16-byte aligned. AGG keeps the warp-aggregated form for
// small tables (every lane of a warp calls `one` the same number of times).
template <bool AGG, bool CHECK, bool SCATTER>
__device__ __forceinline__ void split_pass32(SmemTab16& tab, const u32* __restrict__ kb, u32 p, int t, u32 om,
                                             u32 r, u32 base, u32* __restrict__ out) {
    const u32 lo = (1u << t) - 1u;
    const int lane = threadIdx.x & 31;
    auto one = [&](u32 v, u32 i, bool valid) {
        const bool mine = valid && split_owner(v, om) == r;
        const u32 li = ((v >> 1) & ~lo) | (v & lo);
        if (AGG) {
            const u32 active = __ballot_sync(0xffffffffu, mine);
            if (mine) {
                const u32 peers = __match_any_sync(active, li);
                const int leader = __ffs(peers) - 1;
                u32 pos = 0;
                if (lane == leader) {
                    pos = tab.template add<CHECK>(li, __popc(peers));
                    if (SCATTER) pos += base + tab.chunk_base(li);
                }
                if (SCATTER) out[__shfl_sync(peers, pos, leader) + __popc(peers & lanemask_lt())] = i;
            }
        } else if (mine) {
            const u32 pos = tab.template add<CHECK>(li, 1u);
            if (SCATTER) out[base + tab.chunk_base(li) + pos] = i;
        }
    };
    const u32 mis = u32(reinterpret_cast<uintptr_t>(kb) >> 2) & 3u;
    const u32 head = min(p, (4u - mis) & 3u);
    if (threadIdx.x < 32) {  // head and tail: fewer than 4 keys each, one warp
        const bool hv = u32(lane) < head;
        one(hv ? kb[lane] : 0u, u32(lane), hv);
    }
    const u32 n4 = (p - head) >> 2;
    const u32 tail0 = head + 4 * n4;
    if (threadIdx.x < 32) {
        const bool tv = tail0 + lane < p;
        one(tv ? kb[tail0 + lane] : 0u, tail0 + lane, tv);
    }
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

template <class K, bool AGG, bool CHECK>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kSpThreads, 3) split_group_join(
    const K* __restrict__ keys, u64 p, int M, const K* __restrict__ xorc, u64 guard, u32 hmax,
    u32* __restrict__ grouped, u64* __restrict__ tot, u64* __restrict__ work_run, Item* __restrict__ items,
    u32* __restrict__ nitems, u32 item_cap, u32* __restrict__ npairs, PairRec* __restrict__ pairs, u32 pair_cap,
    u32* __restrict__ gtab, u32* __restrict__ slots) {
    static_assert(sizeof(K) == 4, "the split path runs with u32 keys (M <= 16)");
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) u32 smem[];
    __shared__ u32 ws[68];
    __shared__ u32 s_ovf, s_n, s_slot;
    __shared__ u64 red[2][33];
    __shared__ u64 s_part[2];
    const u32 r = cl.block_rank();
    const u32 b = blockIdx.y;
    const K* kb = keys + u64(b) * p;
    u32* out = grouped + u64(b) * p;
    const int Ml = M - 1;
    const u32 Tl = u32(1) << Ml;
    const int cbits = min(Ml, kCtChunkBits);
    const u32 nbase = max(1u, Tl >> cbits);
    SmemTab16 tab{smem + nbase, smem, Ml, cbits, &s_ovf};
    const u32 mask = (u32(1) << M) - 1;
    const u32 c = u32(xorc[b]) & mask;
    const u32 zb = ~c & mask;
    const bool local = zb != 0;
    const int t = local ? __ffs(zb) - 1 : M - 1;
    const u32 om = local ? zb : (1u << t);

    if (threadIdx.x == 0) s_ovf = 0;
    tab.clear();
    __syncthreads();
    split_pass32<AGG, CHECK, false>(tab, reinterpret_cast<const u32*>(kb), u32(p), t, om, r, 0u,
                                    static_cast<u32*>(nullptr));
    __syncthreads();
    const u32 n_mine = tab.scan(ws);
    if (threadIdx.x == 0) s_n = n_mine;
    __syncthreads();
    cl.sync();  // #1: counts and overflow flags of both CTAs
    const u32 n_other = *cl.map_shared_rank(&s_n, r ^ 1u);
    const bool ovf = CHECK && (s_ovf | *cl.map_shared_rank(&s_ovf, r ^ 1u));
    if (ovf) {
        // a bucket or chunk above 65535 columns: CTA 0 redoes the whole run with
        // 32-bit counters in a global scratch slot (slots taken by CAS, released after)
        if (r == 0) {
            if (threadIdx.x == 0) {
                u32 sl = b % kSMs;
                while (atomicCAS(slots + sl, 0u, 1u) != 0u) sl = (sl + 1) % kSMs;
                s_slot = sl;
            }
            __syncthreads();
            GlobalTab32 g{gtab + (u64(s_slot) << M), M};
            g.clear();
            __syncthreads();
            tab_pass<AGG, false, false>(g, kb, p, static_cast<u32*>(nullptr));
            __syncthreads();
            g.scan(ws);
            __syncthreads();
            tab_pass<AGG, false, false>(g, kb, p, out);
            __syncthreads();
            tab_join<K>(g, M, b, K(c), p, guard, hmax, tot, work_run, items, nitems, item_cap, npairs, pairs,
                        pair_cap, red, ws, grouped);
            __threadfence();
            if (threadIdx.x == 0) atomicExch(slots + s_slot, 0u);
        }
        cl.sync();
        return;
    }
    const u32 n0 = r == 0 ? n_mine : n_other;  // CTA 1's positions follow CTA 0's
    const u32 base = r == 0 ? 0u : n0;
    split_pass32<AGG, false, true>(tab, reinterpret_cast<const u32*>(kb), u32(p), t, om, r, base, out);
    __syncthreads();
    if (!local) cl.sync();  // #2: the partner's table is final before remote reads
    // group of key v: its owner's table (local or, for c = all ones, the partner's)
    SmemTab16 rt = tab;
    rt.w = cl.map_shared_rank(tab.w, r ^ 1u);
    rt.base = cl.map_shared_rank(tab.base, r ^ 1u);
    const u32 other_base = r == 0 ? n0 : 0u;
    auto group = [&](u32 v, u32& beg, u32& cnt) {
        if (split_owner(v, om) == r) {
            tab.group(split_local(v, t), beg, cnt);
            beg += base;
        } else {
            rt.group(split_local(v, t), beg, cnt);
            beg += other_base;
        }
    };
    auto block_of = [&](u32 li) {
        HeadBlock hb;
        const u32 v = split_key(li, r, t, om);
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
    // join pass 1: |E_r| share, canonical work, this thread's item / pair counts
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
    cl.sync();  // #3: both CTAs' shares of |E_r|
    const u64* op = cl.map_shared_rank(s_part, r ^ 1u);
    const u64 run_pairs = s_part[0] + op[0];
    if (r == 0 && threadIdx.x == 0) {
        tot[b] = run_pairs;
        work_run[b] = s_part[1] + op[1];
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
        // pass 2, warp-cooperative: the pairs of small blocks are written by the
        // whole warp, one coalesced 16-byte record per lane (a lane's own blocks
        // would leave most of the warp idle); large blocks become items as before.
        // The warp owns the contiguous slot range of its 32 threads.
        u32 woff = __shfl_sync(0xffffffffu, pbase, 0);
        const u32 off = u32(u64(b) * p);
        uint4* dst = reinterpret_cast<uint4*>(pairs);
        for (u32 li0 = 0; li0 < Tl; li0 += blockDim.x) {
            const u32 li = li0 + threadIdx.x;
            HeadBlock hb;
            if (li < Tl) hb = block_of(li);
            u32 ne, np, nsc;
            emit_count(hb, hmax, pair_list, ne, np, nsc);
            const bool inl = pair_list && hb.work != 0 && hb.work <= kInlinePairs;
            const u32 ni = inl ? np : 0u;
            u32 ea = np, ei = ni;  // inclusive warp scans of all pairs / inline pairs
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t1 = __shfl_up_sync(0xffffffffu, ea, o), t2 = __shfl_up_sync(0xffffffffu, ei, o);
                if (lane >= o) {
                    ea += t1;
                    ei += t2;
                }
            }
            const u32 tot_all = __shfl_sync(0xffffffffu, ea, 31), tot_inl = __shfl_sync(0xffffffffu, ei, 31);
            const u32 xa = ea - np;  // this lane's first slot within the warp's share of the iteration
            if (ne) {  // large blocks: items (their pairs are expanded later at it.pad)
                emit_write(hb, b, hmax, pair_list, ne, nsc, ibase, woff + xa, items, item_cap, pairs, pair_cap, p,
                           grouped);
                ibase += ne;
            }
            for (u32 idx0 = 0; idx0 < tot_inl; idx0 += 32) {
                const u32 idx = idx0 + lane;
                // owner lane: the first lane whose inclusive inline count exceeds idx
                u32 ow = 0;
#pragma unroll
                for (int stp = 16; stp > 0; stp >>= 1) {
                    const u32 v = __shfl_sync(0xffffffffu, ei, int(ow + stp - 1));
                    if (v <= idx) ow += stp;
                }
                ow = min(ow, 31u);
                const u32 o_hs = __shfl_sync(0xffffffffu, hb.hs, ow), o_hc = __shfl_sync(0xffffffffu, hb.hc, ow);
                const u32 o_ss = __shfl_sync(0xffffffffu, hb.ss, ow), o_sc = __shfl_sync(0xffffffffu, hb.sc, ow);
                const u32 o_fl = __shfl_sync(0xffffffffu, hb.flags, ow);
                const u32 o_xa = __shfl_sync(0xffffffffu, xa, ow);
                const u32 o_ei = __shfl_sync(0xffffffffu, ei - ni, ow);  // owner's first inline index
                if (idx < tot_inl) {
                    u32 l = idx - o_ei, h = 0, q;
                    const bool diag = o_fl & 2u;
                    if (diag) {  // pairs (h, q), h < q < hc: walk the rows (hc <= 8 here)
                        while (l >= o_hc - 1 - h) {
                            l -= o_hc - 1 - h;
                            ++h;
                        }
                        q = h + 1 + l;
                    } else {
                        h = l / o_sc;
                        q = l - h * o_sc;
                    }
                    const u32 slot = woff + o_xa + (idx - o_ei);
                    if (slot < pair_cap) {
                        const u32 hcol = grouped[off + o_hs + h], scol = grouped[off + o_ss + q];
                        const bool first_held = diag || (o_fl & 1u);
                        dst[slot] = make_uint4(first_held ? hcol : scol, first_held ? scol : hcol, b, o_fl);
                    }
                }
            }
            woff += tot_all;
        }
    }
    cl.sync();  // #4: the partner may still read this CTA's table and shares
}

inline size_t split_group_smem(int M) {
    const u64 Tl = u64(1) << (M - 1);
    const int cbits = (M - 1) < kCtChunkBits ? (M - 1) : kCtChunkBits;
    return size_t(Tl / 2) * 4 + size_t(std::max<u64>(1, Tl >> cbits)) * 4;
}

template <class K, bool AGG, bool CHECK>
void split_group_join_go(const K* keys, u64 B, u64 p, int M, const K* xorc, u64 guard, u32 hmax, u32* grouped,
                         u64* tot, u64* work_run, Item* items, u32* nitems, u32 item_cap, u32* npairs, PairRec* pairs,
                         u32 pair_cap, u32* gtab, u32* slots, cudaStream_t st) {
    auto kernel = split_group_join<K, AGG, CHECK>;
    func_smem(kernel, split_group_smem(16));
    dim3 grid(2, static_cast<u32>(B));
    kernel<<<grid, kSpThreads, split_group_smem(M), st>>>(keys, p, M, xorc, guard, hmax, grouped, tot, work_run,
                                                          items, nitems, item_cap, npairs, pairs, pair_cap, gtab,
                                                          slots);
}

// M in [2, 16]; gtab / slots: the overflow scratch (p > 65535 only).
template <class K>
void split_group_join_launch(const K* keys, u64 B, u64 p, int M, const K* xorc, u64 guard, u32 hmax, u32* grouped,
                             u64* tot, u64* work_run, Item* items, u32* nitems, u32 item_cap, u32* npairs,
                             PairRec* pairs, u32 pair_cap, u32* gtab, u32* slots, cudaStream_t st) {
    const bool agg = M <= 12;
    const bool check = p > 0xffffu;
    auto go = agg ? (check ? split_group_join_go<K, true, true> : split_group_join_go<K, true, false>)
                  : (check ? split_group_join_go<K, false, true> : split_group_join_go<K, false, false>);
    go(keys, B, p, M, xorc, guard, hmax, grouped, tot, work_run, items, nitems, item_cap, npairs, pairs, pair_cap,
       gtab, slots, st);
}

// Scratch (u32 entries) of the 16-bit overflow fallback: one 2^M table per slot.
inline u64 split_group_scratch(int M, u64 p) { return p > 0xffffu ? (u64(kSMs) << M) : 0; }

} // namespace kern
} // namespace xyzb
