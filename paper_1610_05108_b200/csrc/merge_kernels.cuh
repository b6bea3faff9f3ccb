// Device merge of the pre-dedup hit list (run_pass's slot-ordered merge,
// search.cpp:96-108, as Appendix A.8 states it): keep the first occurrence
// (smallest order key) of each (min(j,k), max(j,k), sign), order the kept
// hits by order key, and rank them for top-K (A.10).
#pragma once

#include "common.cuh"
#include "search_kernels.cuh"

namespace xyzb {
namespace merge {

using kern::DevHit;

constexpr u64 kEmpty = ~0ull;

__device__ __forceinline__ u64 tag_of(const DevHit& h, int8_t sign) {
    const u64 canon = (u64(min(h.j, h.k)) << 32) | max(h.j, h.k);
    return canon ^ (sign < 0 ? (1ull << 63) : 0ull);
}

__device__ __forceinline__ u64 hash64(u64 x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__global__ void fill_u64(u64* a, u64 n, u64 v) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) a[i] = v;
}

// stop_after_first_hit: smallest run id holding a hit
__global__ void min_rid(const DevHit* __restrict__ h, u32 H, u32* __restrict__ out) {
    u32 m = 0xffffffffu;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += u64(gridDim.x) * blockDim.x) m = min(m, h[i].rid);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m != 0xffffffffu) atomicMin(out, m);
}

// Open-addressing table tag -> earliest run holding it (a run verifies each
// unordered pair at most once, so the earliest run identifies the reference's
// first occurrence, A.8).
__global__ void hash_insert(const DevHit* __restrict__ h, u32 H, const int8_t* __restrict__ sign_by_rid,
                            u64* __restrict__ tkeys, u64* __restrict__ tvals, u64 mask) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += u64(gridDim.x) * blockDim.x) {
        const DevHit x = h[i];
        const u64 t = tag_of(x, sign_by_rid[x.rid]);
        u64 slot = hash64(t) & mask;
        while (true) {
            const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(tkeys + slot), kEmpty, t);
            if (prev == kEmpty || prev == t) break;
            slot = (slot + 1) & mask;
        }
        atomicMin(reinterpret_cast<unsigned long long*>(tvals + slot), static_cast<unsigned long long>(x.rid));
    }
}

__global__ void hash_mark(const DevHit* __restrict__ h, u32 H, const int8_t* __restrict__ sign_by_rid,
                          const u64* __restrict__ tkeys, const u64* __restrict__ tvals, u64 mask, const u32* rmax,
                          u32* __restrict__ keep) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += u64(gridDim.x) * blockDim.x) {
        const DevHit x = h[i];
        const u64 t = tag_of(x, sign_by_rid[x.rid]);
        u64 slot = hash64(t) & mask;
        while (tkeys[slot] != t) slot = (slot + 1) & mask;
        keep[i] = (tvals[slot] == u64(x.rid) && x.rid <= *rmax) ? 1u : 0u;
    }
}

__global__ void compact(const DevHit* __restrict__ h, u32 H, const u32* __restrict__ keep, const u32* __restrict__ pos,
                        DevHit* __restrict__ out, u64* __restrict__ jk_key) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += u64(gridDim.x) * blockDim.x) {
        if (keep[i]) {
            out[pos[i]] = h[i];
            jk_key[pos[i]] = (u64(h[i].j) << 32) | h[i].k;
        }
    }
}

// Next LSD key of the (rid, v, j, k) order in the current permutation:
// which = 0 -> v, 1 -> rid.
__global__ void order_key(const DevHit* __restrict__ kept, const u32* __restrict__ perm, u32 K, int which,
                          u64* __restrict__ key) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < K; i += u64(gridDim.x) * blockDim.x) {
        const DevHit& h = kept[perm[i]];
        key[i] = which == 0 ? h.order : u64(h.rid);
    }
}

// perm_out[i] = perm_in[sub[i]]
__global__ void compose_perm(const u32* __restrict__ perm_in, const u32* __restrict__ sub, u32 K,
                             u32* __restrict__ perm_out) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < K; i += u64(gridDim.x) * blockDim.x)
        perm_out[i] = perm_in[sub[i]];
}

// Final records in reference order; also the top-K tie key
// (min asc, max asc, sign desc) packed as (min << (bp+1)) | (max << 1) | (sign < 0).
__global__ void gather_final(const DevHit* __restrict__ kept, const u32* __restrict__ idx, u32 K,
                             const int8_t* __restrict__ sign_by_rid, u64 L, int bp, xyzb_hit* __restrict__ out,
                             u64* __restrict__ order_out, u64* __restrict__ tie_key) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < K; i += u64(gridDim.x) * blockDim.x) {
        const DevHit h = kept[idx[i]];
        const int8_t sg = sign_by_rid[h.rid];
        xyzb_hit o;
        o.j = h.j;
        o.k = h.k;
        o.strength = h.s;
        o.found_at_repetition = u32(h.rid % L) + 1;
        o.sign = sg;
        out[i] = o;
        order_out[i] = h.order;
        const u64 lo = min(h.j, h.k), hi = max(h.j, h.k);
        tie_key[i] = (lo << (bp + 1)) | (hi << 1) | (sg < 0 ? 1ull : 0ull);
    }
}

// Primary top-K key in tie-sorted order: strength descending as an unsigned
// ascending key. Binary: n - sint (exact). Real: inverted IEEE order bits.
__global__ void primary_key(const xyzb_hit* __restrict__ fin, const DevHit* __restrict__ kept_unused,
                            const u32* __restrict__ tie_idx, u32 K, int binary, u32 n, u64* __restrict__ key) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < K; i += u64(gridDim.x) * blockDim.x) {
        const double s = fin[tie_idx[i]].strength;
        u64 k;
        if (binary) {
            const u64 si = u64(llrint(s * double(n)));
            k = u64(n) - si;
        } else {
            u64 b = __double_as_longlong(s);
            b = (b >> 63) ? ~b : (b | (1ull << 63));  // ascending order bits
            k = ~b;                                   // descending strength
        }
        key[i] = k;
    }
}

__global__ void compose_idx(const u32* __restrict__ tie_idx, const u32* __restrict__ prim_idx, u32 K,
                            u64* __restrict__ out) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < K; i += u64(gridDim.x) * blockDim.x)
        out[i] = tie_idx[prim_idx[i]];
}

// ---- single-CTA merge for short hit lists (one launch, no host sync) ----

constexpr int kSmallMerge = 4096;
constexpr int kSmallThreads = 1024;

// In-place bitonic sort of idx[0..N) (N a power of two) by less(a, b).
// Element i lives with thread i % blockDim.x, so the compare-exchange
// partners i ^ j of the stages j < 32 share a warp: those stages run in
// registers (one shuffle each, no barrier); only j >= 32 goes through shared
// memory with a CTA barrier (N = 4096: 40 barriers instead of 78).
template <class Less>
__device__ __forceinline__ void bitonic(u32* idx, int N, Less less) {
    if (N < 32) {  // partial warps: every stage through shared memory
        for (int k = 2; k <= N; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                const int i = threadIdx.x, l = i ^ j;
                if (i < N && l > i) {
                    const u32 a = idx[i], b = idx[l];
                    const bool up = (i & k) == 0;
                    if (up ? less(b, a) : less(a, b)) {
                        idx[i] = b;
                        idx[l] = a;
                    }
                }
                __syncthreads();
            }
        }
        return;
    }
    for (int k = 2; k <= N; k <<= 1) {
        int j = k >> 1;
        for (; j >= 32; j >>= 1) {
            for (int i = threadIdx.x; i < N; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const u32 a = idx[i], b = idx[l];
                    const bool up = (i & k) == 0;
                    if (up ? less(b, a) : less(a, b)) {
                        idx[i] = b;
                        idx[l] = a;
                    }
                }
            }
            __syncthreads();
        }
        for (int i = threadIdx.x; i < N; i += blockDim.x) {  // whole warps: N is a multiple of 32
            u32 mine = idx[i];
            const bool up = (i & k) == 0;
            for (int jj = j; jj > 0; jj >>= 1) {
                const u32 other = __shfl_xor_sync(0xffffffffu, mine, jj);
                const bool lower = (i & jj) == 0;
                const u32 a = lower ? mine : other, b = lower ? other : mine;
                if (up ? less(b, a) : less(a, b)) mine = other;
            }
            idx[i] = mine;
        }
        __syncthreads();
    }
}

// Block-wide exclusive scan of v over threads (blockDim.x <= 1024).
__device__ __forceinline__ u32 block_excl_scan(u32 v, u32* warp_tot, u32* total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u32 incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        const u32 x = lane < nw ? warp_tot[lane] : 0u;
        u32 xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < nw) warp_tot[lane] = xi - x;
        if (lane == nw - 1) warp_tot[32] = xi;
    }
    __syncthreads();
    const u32 r = warp_tot[wid] + incl - v;
    *total = warp_tot[32];
    __syncthreads();
    return r;
}

// Dynamic shared memory: u64 tag[N], u64 v[N], u64 jk[N], u32 rid[N], u32 idx[N], u32 aux[N].
constexpr size_t small_merge_smem(int N) { return size_t(N) * 36; }

// out_counts[0] = kept hits K, out_counts[1] = top-K length. H <= kSmallMerge.
// With Hdev the hit count is read on the device (the merge is queued right
// behind the search, no host round trip); above Hcap the kernel only flags
// out_counts[0] = ~0 and the host takes the multi-kernel merge.
__global__ void __launch_bounds__(kSmallThreads) merge_small(const DevHit* __restrict__ h, u32 H,
                                                             const int8_t* __restrict__ sign_by_rid, u32 rmax, u64 L,
                                                             u64 top_k, xyzb_hit* __restrict__ out,
                                                             u64* __restrict__ order_out, u64* __restrict__ top_out,
                                                             u32* __restrict__ out_counts,
                                                             const u32* __restrict__ Hdev = nullptr, u32 Hcap = 0) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ u32 warp_tot[33];
    if (Hdev) {
        H = *Hdev;
        if (H > Hcap) {
            if (threadIdx.x == 0) {
                out_counts[0] = 0xffffffffu;
                out_counts[1] = 0;
            }
            return;
        }
    }
    int N = 1;
    while (N < int(H)) N <<= 1;
    u64* s_tag = reinterpret_cast<u64*>(smem);
    u64* s_v = s_tag + N;
    u64* s_jk = s_v + N;
    u32* s_rid = reinterpret_cast<u32*>(s_jk + N);
    u32* s_idx = s_rid + N;
    u32* s_aux = s_idx + N;
    const u64 INF = ~0ull;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        if (i < int(H) && h[i].rid <= rmax) {
            s_tag[i] = tag_of(h[i], sign_by_rid[h[i].rid]);
            s_v[i] = h[i].order;
            s_jk[i] = (u64(h[i].j) << 32) | h[i].k;
            s_rid[i] = h[i].rid;
        } else {
            s_tag[i] = INF;
            s_v[i] = INF;
            s_jk[i] = INF;
            s_rid[i] = 0xffffffffu;
        }
        s_idx[i] = i;
    }
    __syncthreads();
    // dedup: sort by (tag, run); the first of each tag is the kept occurrence
    bitonic(s_idx, N, [&](u32 a, u32 b) {
        return s_tag[a] != s_tag[b] ? s_tag[a] < s_tag[b] : s_rid[a] < s_rid[b];
    });
    // compact kept hit indices into s_aux[0..K) (stable scan over the sorted list)
    u32 K = 0;
    const int per = (N + int(blockDim.x) - 1) / int(blockDim.x);
    {
        const int b0 = threadIdx.x * per, b1 = min(N, b0 + per);
        u32 cnt = 0;
        for (int i = b0; i < b1; ++i) {
            const u32 a = s_idx[i];
            cnt += (s_tag[a] != INF && (i == 0 || s_tag[s_idx[i - 1]] != s_tag[a])) ? 1u : 0u;
        }
        u32 pos = block_excl_scan(cnt, warp_tot, &K);
        for (int i = b0; i < b1; ++i) {
            const u32 a = s_idx[i];
            if (s_tag[a] != INF && (i == 0 || s_tag[s_idx[i - 1]] != s_tag[a])) s_aux[pos++] = a;
        }
    }
    __syncthreads();
    // reference order: kept hits by (run, v, j, k)
    int NK = 1;
    while (NK < int(K)) NK <<= 1;
    for (int i = threadIdx.x; i < NK; i += blockDim.x) s_idx[i] = i < int(K) ? s_aux[i] : u32(0xffffffffu);
    __syncthreads();
    bitonic(s_idx, NK, [&](u32 a, u32 b) {
        if (a == 0xffffffffu || b == 0xffffffffu) return a != 0xffffffffu && b == 0xffffffffu;
        if (s_rid[a] != s_rid[b]) return s_rid[a] < s_rid[b];
        if (s_v[a] != s_v[b]) return s_v[a] < s_v[b];
        return s_jk[a] < s_jk[b];
    });
    // output records; the top-K keys go to shared memory (s_v, s_jk are free
    // once the order sort is done): strength, then (min, max, sign desc)
    double* s_str = reinterpret_cast<double*>(s_tag);
    for (int i = threadIdx.x; i < int(K); i += blockDim.x) {
        const DevHit x = h[s_idx[i]];
        const int8_t sg = sign_by_rid[x.rid];
        xyzb_hit o;
        o.j = x.j;
        o.k = x.k;
        o.strength = x.s;
        o.found_at_repetition = u32(x.rid % L) + 1;
        o.sign = sg;
        out[i] = o;
        order_out[i] = x.order;
    }
    __syncthreads();
    if (top_k > 0 && K > 0) {
        // A.10: strength desc, min asc, max asc, sign desc (positions in `out`)
        for (int i = threadIdx.x; i < int(K); i += blockDim.x) {
            const DevHit x = h[s_idx[i]];
            s_str[i] = x.s;
            s_jk[i] = (u64(min(x.j, x.k)) << 33) | (u64(max(x.j, x.k)) << 1) | (sign_by_rid[x.rid] > 0 ? 0ull : 1ull);
        }
        for (int i = threadIdx.x; i < NK; i += blockDim.x) s_aux[i] = u32(i);
        __syncthreads();
        bitonic(s_aux, NK, [&](u32 a, u32 b) {
            const bool va = a < K, vb = b < K;
            if (!va || !vb) return va && !vb;
            if (s_str[a] != s_str[b]) return s_str[a] > s_str[b];
            return s_jk[a] < s_jk[b];
        });
        const u64 kk = top_k < u64(K) ? top_k : u64(K);
        for (int i = threadIdx.x; i < int(kk); i += blockDim.x) top_out[i] = s_aux[i];
        if (threadIdx.x == 0) out_counts[1] = u32(kk);
    } else if (threadIdx.x == 0) {
        out_counts[1] = 0;
    }
    if (threadIdx.x == 0) out_counts[0] = K;
}

} // namespace merge
} // namespace xyzb
