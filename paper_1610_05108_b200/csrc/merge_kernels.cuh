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

// Open-addressing table tag -> min order key.
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
        atomicMin(reinterpret_cast<unsigned long long*>(tvals + slot), x.order);
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
        keep[i] = (tvals[slot] == x.order && x.rid <= *rmax) ? 1u : 0u;
    }
}

__global__ void compact(const DevHit* __restrict__ h, u32 H, const u32* __restrict__ keep, const u32* __restrict__ pos,
                        DevHit* __restrict__ out, u64* __restrict__ order_keys) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < H; i += u64(gridDim.x) * blockDim.x) {
        if (keep[i]) {
            out[pos[i]] = h[i];
            order_keys[pos[i]] = h[i].order;
        }
    }
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

} // namespace merge
} // namespace xyzb
