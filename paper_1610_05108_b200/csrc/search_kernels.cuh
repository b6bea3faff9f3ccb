// Device kernels of one batch of xyz runs (sm_100a).
//
//   transpose_bits   column-major packed X -> row planes (once per dataset)
//   project_bits     M-bit keys of every column for every run of the batch
//                    (project_keys, projection.cpp:32-57) + the per-run XOR
//                    constant c that turns x-keys into z-keys (A.3)
//   join             bucket join over the sorted keys: equal-key groups,
//                    partner group of key^c, |E_r| incl. the diagonal, and
//                    canonical work items (equal_pairs, pair_search.cpp:35-53;
//                    guard pair_search.hpp:91-94 applied per run)
//   verify_*         exact strength of every canonical candidate, hit test,
//                    warp-aggregated hit append (filter_strong,
//                    pair_search.hpp:95-109; strengths transforms.cpp:33-76,
//                    search.cpp:477-493)
#pragma once

#include "common.cuh"

namespace xyzb {
namespace kern {

// A verified candidate with strength >= gamma (pre-dedup).
struct DevHit {
    u64 order;     // x-side key v: the reference order is (rid, v, j, k) (A.5)
    double s;      // strength (binary: exact sint / n)
    u32 j, k;      // oriented as the reference emits it (first in A.5 order)
    u32 rid;       // global run index: pass * L + rep - 1
    int32_t sint;  // binary: integer strength numerator; else -1
};

// A tile of one canonical block of one run: `hc` (<= kHeld) held columns at
// sorted positions [hs, hs+hc) against `sc` streamed columns at [ss, ss+sc).
// flags: bit0 = held side is the x side, bit1 = diagonal block (c == 0,
// group paired with itself; only pairs with streamed pos > held pos count).
constexpr int kHeld = 8;
constexpr u32 kStreamChunk = 64;  // max streamed columns per item
struct Item {
    u32 run;  // batch-local run
    u32 hs, ss, sc;
    u32 hc_flags;  // hc | flags << 8
    u32 pad;
};

// One canonical candidate of the pair-list path: batch-global sorted
// positions of the x side and the z side (x side first; diagonal blocks are
// re-oriented by column index at hit time), the batch-local run, and the
// block flags.
struct __align__(16) PairRec {
    u32 pa, pb, run, pad;  // pa / pb: the COLUMNS of the x side and the z side
};
constexpr u64 kInlinePairs = 32;  // blocks up to this many pairs are expanded by join_emit

// ---------------------------------------------------------------- layout --

// Xc: u64 [p][Wp] column-major words -> Xr: u32 [n][P32] row planes, bit
// (j & 31) of word j >> 5 of row i is X_ij. One CTA per tile of 1024 columns
// x 256 rows: warp q loads 4 words (one 32 B sector) of each of its 32
// columns, shuffle-butterfly bit transposes give the 32-column plane words
// of 256 rows (lane l holds rows l, l+32, ...), stored to a shared tile
// which the CTA writes out as 128 B row segments.
constexpr int kTrWords = 4;  // words per column per tile (Wp is a multiple of 4)
__global__ void __launch_bounds__(1024) transpose_bits(const u64* __restrict__ Xc, u64 Wp, u64 W, u64 n, u64 p,
                                                       u64 P32, u32* __restrict__ Xr) {
    __shared__ u32 tile[kTrWords * 64][33];
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const u64 c0 = u64(blockIdx.x) * 32;  // first column group of the tile
    const u64 w0 = u64(blockIdx.y) * kTrWords;
    const u64 col = (c0 + q) * 32 + lane;
    u64 wd[kTrWords];
    if (col < p) {
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(Xc + col * Wp + w0);
        const ulonglong2 a = __ldg(src), b = __ldg(src + 1);
        wd[0] = a.x; wd[1] = a.y; wd[2] = b.x; wd[3] = b.y;
    } else {
        wd[0] = wd[1] = wd[2] = wd[3] = 0;
    }
    // 32x32 bit transposes across the warp (butterfly of shuffles): lane l's
    // half-word t (rows 32t.. of its column) becomes row 32t + l of the 32 columns
    u32 mine[kTrWords * 2];
#pragma unroll
    for (int k = 0; k < kTrWords; ++k) {
        mine[2 * k] = u32(wd[k]);
        mine[2 * k + 1] = u32(wd[k] >> 32);
    }
#pragma unroll
    for (int j = 16; j != 0; j >>= 1) {
        const u32 m = j == 16 ? 0x0000ffffu : j == 8 ? 0x00ff00ffu : j == 4 ? 0x0f0f0f0fu : j == 2 ? 0x33333333u
                                                                                               : 0x55555555u;
        const bool up = lane & j;
#pragma unroll
        for (int t = 0; t < kTrWords * 2; ++t) {
            const u32 o = __shfl_xor_sync(0xffffffffu, mine[t], j);
            mine[t] = up ? (mine[t] & ~m) | ((o >> j) & m) : (mine[t] & m) | ((o & m) << j);
        }
    }
#pragma unroll
    for (int t = 0; t < kTrWords * 2; ++t) tile[t * 32 + lane][q] = mine[t];
    __syncthreads();
    for (u32 idx = threadIdx.x; idx < kTrWords * 64 * 32; idx += 1024) {
        const u32 r = idx >> 5, g = idx & 31;
        const u64 row = w0 * 64 + r, c = c0 + g;
        if (row < n && c < P32) Xr[row * P32 + c] = tile[r][g];
    }
}

// --------------------------------------------------------------- project --

template <class K>
__device__ __forceinline__ K key_mask(int m) {
    return m >= int(sizeof(K) * 8) ? ~K(0) : ((K(1) << m) - 1);
}

// In-register 32 x 32 bit transpose, LSB-first: afterwards a[c] bit s equals
// the original a[s] bit c (5 butterfly stages, 80 swaps).
__device__ __forceinline__ void transpose32(u32 (&a)[32]) {
#pragma unroll
    for (int j = 16, m = 0x0000ffff; j != 0; j >>= 1, m ^= (m << j)) {
#pragma unroll
        for (int k = 0; k < 32; k = ((k | j) + 1) & ~j) {
            const u32 t = ((a[k] >> j) ^ a[k | j]) & u32(m);
            a[k] ^= t << j;
            a[k | j] ^= t;
        }
    }
}

// Keys for one run from the row planes, 32 columns per thread: the M
// row-plane words of the thread's 32 columns are loaded with coalesced 128 B
// warp requests (one per sampled row), then bit-transposed so word c becomes
// the key of column c (key bit s = X[row_s, c]).
template <class K>
__global__ void __launch_bounds__(128) project_bits_t(const u32* __restrict__ Xr, u64 P32, u64 p,
                                                      const u32* __restrict__ rows, int M, K* __restrict__ keys) {
    __shared__ u32 srow[64];
    const u64 b = blockIdx.y;
    if (threadIdx.x < M) srow[threadIdx.x] = rows[b * M + threadIdx.x];
    __syncthreads();
    const u64 word = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (word >= P32) return;
    const u64 col0 = word * 32;
    const u32 ncol = u32(minu(32, p - col0));
    u32* out = reinterpret_cast<u32*>(keys + b * p + col0);
    constexpr int halves = sizeof(K) / 4;
#pragma unroll
    for (int half = 0; half < halves; ++half) {
        if (half * 32 >= M) {
            if (halves == 2)
                for (u32 c = 0; c < ncol; ++c) out[2 * c + 1] = 0u;
            break;
        }
        u32 a[32];
#pragma unroll
        for (int s = 0; s < 32; ++s) {
            const int ss = half * 32 + s;
            a[s] = ss < M ? __ldg(Xr + u64(srow[ss]) * P32 + word) : 0u;
        }
        transpose32(a);
        if (halves == 1) {
            if (ncol == 32 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
                uint4* o4 = reinterpret_cast<uint4*>(out);
#pragma unroll
                for (int c = 0; c < 8; ++c) o4[c] = make_uint4(a[4 * c], a[4 * c + 1], a[4 * c + 2], a[4 * c + 3]);
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (u32(c) < ncol) out[c] = a[c];
            }
        } else {
#pragma unroll
            for (int c = 0; c < 32; ++c)
                if (u32(c) < ncol) out[2 * c + half] = a[c];
        }
    }
}

// Per-run XOR constant c from the response bits at the sampled rows (A.3):
// z+ = ~(x ^ y) & mask = x ^ (~y & mask); z- = x ^ y.
template <class K>
__global__ void ykey_xorc(const u32* __restrict__ rows, int M, const u64* __restrict__ ykey_bits,
                          const int8_t* __restrict__ run_sign, u32 B, K* __restrict__ xorc) {
    const u32 b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    u64 yk = 0;
    for (int s = 0; s < M; ++s) {
        const u32 r = rows[u64(b) * M + s];
        yk |= ((ykey_bits[r >> 6] >> (r & 63)) & 1ull) << s;
    }
    const K mask = key_mask<K>(M);
    const K ykk = K(yk) & mask;
    xorc[b] = run_sign[b] > 0 ? K(~ykk & mask) : ykk;
}

// ------------------------------------------------------------------ join --

// first index in [lo, hi) with a[idx] != v, given a[lo] == v (galloping)
template <class K>
__device__ __forceinline__ u64 run_end(const K* a, u64 lo, u64 hi, K v) {
    u64 step = 1, last = lo;
    u64 probe = lo + 1;
    while (probe < hi && a[probe] == v) {
        last = probe;
        step <<= 1;
        probe = lo + step;
    }
    u64 l = last + 1, h = minu(probe, hi);
    while (l < h) {
        const u64 mid = (l + h) >> 1;
        if (a[mid] == v) l = mid + 1; else h = mid;
    }
    return l;
}

template <class K>
__device__ __forceinline__ u64 lower_bound(const K* a, u64 lo, u64 hi, K v) {
    while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// The canonical block owned by the head of an equal-key group at sorted
// position i of run b (nothing if i is not a head, or the partner group is
// absent, or its key is smaller — the partner's head owns the block then).
struct HeadBlock {
    u64 pairs = 0;  // contribution to |E_r|: both orientations, diagonal included
    u64 work = 0;   // canonical off-diagonal pairs
    u32 hs = 0, hc = 0, ss = 0, sc = 0, flags = 0;  // held / streamed ranges
};

template <class K>
__device__ __forceinline__ HeadBlock head_block(const K* a, u64 i, u64 S, int M, K c, const u32* table, u32 b) {
    HeadBlock hb;
    if (i >= S) return hb;
    const K v = a[i];
    if (i != 0 && a[i - 1] == v) return hb;
    const u64 e = run_end(a, i, S, v);
    const u64 cnt = e - i;
    const K v2 = v ^ c;
    if (v2 == v) {
        hb.pairs = cnt * cnt;  // the diagonal j == k counts (pair_search.cpp:48-49)
        if (cnt >= 2) {
            hb.work = cnt * (cnt - 1) / 2;
            hb.hs = u32(i);
            hb.hc = u32(cnt);
            hb.ss = u32(i);
            hb.sc = u32(cnt);
            hb.flags = 3u;
        }
    } else if (v2 > v) {
        u64 lo = S;
        if (table) {
            const u32 t = table[(u64(b) << M) + u64(v2)];
            if (t < S && a[t] == v2) lo = t;
        } else {
            const u64 l2 = lower_bound(a, e, S, v2);
            if (l2 < S && a[l2] == v2) lo = l2;
        }
        if (lo < S) {
            const u64 zc = run_end(a, lo, S, v2) - lo;
            hb.pairs = 2 * cnt * zc;  // (j,k) in block v and (k,j) in block v^c
            hb.work = cnt * zc;
            // hold the smaller side in registers, stream the larger
            if (cnt <= zc) {
                hb.hs = u32(i); hb.hc = u32(cnt); hb.ss = u32(lo); hb.sc = u32(zc); hb.flags = 1u;
            } else {
                hb.hs = u32(lo); hb.hc = u32(zc); hb.ss = u32(i); hb.sc = u32(cnt); hb.flags = 0u;
            }
        }
    }
    return hb;
}

// Pass 1: |E_r| and canonical work per run (the guard needs the whole run).
template <class K>
__global__ void __launch_bounds__(256) join_count(const K* __restrict__ sk, u64 S, int M, const K* __restrict__ xorc,
                                                  const u32* __restrict__ table, u64* __restrict__ tot,
                                                  u64* __restrict__ work_run) {
    __shared__ u64 red[2][8];
    const u32 b = blockIdx.y;
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    const HeadBlock hb = head_block(sk + u64(b) * S, i, S, M, xorc[b], table, b);
    const u64 ws = warp_sum(hb.pairs), ww = warp_sum(hb.work);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = ws;
        red[1][threadIdx.x >> 5] = ww;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 t0 = 0, t1 = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            t0 += red[0][w];
            t1 += red[1][w];
        }
        if (t0) atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), static_cast<unsigned long long>(t0));
        if (t1) atomicAdd(reinterpret_cast<unsigned long long*>(work_run + b), static_cast<unsigned long long>(t1));
    }
}

// How many work items and inline pairs block `hb` emits (pairs: canonical
// candidates, all of them whether inline or through items).
__device__ __forceinline__ void emit_count(const HeadBlock& hb, u32 hmax, bool pair_list, u32& nemit, u32& npair,
                                           u32& nsc) {
    nsc = 1;
    nemit = 0;
    const bool inline_pairs = pair_list && hb.work != 0 && hb.work <= kInlinePairs;
    if (hb.work && !inline_pairs) {
        const bool diag = hb.flags & 2u;
        const u32 slen = diag ? hb.hc - 1 : hb.sc;
        const u32 hlen = diag ? hb.hc - 1 : hb.hc;  // the last diagonal column has no later partner
        nsc = (slen + kStreamChunk - 1) / kStreamChunk;
        nemit = (hlen + hmax - 1) / hmax * nsc;
    }
    npair = u32(hb.work);
}

// Write block `hb`'s items from slot `base` and its pairs from slot `poff`.
// Pairs carry column indices (grp: the grouped columns, position -> column),
// so the verify reads no position table.
__device__ __forceinline__ void emit_write(const HeadBlock& hb, u32 b, u32 hmax, bool pair_list, u32 nemit, u32 nsc,
                                           u32 base, u32 poff, Item* __restrict__ items, u32 item_cap,
                                           PairRec* __restrict__ pairs, u32 pair_cap, u64 S,
                                           const u32* __restrict__ grp) {
    const bool inline_pairs = pair_list && hb.work != 0 && hb.work <= kInlinePairs;
    const bool diag = hb.flags & 2u;
    if (inline_pairs) {
        const bool first_held = diag || (hb.flags & 1u);
        const u32 off = u32(u64(b) * S);  // pair positions are u32 (b * S + pos < 2^32, checked by the host)
        uint4* dst = reinterpret_cast<uint4*>(pairs);
        for (u32 h = 0; h < hb.hc && poff < pair_cap; ++h) {
            const u32 hcol = grp[off + hb.hs + h];
            for (u32 q = diag ? h + 1 : 0; q < hb.sc; ++q, ++poff) {
                if (poff >= pair_cap) break;
                const u32 scol = grp[off + hb.ss + q];
                dst[poff] = make_uint4(first_held ? hcol : scol, first_held ? scol : hcol, b, hb.flags);
            }
        }
    }
    const u32 sbeg = diag ? hb.hs + 1 : hb.ss;
    const u32 slen = diag ? hb.hc - 1 : hb.sc;
    for (u32 t = 0; t < nemit; ++t) {
        const u32 slot = base + t;
        if (slot >= item_cap) break;
        const u32 hci = t / nsc, sci = t - hci * nsc;
        const u32 h0 = hci * hmax;
        Item it;
        it.run = b;
        it.hs = hb.hs + h0;
        // diagonal: each held chunk streams hs+1.. (pairs with spos <= hpos are masked)
        it.ss = sbeg + sci * kStreamChunk;
        it.sc = min(kStreamChunk, slen - sci * kStreamChunk);
        const u32 hcnt = min(hmax, hb.hc - h0);
        it.hc_flags = hcnt | (hb.flags << 8);
        it.pad = poff;  // first slot of this item's pairs in the pair list
        items[slot] = it;
        if (diag) {
            for (u32 h = 0; h < hcnt; ++h) {
                const u32 hpos = it.hs + h, lo = max(it.ss, hpos + 1), hi = it.ss + it.sc;
                poff += hi > lo ? hi - lo : 0;
            }
        } else {
            poff += hcnt * it.sc;
        }
    }
}

// --------------------------------------------------------- block emission --

// Pass 2 of a join over T block heads. Every thread owns the contiguous item
// and pair slot ranges its counting pass reserved (ibase / pbase, thread-major
// head order). Large blocks become items (their pairs expanded later at
// it.pad, from the global grouped array); a block of at most kLanePairs
// inline pairs is written by its lane, a larger inline block (<= kInlinePairs)
// by the whole warp, one 16-byte record per lane. Columns of grouped position
// pos are read from gl[pos - gbias] (shared memory when the partition is
// staged there).
constexpr u32 kLanePairs = 4;
template <class BlockOf>
__device__ __forceinline__ void emit_blocks_coop(BlockOf block_of, u32 T, u32 b, u32 hmax, u64 p, bool pair_list,
                                                 u32 ibase, u32 pbase, Item* __restrict__ items, u32 item_cap,
                                                 PairRec* __restrict__ pairs, u32 pair_cap,
                                                 const u32* __restrict__ grouped, const u32* gl, u32 gbias) {
    const int lane = threadIdx.x & 31;
    uint4* dst = reinterpret_cast<uint4*>(pairs);
    for (u32 li0 = 0; li0 < T; li0 += blockDim.x) {
        const u32 li = li0 + threadIdx.x;
        HeadBlock hb;
        if (li < T) hb = block_of(li);
        u32 ne, np, nsc;
        emit_count(hb, hmax, pair_list, ne, np, nsc);
        const bool inl = pair_list && hb.work != 0 && hb.work <= kInlinePairs;
        const bool big = inl && np > kLanePairs;
        if (ne) {
            emit_write(hb, b, hmax, pair_list, ne, nsc, ibase, pbase, items, item_cap, pairs, pair_cap, p, grouped);
            ibase += ne;
        }
        if (inl && !big) {  // a few pairs: this lane writes them
            const bool diag = hb.flags & 2u;
            const bool first_held = diag || (hb.flags & 1u);
            u32 slot = pbase;
            for (u32 h = 0; h < hb.hc; ++h) {
                const u32 hcol = gl[hb.hs + h - gbias];
                for (u32 q = diag ? h + 1 : 0; q < hb.sc; ++q, ++slot) {
                    const u32 scol = gl[hb.ss + q - gbias];
                    if (slot < pair_cap)
                        dst[slot] = make_uint4(first_held ? hcol : scol, first_held ? scol : hcol, b, hb.flags);
                }
            }
        }
        for (u32 bal = __ballot_sync(0xffffffffu, big); bal; bal &= bal - 1) {  // warp-written blocks
            const int ow = __ffs(bal) - 1;
            const u32 o_hs = __shfl_sync(0xffffffffu, hb.hs, ow), o_hc = __shfl_sync(0xffffffffu, hb.hc, ow);
            const u32 o_ss = __shfl_sync(0xffffffffu, hb.ss, ow), o_sc = __shfl_sync(0xffffffffu, hb.sc, ow);
            const u32 o_fl = __shfl_sync(0xffffffffu, hb.flags, ow);
            const u32 o_np = __shfl_sync(0xffffffffu, np, ow), o_slot = __shfl_sync(0xffffffffu, pbase, ow);
            if (u32(lane) < o_np) {
                u32 l = lane, h = 0, q;
                const bool diag = o_fl & 2u;
                if (diag) {
                    while (l >= o_hc - 1 - h) {
                        l -= o_hc - 1 - h;
                        ++h;
                    }
                    q = h + 1 + l;
                } else {
                    // l < 32, o_sc <= 32: the fp32 quotient of l + 0.5 is at least 1/64 from an integer
                    h = __float2uint_rz((float(l) + 0.5f) * __frcp_rn(float(o_sc)));
                    q = l - h * o_sc;
                }
                const u32 slot = o_slot + lane;
                if (slot < pair_cap) {
                    const u32 hcol = gl[o_hs + h - gbias], scol = gl[o_ss + q - gbias];
                    const bool first_held = diag || (o_fl & 1u);
                    dst[slot] = make_uint4(first_held ? hcol : scol, first_held ? scol : hcol, b, o_fl);
                }
            }
        }
        pbase += np;
    }
}

// The same pass with every inline block written by the whole warp: the 32
// heads of a warp step hold ~30 pairs in ~12 non-empty blocks (Poisson
// buckets), so a lane walking its own block leaves most of the warp idle.
// The warp owns the contiguous slot range of its 32 threads (pbase is a
// thread-major exclusive scan); within it each step lays its blocks out lane
// after lane, and pair idx of the step goes to the lane idx % 32: the owner
// block by a binary search over the lanes' inclusive inline counts, its
// fields by shuffles, one 16-byte record per lane.
template <class BlockOf>
__device__ __forceinline__ void emit_blocks_warp(BlockOf block_of, u32 T, u32 b, u32 hmax, u64 p, bool pair_list,
                                                 u32 ibase, u32 pbase, Item* __restrict__ items, u32 item_cap,
                                                 PairRec* __restrict__ pairs, u32 pair_cap,
                                                 const u32* __restrict__ grouped, const u32* gl, u32 gbias) {
    const int lane = threadIdx.x & 31;
    uint4* dst = reinterpret_cast<uint4*>(pairs);
    u32 woff = __shfl_sync(0xffffffffu, pbase, 0);
    for (u32 li0 = 0; li0 < T; li0 += blockDim.x) {
        const u32 li = li0 + threadIdx.x;
        HeadBlock hb;
        if (li < T) hb = block_of(li);
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
        const u32 xa = ea - np;  // this lane's first slot within the warp's share of the step
        if (ne) {  // large blocks: items (their pairs are expanded later at it.pad)
            emit_write(hb, b, hmax, pair_list, ne, nsc, ibase, woff + xa, items, item_cap, pairs, pair_cap, p, grouped);
            ibase += ne;
        }
        for (u32 idx0 = 0; idx0 < tot_inl; idx0 += 32) {
            const u32 idx = idx0 + lane;
            u32 ow = 0;  // owner lane: the first whose inclusive inline count exceeds idx
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
                if (diag) {  // pairs (h, q), h < q < hc
                    while (l >= o_hc - 1 - h) {
                        l -= o_hc - 1 - h;
                        ++h;
                    }
                    q = h + 1 + l;
                } else {
                    // l < 32, o_sc <= 32: the fp32 quotient of l + 0.5 is at least 1/64 from an integer
                    h = __float2uint_rz((float(l) + 0.5f) * __frcp_rn(float(o_sc)));
                    q = l - h * o_sc;
                }
                const u32 slot = woff + o_xa + (idx - o_ei);
                if (slot < pair_cap) {
                    const u32 hcol = gl[o_hs + h - gbias], scol = gl[o_ss + q - gbias];
                    const bool first_held = diag || (o_fl & 1u);
                    dst[slot] = make_uint4(first_held ? hcol : scol, first_held ? scol : hcol, b, o_fl);
                }
            }
        }
        woff += tot_all;
    }
}

// Emit the canonical work items of one block (per thread; CTA-aggregated
// slot reservation). Item t of a block: held chunk t / nsc (<= hmax
// columns), streamed chunk t % nsc (<= kStreamChunk columns), so one big
// group cannot serialise on one team. Small blocks (<= kInlinePairs pairs)
// write their pairs directly. Counters keep counting past the capacities so
// the host can regrow.
__device__ __forceinline__ void emit_items(const HeadBlock& hb, u32 b, u32 hmax, Item* __restrict__ items,
                                           u32* __restrict__ nitems, u32 item_cap, u32* __restrict__ npairs,
                                           PairRec* __restrict__ pairs, u32 pair_cap, u64 S,
                                           const u32* __restrict__ grp) {
    u32 nemit, npair, nsc;
    emit_count(hb, hmax, npairs != nullptr, nemit, npair, nsc);
    u32 incl = nemit, pincl = npair;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        const u32 t2 = __shfl_up_sync(0xffffffffu, pincl, o);
        if (lane >= o) {
            incl += t;
            pincl += t2;
        }
    }
    // CTA-level aggregation: one atomic per counter per CTA (a single global
    // counter hit once per warp serialises at the L2 slice)
    __shared__ u32 s_items[33], s_pairs[33];
    const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 31) {
        s_items[wid] = incl;
        s_pairs[wid] = pincl;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 ti = 0, tp = 0;
        for (int w = 0; w < nw; ++w) {
            const u32 a = s_items[w], c = s_pairs[w];
            s_items[w] = ti;
            s_pairs[w] = tp;
            ti += a;
            tp += c;
        }
        s_items[32] = ti ? atomicAdd(nitems, ti) : 0u;
        s_pairs[32] = (npairs && tp) ? atomicAdd(npairs, tp) : 0u;
    }
    __syncthreads();
    const u32 base = s_items[32] + s_items[wid] + incl - nemit;
    const u32 poff = s_pairs[32] + s_pairs[wid] + pincl - npair;  // this block's first pair slot
    emit_write(hb, b, hmax, npairs != nullptr, nemit, nsc, base, poff, items, item_cap, pairs, pair_cap, S, grp);
}

// Pass 2 (sorted keys): canonical work items of the runs the guard keeps.
template <class K>
__global__ void __launch_bounds__(256) join_emit(const K* __restrict__ sk, u64 S, int M, const K* __restrict__ xorc,
                                                 const u32* __restrict__ table, const u64* __restrict__ tot,
                                                 u64 guard, u32 hmax, Item* __restrict__ items,
                                                 u32* __restrict__ nitems, u32 item_cap,
                                                 u32* __restrict__ npairs, PairRec* __restrict__ pairs,
                                                 u32 pair_cap, const u32* __restrict__ grp) {
    const u32 b = blockIdx.y;
    const bool aborted = tot[b] > guard;
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    HeadBlock hb;
    if (!aborted) hb = head_block(sk + u64(b) * S, i, S, M, xorc[b], table, b);
    emit_items(hb, b, hmax, items, nitems, item_cap, npairs, pairs, pair_cap, S, grp);
}

// ------------------------------------------------ symmetric sorted keys --
//
// Candidates pair key v with key v ^ c. Sorting by u = min(v, v ^ c) with a
// side bit (0: v == u, the x side whose key is the smaller; 1: v == u ^ c)
// puts both groups of a block next to each other — [x side][z side] — so the
// join needs no partner lookup at all: one galloping search for the end of
// the u-group and one for the side split (the reference sorts (key, side,
// index) the same way, pair_search.cpp:17-21). c == 0 makes every group
// diagonal (side 0 only).

template <class K>
__global__ void ukey_transform(K* __restrict__ keys, u64 p, u64 count, const K* __restrict__ xorc) {
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < count; t += u64(gridDim.x) * blockDim.x) {
        const K v = keys[t];
        const K v2 = v ^ xorc[t / p];
        keys[t] = v2 < v ? K((v2 << 1) | 1) : K(v << 1);
    }
}

template <class K>
__device__ __forceinline__ HeadBlock u_block(const K* a, u64 i, u64 S) {
    HeadBlock hb;
    if (i >= S) return hb;
    const K w = a[i];
    const K u = w >> 1;
    if (i != 0 && (a[i - 1] >> 1) == u) return hb;  // not the head of its u-group
    // the group starts on side 0 if it has an x side; find the side split and the group end
    const u64 s = (w & 1) ? i : run_end(a, i, S, w);
    u64 e = s;
    if (s < S && (a[s] >> 1) == u) e = run_end(a, s, S, a[s]);
    const u64 xc = s - i, zc = e - s;
    if (zc == 0) {
        // only one side present: a diagonal group when c == 0 (u == u ^ c), else no candidates
        // (diagonal iff the partner key is the key itself, signalled by the caller through diag)
        hb.hs = u32(i);
        hb.hc = u32(xc);
        return hb;
    }
    if (xc == 0) return hb;
    hb.pairs = 2 * xc * zc;  // (j,k) in block u and (k,j) in block u ^ c
    hb.work = xc * zc;
    if (xc <= zc) {
        hb.hs = u32(i); hb.hc = u32(xc); hb.ss = u32(s); hb.sc = u32(zc); hb.flags = 1u;
    } else {
        hb.hs = u32(s); hb.hc = u32(zc); hb.ss = u32(i); hb.sc = u32(xc); hb.flags = 0u;
    }
    return hb;
}

// c == 0: every group pairs with itself (diagonal, |E| counts the j == k pairs)
__device__ __forceinline__ void make_diag(HeadBlock& hb) {
    const u64 cnt = hb.hc;
    hb.pairs = cnt * cnt;
    if (cnt >= 2) {
        hb.work = cnt * (cnt - 1) / 2;
        hb.ss = hb.hs;
        hb.sc = hb.hc;
        hb.flags = 3u;
    } else {
        hb.hc = 0;
    }
}

template <class K>
__global__ void __launch_bounds__(256) ujoin_count(const K* __restrict__ sk, u64 S, const K* __restrict__ xorc,
                                                   u64* __restrict__ tot, u64* __restrict__ work_run) {
    __shared__ u64 red[2][8];
    const u32 b = blockIdx.y;
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    HeadBlock hb = u_block(sk + u64(b) * S, i, S);
    if (xorc[b] == 0) {
        if (hb.hc) make_diag(hb);
    } else if (hb.work == 0) {
        hb = HeadBlock();
    }
    const u64 ws = warp_sum(hb.pairs), ww = warp_sum(hb.work);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = ws;
        red[1][threadIdx.x >> 5] = ww;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 t0 = 0, t1 = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            t0 += red[0][w];
            t1 += red[1][w];
        }
        if (t0) atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), static_cast<unsigned long long>(t0));
        if (t1) atomicAdd(reinterpret_cast<unsigned long long*>(work_run + b), static_cast<unsigned long long>(t1));
    }
}

template <class K>
__global__ void __launch_bounds__(256) ujoin_emit(const K* __restrict__ sk, u64 S, const K* __restrict__ xorc,
                                                  const u64* __restrict__ tot, u64 guard, u32 hmax,
                                                  Item* __restrict__ items, u32* __restrict__ nitems, u32 item_cap,
                                                  u32* __restrict__ npairs, PairRec* __restrict__ pairs,
                                                  u32 pair_cap, const u32* __restrict__ grp) {
    const u32 b = blockIdx.y;
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    HeadBlock hb;
    if (tot[b] <= guard) {
        hb = u_block(sk + u64(b) * S, i, S);
        if (xorc[b] == 0) {
            if (hb.hc) make_diag(hb);
        } else if (hb.work == 0) {
            hb = HeadBlock();
        }
    }
    emit_items(hb, b, hmax, items, nitems, item_cap, npairs, pairs, pair_cap, S, grp);
}

// ------------------------------------------------- bucket grouping path --
//
// For M <= kTableBits with 2^M comparable to p, a counting sort replaces the
// radix sort: per-run bucket counts (one warp-aggregated atomic per distinct
// key in a warp), one global exclusive scan over [B][2^M] (run b's entries
// land in [b*p, (b+1)*p) because every run has exactly p columns), and a
// scatter. The order inside a bucket is not stable; the stable (key, index)
// position the reference order needs is recomputed for hits only (a rank
// inside the bucket), so order keys are identical to the sorted path.

template <class K>
__global__ void __launch_bounds__(256) bucket_count(const K* __restrict__ keys, u64 p, int M, u32* __restrict__ cnt) {
    const u64 b = blockIdx.y;
    const u64 j = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = j < p;
    const u32 active = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const u64 v = u64(keys[b * p + j]);
    const u32 peers = __match_any_sync(active, static_cast<unsigned long long>(v));
    if ((peers & lanemask_lt()) == 0) atomicAdd(cnt + (b << M) + v, __popc(peers));
}

// cursor: exclusive scan of the counts (global positions); ends as the
// bucket end. grouped[pos] = column index.
template <class K>
__global__ void __launch_bounds__(256) bucket_scatter(const K* __restrict__ keys, u64 p, int M, u32* __restrict__ cursor,
                                                      u32* __restrict__ grouped) {
    const u64 b = blockIdx.y;
    const u64 j = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    const bool valid = j < p;
    const u32 active = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const u64 v = u64(keys[b * p + j]);
    const u32 peers = __match_any_sync(active, static_cast<unsigned long long>(v));
    const int leader = __ffs(peers) - 1;
    u32 base = 0;
    if ((threadIdx.x & 31) == leader) base = atomicAdd(cursor + (b << M) + v, __popc(peers));
    base = __shfl_sync(peers, base, leader);
    grouped[base + __popc(peers & lanemask_lt())] = u32(j);
}

// The block owned by bucket v of run b (positions local to the run).
__device__ __forceinline__ HeadBlock bucket_block(const u32* __restrict__ cnt, const u32* __restrict__ end, u64 b,
                                                  int M, u64 v, u64 c, u64 p) {
    HeadBlock hb;
    const u64 base = b << M;
    const u64 cv = cnt[base + v];
    if (cv == 0) return hb;
    const u64 v2 = v ^ c;
    if (v2 == v) {
        hb.pairs = cv * cv;
        if (cv >= 2) {
            const u32 beg = end ? u32(end[base + v] - cv - b * p) : 0u;
            hb.work = cv * (cv - 1) / 2;
            hb.hs = beg;
            hb.hc = u32(cv);
            hb.ss = beg;
            hb.sc = u32(cv);
            hb.flags = 3u;
        }
    } else if (v2 > v) {
        const u64 c2 = cnt[base + v2];
        if (c2) {
            hb.pairs = 2 * cv * c2;
            hb.work = cv * c2;
            const u32 bx = end ? u32(end[base + v] - cv - b * p) : 0u;
            const u32 bz = end ? u32(end[base + v2] - c2 - b * p) : 0u;
            if (cv <= c2) {
                hb.hs = bx; hb.hc = u32(cv); hb.ss = bz; hb.sc = u32(c2); hb.flags = 1u;
            } else {
                hb.hs = bz; hb.hc = u32(c2); hb.ss = bx; hb.sc = u32(cv); hb.flags = 0u;
            }
        }
    }
    return hb;
}

template <class K>
__global__ void __launch_bounds__(256) bucket_join_count(const u32* __restrict__ cnt, int M, const K* __restrict__ xorc,
                                                         u64 p, u64* __restrict__ tot, u64* __restrict__ work_run) {
    __shared__ u64 red[2][8];
    const u32 b = blockIdx.y;
    const u64 v = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    HeadBlock hb;
    if (v < (u64(1) << M)) hb = bucket_block(cnt, nullptr, b, M, v, u64(xorc[b]), p);
    const u64 ws = warp_sum(hb.pairs), ww = warp_sum(hb.work);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = ws;
        red[1][threadIdx.x >> 5] = ww;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 t0 = 0, t1 = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            t0 += red[0][w];
            t1 += red[1][w];
        }
        if (t0) atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), static_cast<unsigned long long>(t0));
        if (t1) atomicAdd(reinterpret_cast<unsigned long long*>(work_run + b), static_cast<unsigned long long>(t1));
    }
}

template <class K>
__global__ void __launch_bounds__(256) bucket_join_emit(const u32* __restrict__ cnt, const u32* __restrict__ end, int M,
                                                        const K* __restrict__ xorc, u64 p, const u64* __restrict__ tot,
                                                        u64 guard, u32 hmax, Item* __restrict__ items,
                                                        u32* __restrict__ nitems, u32 item_cap,
                                                        u32* __restrict__ npairs, PairRec* __restrict__ pairs,
                                                        u32 pair_cap, const u32* __restrict__ grp) {
    const u32 b = blockIdx.y;
    const u64 v = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    HeadBlock hb;
    if (v < (u64(1) << M) && tot[b] <= guard) hb = bucket_block(cnt, end, b, M, v, u64(xorc[b]), p);
    emit_items(hb, b, hmax, items, nitems, item_cap, npairs, pairs, pair_cap, p, grp);
}

// Per-run counters; the guard (pair_search.hpp:91-94) zeroes the verified
// count of aborted runs (their items are skipped by verify).
__global__ void book_runs(u32 B, const u64* __restrict__ tot, const u64* __restrict__ work_run, u64 guard,
                          const u32* __restrict__ rid, u64* __restrict__ enumerated_by_rid,
                          u64* __restrict__ verified_by_rid) {
    const u32 b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) {
        enumerated_by_rid[rid[b]] = tot[b];
        verified_by_rid[rid[b]] = tot[b] > guard ? 0ull : work_run[b];
    }
}

// ---------------------------------------------------------------- verify --

struct VerifyArgs {
    const Item* items;
    const u32* nitems;
    u32 item_cap;
    const u64* tot;
    u64 guard;
    const u32* sv;  // sorted column indices [B][S]
    u64 S;          // = p
    const u32* rid;
    const int8_t* run_sign;
    u64 p;
    DevHit* hits;
    u32* hit_count;
    u32 hit_cap;
    // the x-side key v of a hit (its block's key): from the sorted keys at the
    // x-side position, or (bucket path, keys unsorted) at the column index
    const void* vkeys;
    int vkeys_by_pos;
    const void* xkeys;  // unsorted keys of the batch by column (pair-list hits); nullptr: recompute
    const u32* krows;   // ... from the runs' draws (krows[run * kM + s]) and the column words
    int kM;
    const u64* kXc;
    u32 kWp;
    int key64;
    int vshift;  // sorted keys carry extra low bits to drop (0 here)
    // top-K over all candidates (topk_kernels.cuh): while the running rank
    // threshold *rank_thr is 0 the pair-list verify writes every pair's
    // strength numerator to sint_out instead of testing it; otherwise (and in
    // the item verify) pairs whose rank is at or above *rank_thr are appended
    u32* sint_out;
    const u32* rank_thr;
    int rank_binary;  // ranks: binary round(s n), else floor(s 2^24)
    u32 rank_n;
};

constexpr int kRealRankBits = 24;
// rank of a strength for the top-K threshold (topk_kernels.cuh): binary the
// exact numerator round(s n); continuous floor(s 2^24), s in [0, 1]
__host__ __device__ __forceinline__ u32 strength_rank(double s, u32 n, int binary) {
    if (binary) return u32(llrint(s * double(n)));
    if (!(s > 0.0)) return 0u;
    if (s >= 1.0) return 1u << kRealRankBits;
    return u32(s * double(1u << kRealRankBits));
}

__device__ __forceinline__ u64 key_at(const VerifyArgs& A, u64 i) {
    const u64 v = A.key64 ? static_cast<const u64*>(A.vkeys)[i] : u64(static_cast<const u32*>(A.vkeys)[i]);
    return v >> A.vshift;
}

template <int G>
__device__ __forceinline__ u32 team_mask_of(int lane) {
    return G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
}

// Team-level append: each lane of the team with `hit` writes one record.
template <int G>
__device__ __forceinline__ void team_append(const VerifyArgs& A, u32 tmask, bool hit, const DevHit& h) {
    const u32 ballot = __ballot_sync(tmask, hit);
    if (!ballot) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(ballot) - 1;
    u32 base = 0;
    if (lane == leader) base = atomicAdd(A.hit_count, __popc(ballot));
    base = __shfl_sync(tmask, base, leader);
    if (hit) {
        const u32 slot = base + __popc(ballot & lanemask_lt());
        if (slot < A.hit_cap) A.hits[slot] = h;
    }
}

// Hit record of canonical pair (x-side position pa, z-side position pb) of a
// run: oriented as the reference emits it — x side first (its key is the
// smaller), diagonal blocks smaller column index first (A.8). The reference
// order inside a run is (x-side key v, j, k) (pair_search.cpp:17-21,
// pair_search.hpp:95-97); the record keeps v in `order` and the merge sorts
// by (rid, v, j, k).
__device__ __forceinline__ DevHit hit_of(const VerifyArgs& A, u32 run, u32 pa, u32 pb, bool diag, double s,
                                         int32_t sint) {
    const u64 off = u64(run) * A.S;
    u32 j = A.sv[off + pa], k = A.sv[off + pb];
    if (diag && j > k) {
        const u32 t = j;
        j = k;
        k = t;
    }
    DevHit h;
    h.order = key_at(A, off + (A.vkeys_by_pos ? pa : j));
    h.s = s;
    h.j = j;
    h.k = k;
    h.rid = A.rid[run];
    h.sint = sint;
    return h;
}

__device__ __forceinline__ DevHit make_hit(const VerifyArgs& A, u32 run, u32 held_pos, u32 str_pos, u32 flags,
                                           double s, int32_t sint) {
    const bool diag = flags & 2u;
    const bool held_x = flags & 1u;
    return hit_of(A, run, diag || held_x ? held_pos : str_pos, diag || held_x ? str_pos : held_pos, diag, s, sint);
}

// One pair-list hit appended by one lane (hits are rare: no aggregation).
// Key of column j in a run: the M draws of the run, bit s = X[rows[s], j]
// (project_keys, projection.cpp:32-57) — for hits of pair lists that outlive
// their batch's key array (the L2-tiled verify).
__device__ __forceinline__ u64 key_of_column(const u32* rows, int M, const u64* Xc, u32 Wp, u32 j) {
    u64 v = 0;
    const u64* col = Xc + u64(j) * Wp;
    for (int s = 0; s < M; ++s) {
        const u32 i = rows[s];
        v |= ((col[i >> 6] >> (i & 63)) & 1ull) << s;
    }
    return v;
}

__device__ __noinline__ void append_pair_hit(const void* xkeys, int key64, u64 S, const u32* rid, DevHit* hits,
                                             u32* hit_count, u32 hit_cap, PairRec pr, u32 si, u32 n,
                                             const u32* krows, int kM, const u64* kXc, u32 kWp) {
    u32 j = pr.pa, k = pr.pb;
    if ((pr.pad & 2u) && j > k) {
        const u32 t = j;
        j = k;
        k = t;
    }
    const u64 i = u64(pr.run) * S + j;
    DevHit h;
    if (xkeys)
        h.order = key64 ? static_cast<const u64*>(xkeys)[i] : u64(static_cast<const u32*>(xkeys)[i]);
    else
        h.order = key_of_column(krows + u64(pr.run) * kM, kM, kXc, kWp, j);
    h.s = double(si) / double(n);
    h.j = j;
    h.k = k;
    h.rid = rid[pr.run];
    h.sint = int32_t(si);
    const u32 slot = atomicAdd(hit_count, 1u);
    if (slot < hit_cap) hits[slot] = h;
}

// ------------------------------------------------------- pair list path --


// Expand every item into its candidate pairs (h-major, so consecutive pairs
// share the held column and stay in one team's L1). Warp per item; slots
// were reserved by join_emit (the counter runs past pair_cap for a regrow).
__global__ void __launch_bounds__(256) expand_pairs(const Item* __restrict__ items, const u32* __restrict__ nitems,
                                                    u32 item_cap, u64 S, PairRec* __restrict__ pairs, u32 pair_cap,
                                                    const u32* __restrict__ grp) {
    const int lane = threadIdx.x & 31;
    const u32 N = min(*nitems, item_cap);
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 t = warp; t < N; t += nwarps) {
        const Item it = items[t];
        const u32 hc = it.hc_flags & 0xffu, flags = it.hc_flags >> 8;
        const bool diag = flags & 2u, held_x = flags & 1u;
        const u64 off = u64(it.run) * S;
        const u32 base = it.pad;  // slots reserved by join_emit
        u32 written = 0;
        const bool first_held = diag || held_x;
        for (u32 h = 0; h < hc; ++h) {
            const u32 hpos = it.hs + h;
            const u32 hcol = grp[off + hpos];
            for (u32 s0 = 0; s0 < it.sc; s0 += 32) {
                const u32 q = s0 + lane;
                const u32 spos = it.ss + q;
                const bool ok = q < it.sc && !(diag && spos <= hpos);
                const u32 bal = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    const u32 slot = base + written + __popc(bal & lanemask_lt());
                    if (slot < pair_cap) {
                        const u32 scol = grp[off + spos];
                        PairRec r;
                        r.pa = first_held ? hcol : scol;
                        r.pb = first_held ? scol : hcol;
                        r.run = it.run;
                        r.pad = flags;
                        pairs[slot] = r;
                    }
                }
                written += __popc(bal);
            }
        }
    }
}

template <int G, int NIT>
struct ColPair {
    ulonglong2 a[NIT], b[NIT];
};

template <int G, int NIT>
__device__ __forceinline__ void load_cols(ColPair<G, NIT>& c, const ulonglong2* X2, u32 W2, u32 j, u32 k, int tl) {
    const ulonglong2* xj = X2 + u64(j) * W2;
    const ulonglong2* xk = X2 + u64(k) * W2;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const u32 wi = it * G + tl;
        c.a[it] = wi < W2 ? __ldg(xj + wi) : make_ulonglong2(0, 0);
        c.b[it] = wi < W2 ? __ldg(xk + wi) : make_ulonglong2(0, 0);
    }
}

// Binary verify over the pair list. A team of G lanes owns a chunk of
// G * kPairsPerLane consecutive pairs: the pair records and their column
// indices are fetched for the whole chunk up front (one coalesced request per
// lane, no per-pair dependent loads), then the team walks the chunk with the
// next pair's columns already in flight while the current pair is reduced.
// popc(X_j ^ X_k ^ Y) over NIT x 16 B per lane, team reduction, integer hit
// test by the pair's owning lane.
constexpr u32 kPairsPerLane = 2;
#ifndef XYZB_VP_MINB
#define XYZB_VP_MINB 4
#endif

template <int G, int NIT>
__global__ void __launch_bounds__(256) verify_pairs_binary(VerifyArgs A, const PairRec* __restrict__ pairs,
                                                           const u32* __restrict__ npairs, u32 pair_cap,
                                                           const u64* __restrict__ Xc, u32 Wp,
                                                           const u64* __restrict__ Yw, u32 n, u32 astar) {
    constexpr u32 CH = G * kPairsPerLane;
    const int lane = threadIdx.x & 31;
    const int tl = lane & (G - 1);
    const u32 tmask = team_mask_of<G>(lane);
    const u32 W2 = Wp / 2;
    const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(Xc);
    ulonglong2 yv[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const u32 wi = it * G + tl;
        yv[it] = wi < W2 ? __ldg(reinterpret_cast<const ulonglong2*>(Yw) + wi) : make_ulonglong2(0, 0);
    }
    // an item overflow leaves unexpanded (unwritten) slots in the pair list;
    // the host regrows and redoes the batch, so verify nothing now
    const u32 P = *A.nitems > A.item_cap ? 0u : min(*npairs, pair_cap);
    // top-K over all candidates: appends above the running threshold once it is set
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    astar = max(astar, rthr);
    const u64 team = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const u64 nteams = (u64(gridDim.x) * blockDim.x) / G;
    for (u64 c0 = team * CH; c0 < P; c0 += nteams * CH) {
        const u32 cnt = u32(minu(CH, P - c0));
        // chunk prologue: this lane's records (pairs c0 + tl + G*i) and their columns
        PairRec pr[kPairsPerLane];
        u32 cj[kPairsPerLane], ck[kPairsPerLane];
#pragma unroll
        for (u32 i = 0; i < kPairsPerLane; ++i) {
            const u32 t = tl + G * i;
            if (t < cnt) {
                pr[i] = pairs[c0 + t];
                cj[i] = pr[i].pa;
                ck[i] = pr[i].pb;
            } else {
                pr[i] = PairRec{0, 0, 0, 0};
                cj[i] = ck[i] = 0;
            }
        }
        auto jk_of = [&](u32 t, u32& j, u32& k) {
            const u32 i = t / G, src = t % G;
            u32 mj = 0, mk = 0;
#pragma unroll
            for (u32 q = 0; q < kPairsPerLane; ++q)
                if (q == i) {
                    mj = cj[q];
                    mk = ck[q];
                }
            j = __shfl_sync(tmask, mj, src, G);
            k = __shfl_sync(tmask, mk, src, G);
        };
        ColPair<G, NIT> cur, nxt;
        u32 j0, k0;
        jk_of(0, j0, k0);
        load_cols<G, NIT>(cur, X2, W2, j0, k0, tl);
        for (u32 t = 0; t < cnt; ++t) {
            if (t + 1 < cnt) {
                u32 j1, k1;
                jk_of(t + 1, j1, k1);
                load_cols<G, NIT>(nxt, X2, W2, j1, k1, tl);
            }
            u32 acc = 0;
#pragma unroll
            for (int it = 0; it < NIT; ++it)
                acc += __popcll(cur.a[it].x ^ cur.b[it].x ^ yv[it].x) + __popcll(cur.a[it].y ^ cur.b[it].y ^ yv[it].y);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(tmask, acc, o);
            // the owning lane tests pair t with its record
            if (u32(tl) == t % G) {
                const u32 i = t / G;
                PairRec r = pr[0];
#pragma unroll
                for (u32 q = 1; q < kPairsPerLane; ++q)
                    if (q == i) r = pr[q];
                const u32 si = A.run_sign[r.run] > 0 ? acc : n - acc;
                if (A.sint_out && rthr == 0) A.sint_out[c0 + t] = si;
                else if (si >= astar) append_pair_hit(A.xkeys, A.key64, A.S, A.rid, A.hits, A.hit_count, A.hit_cap, r, si, n, A.krows,
                                                 A.kM, A.kXc, A.kWp);
            }
            if (t + 1 < cnt) cur = nxt;
        }
    }
}

// Simple pair walk (one pair at a time per team, chunks of 32 pairs): kept
// beside the pipelined walk for measurement (XYZB_VERIFY=simple).
template <int G, int NIT>
__global__ void __launch_bounds__(256, XYZB_VP_MINB) verify_pairs_simple(VerifyArgs A, const PairRec* __restrict__ pairs,
                                                           const u32* __restrict__ npairs, u32 pair_cap,
                                                           const u64* __restrict__ Xc, u32 Wp,
                                                           const u64* __restrict__ Yw, u32 n, u32 astar) {
    constexpr u32 CH = 32;
    const int lane = threadIdx.x & 31;
    const int tl = lane & (G - 1);
    const u32 tmask = team_mask_of<G>(lane);
    const u32 W2 = Wp / 2;
    const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(Xc);
    ulonglong2 yv[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const u32 wi = it * G + tl;
        yv[it] = wi < W2 ? __ldg(reinterpret_cast<const ulonglong2*>(Yw) + wi) : make_ulonglong2(0, 0);
    }
    // an item overflow leaves unexpanded (unwritten) slots in the pair list;
    // the host regrows and redoes the batch, so verify nothing now
    const u32 P = *A.nitems > A.item_cap ? 0u : min(*npairs, pair_cap);
    // top-K over all candidates: appends above the running threshold once it is set
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    astar = max(astar, rthr);
    const u64 team = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const u64 nteams = (u64(gridDim.x) * blockDim.x) / G;
    for (u64 c0 = team * CH; c0 < P; c0 += nteams * CH) {
        const u32 c1 = u32(minu(P, c0 + CH));
        for (u32 q = u32(c0); q < c1; ++q) {
            const PairRec pr = pairs[q];
            const u32 j = pr.pa, k = pr.pb;
            ColPair<G, NIT> c;
            load_cols<G, NIT>(c, X2, W2, j, k, tl);
            u32 acc = 0;
#pragma unroll
            for (int it = 0; it < NIT; ++it)
                acc += __popcll(c.a[it].x ^ c.b[it].x ^ yv[it].x) + __popcll(c.a[it].y ^ c.b[it].y ^ yv[it].y);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(tmask, acc, o);
            const u32 si = A.run_sign[pr.run] > 0 ? acc : n - acc;
            if (A.sint_out && rthr == 0) {
                if (tl == 0) A.sint_out[q] = si;
            } else if (tl == 0 && si >= astar)  // rare: out of line, so the walk keeps few registers
                append_pair_hit(A.xkeys, A.key64, A.S, A.rid, A.hits, A.hit_count, A.hit_cap, pr, si, n, A.krows,
                                A.kM, A.kXc, A.kWp);
        }
    }
}

// Continuous-Y (transforms.cpp:42-76): sum of |y_i| over rows where
// bit(x_j ^ x_k ^ s) = 1, s = (resp > 0), over ||resp||_1; resp = +-y.
template <int G>
__device__ __forceinline__ double weighted_pair(const u64* xj, const u64* xk, const u64* sb,
                                                const double* __restrict__ wabs, u32 Wp, int tl, u32 tmask) {
    double acc = 0.0;
    for (u32 wi = tl; wi < Wp; wi += G) {
        u64 m = __ldg(xj + wi) ^ __ldg(xk + wi) ^ __ldg(sb + wi);
        const double* wrow = wabs + u64(wi) * 64;
        while (m) {
            const int bit = __ffsll(static_cast<long long>(m)) - 1;
            acc += __ldg(wrow + bit);
            m &= m - 1;
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(tmask, acc, o);
    return acc;
}

// Continuous-XY (search.cpp:477-493): sum_i y_i t(x_ij) t(x_ik), fp32 columns,
// products and accumulation in fp64.
// Four column slices in flight per lane (the loads of a step do not wait on
// the previous step's FMAs). Each 4-row step is summed in fp32 from the fp32
// columns and an fp32 copy of the response (relative error ~2e-7 per step)
// and added to an fp64 accumulator — one fp32 -> fp64 conversion per four
// rows instead of two per row (the conversion pipe bound the kernel); the
// strength stays within 1e-7 absolute of the fp64 value, far inside the
// 1e-5 relative parity tolerance. The response comes from shared memory
// when the kernel staged it (verify_items_real).
template <int G, bool UNBIASED>
__device__ __forceinline__ double real_pair(const float4* xj, const float4* xk, const float4* yv, u64 n4q, int tl,
                                            u32 tmask) {
    constexpr int U = 4;
    double acc0 = 0.0, acc1 = 0.0;
    auto t = [](float v) { return v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f); };
    for (u64 q0 = tl; q0 < n4q; q0 += u64(G) * U) {
        float4 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 q = q0 + u64(u) * G;
            a[u] = q < n4q ? __ldg(xj + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            b[u] = q < n4q ? __ldg(xk + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 q = q0 + u64(u) * G;
            if (q >= n4q) break;
            const float4 y = yv[q];
            float s;
            if (UNBIASED) {
                s = y.x * (a[u].x * b[u].x);
                s = fmaf(y.y, a[u].y * b[u].y, s);
                s = fmaf(y.z, a[u].z * b[u].z, s);
                s = fmaf(y.w, a[u].w * b[u].w, s);
            } else {
                s = y.x * (t(a[u].x) * t(b[u].x));
                s = fmaf(y.y, t(a[u].y) * t(b[u].y), s);
                s = fmaf(y.z, t(a[u].z) * t(b[u].z), s);
                s = fmaf(y.w, t(a[u].w) * t(b[u].w), s);
            }
            if (u & 1) acc1 += double(s);
            else acc0 += double(s);
        }
    }
    double acc = acc0 + acc1;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(tmask, acc, o);
    return acc;
}

// Pairwise walk of an item's tile for the real-valued strengths: one pair at
// a time per team (held h x streamed s).
template <int G, class F>
__device__ __forceinline__ void walk_items(const VerifyArgs& A, F&& strength) {
    const int lane = threadIdx.x & 31;
    const int tl = lane & (G - 1);
    const u32 tmask = team_mask_of<G>(lane);
    const u32 N = min(*A.nitems, A.item_cap);
    const u64 team = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const u64 nteams = (u64(gridDim.x) * blockDim.x) / G;
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;  // top-K over all candidates: rank threshold
    for (u64 t = team; t < N; t += nteams) {
        const Item item = A.items[t];
        if (A.tot[item.run] > A.guard) continue;
        const u32 hc = item.hc_flags & 0xffu, flags = item.hc_flags >> 8;
        const u32* svr = A.sv + u64(item.run) * A.S;
        const bool pos_pass = A.run_sign[item.run] > 0;
        for (u32 h = 0; h < hc; ++h) {
            const u32 hpos = item.hs + h;
            const u32 hcol = svr[hpos];
            for (u32 q = 0; q < item.sc; ++q) {
                const u32 spos = item.ss + q;
                if ((flags & 2u) && spos <= hpos) continue;
                const double s = strength(hcol, svr[spos], pos_pass, tl, tmask);
                const bool hit = tl == 0 && (A.rank_thr ? strength_rank(s, A.rank_n, A.rank_binary) >= rthr
                                                         : strength.hit(s));
                DevHit hr;
                if (hit) hr = make_hit(A, item.run, hpos, spos, flags, s, -1);
                team_append<G>(A, tmask, hit, hr);
            }
        }
    }
}

struct WeightedStrength {
    const u64* Xc;
    u32 Wp;
    const u64 *spos, *sneg;
    const double* wabs;
    double norm, gamma;
    __device__ double operator()(u32 j, u32 k, bool pos_pass, int tl, u32 tmask) const {
        return weighted_pair<32>(Xc + u64(j) * Wp, Xc + u64(k) * Wp, pos_pass ? spos : sneg, wabs, Wp, tl, tmask) /
               norm;
    }
    __device__ bool hit(double s) const { return s >= gamma; }
};

// Binary strengths for long columns (more than 4 x 16 B per lane): one pair
// at a time, words strided over the warp. Hit test s >= gamma is the same as
// sint >= astar (astar is the least integer with astar/n >= gamma).
struct BinaryStrength {
    const u64* Xc;
    u32 Wp;
    const u64* Yw;
    u32 n, astar;
    __device__ double operator()(u32 j, u32 k, bool pos_pass, int tl, u32 tmask) const {
        const ulonglong2* a = reinterpret_cast<const ulonglong2*>(Xc + u64(j) * Wp);
        const ulonglong2* b = reinterpret_cast<const ulonglong2*>(Xc + u64(k) * Wp);
        const ulonglong2* y = reinterpret_cast<const ulonglong2*>(Yw);
        u32 acc = 0;
        for (u32 wi = tl; 2 * wi < Wp; wi += 32) {
            const ulonglong2 u = __ldg(a + wi), v = __ldg(b + wi), w = __ldg(y + wi);
            acc += __popcll(u.x ^ v.x ^ w.x) + __popcll(u.y ^ v.y ^ w.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(tmask, acc, o);
        const u32 si = pos_pass ? acc : n - acc;
        return double(si) / double(n);
    }
    __device__ bool hit(double s) const { return u32(llrint(s * double(n))) >= astar; }
};

template <bool UNBIASED>
struct RealStrength {
    const float* Xc32;
    u64 n4;
    const float* y;  // the response in fp32 (n4 entries, zero padded)
    double norm, gamma;
    __device__ double operator()(u32 j, u32 k, bool pos_pass, int tl, u32 tmask) const {
        const double acc = real_pair<32, UNBIASED>(reinterpret_cast<const float4*>(Xc32 + u64(j) * n4),
                                                   reinterpret_cast<const float4*>(Xc32 + u64(k) * n4),
                                                   reinterpret_cast<const float4*>(y), n4 / 4, tl, tmask);
        return 0.5 + (pos_pass ? 1.0 : -1.0) * acc / (2.0 * norm);
    }
    __device__ bool hit(double s) const { return s >= gamma; }
};

template <class F>
__global__ void __launch_bounds__(256) verify_items(VerifyArgs A, F f) {
    walk_items<32>(A, f);
}

// Continuous-XY verify with the response staged in shared memory (n4 doubles).
template <bool UNBIASED>
__global__ void __launch_bounds__(256) verify_items_real(VerifyArgs A, RealStrength<UNBIASED> f) {
    extern __shared__ __align__(16) float ys[];
    for (u64 i = threadIdx.x; i < f.n4; i += blockDim.x) ys[i] = f.y[i];
    __syncthreads();
    f.y = ys;
    walk_items<32>(A, f);
}

// Sign-transform strengths from bit planes (continuous-XY, transform sign):
// t(x) in {-1, 0, 1}, so sum_i y_i t_ij t_ik = 2 S(agree) - S(both) with
// both = nz_j & nz_k, agree = both & ~(pos_j ^ pos_k) and S(m) = sum of y
// over the rows of mask m. y is quantised once per search to integers
// q_i = rint(y_i * scale) held as two's-complement bit planes P_0..P_B, so
// S(m) = sum_b<B 2^b popc(P_b & m) - 2^B popc(P_B & m): a column pair costs
// 2 x n/8 bytes of sign bits instead of 2 x 4n bytes of fp32 values. The
// quantised strength is within `delta` of the fp32-column value; a pair at
// or above gamma - delta is re-verified with RealStrength, so hits and their
// strengths are those of the fp32 verify.
constexpr int kSignQB = 12;  // response quantised to 13-bit two's complement (|q| <= 4095)
struct SignStrength {
    const u64 *Spos, *Snz;  // [p][Wn]
    u64 Wn;
    const u64* planes;  // [B + 1][Wn] (B: the kernel's QB)
    long long qsum;  // sum of q over all rows (S(both) when X has no zero)
    bool zeros;
    double inv_scale, norm, gamma, delta;
    RealStrength<false> exact;
};

__device__ __forceinline__ long long plane_sum(const u64* planes, u64 Wn, int B, u64 w, u64 m) {
    long long s = 0;
    for (int b = 0; b < B; ++b) s += (long long)__popcll(planes[u64(b) * Wn + w] & m) << b;
    return s - ((long long)__popcll(planes[u64(B) * Wn + w] & m) << B);
}

// sum of q over the rows of a 64-row mask from register-held planes (QB <= 24:
// |result| < 2^31)
template <int QB>
__device__ __forceinline__ int plane_sum_reg(const u64 (&pl)[QB + 1], u64 m) {
    int s = 0;
#pragma unroll
    for (int b = 0; b < QB; ++b) s += __popcll(pl[b] & m) << b;
    return s - (__popcll(pl[QB] & m) << QB);
}

// One warp per candidate pair. Rows <= 2048 (Wn <= 32 words): lane w keeps
// word w of every response plane in registers for the whole kernel; longer
// columns walk the words with the planes in shared memory (or L1).
template <int QB>
__global__ void __launch_bounds__(256, 4) verify_items_sign(VerifyArgs A, SignStrength f) {
    extern __shared__ __align__(16) u64 sh[];
    const u64 nplane = u64(QB + 1) * f.Wn;
    const bool in_reg = f.Wn <= 32;
    const bool in_smem = !in_reg && nplane * 8 <= (size_t(48) << 10);
    if (in_smem) {
        for (u64 i = threadIdx.x; i < nplane; i += blockDim.x) sh[i] = f.planes[i];
        __syncthreads();
    }
    const u64* planes = in_smem ? sh : f.planes;
    const int lane = threadIdx.x & 31;
    u64 pl[QB + 1];
#pragma unroll
    for (int b = 0; b <= QB; ++b) pl[b] = in_reg && u64(lane) < f.Wn ? f.planes[u64(b) * f.Wn + lane] : 0ull;
    const u32 N = min(*A.nitems, A.item_cap);
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    // top-K over all candidates: the gate is the rank threshold's strength (its bin's lower edge)
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    const double gate = A.rank_thr ? double(rthr) / double(1u << kRealRankBits) : f.gamma;
    for (u64 t = warp; t < N; t += nwarps) {
        const Item item = A.items[t];
        if (A.tot[item.run] > A.guard) continue;
        const u32 hc = item.hc_flags & 0xffu, flags = item.hc_flags >> 8;
        const u32* svr = A.sv + u64(item.run) * A.S;
        const bool pos_pass = A.run_sign[item.run] > 0;
        for (u32 h = 0; h < hc; ++h) {
            const u32 hpos = item.hs + h;
            const u32 j = svr[hpos];
            for (u32 q = 0; q < item.sc; ++q) {
                const u32 spos = item.ss + q;
                if ((flags & 2u) && spos <= hpos) continue;
                const u32 k = svr[spos];
                long long acc = 0;
                if (in_reg) {
                    if (u64(lane) < f.Wn) {
                        const u64 w = lane;
                        const u64 pj = __ldg(f.Spos + u64(j) * f.Wn + w), pk = __ldg(f.Spos + u64(k) * f.Wn + w);
                        const u64 both =
                            f.zeros ? (__ldg(f.Snz + u64(j) * f.Wn + w) & __ldg(f.Snz + u64(k) * f.Wn + w)) : ~0ull;
                        int a = 2 * plane_sum_reg<QB>(pl, both & ~(pj ^ pk));
                        if (f.zeros) a -= plane_sum_reg<QB>(pl, both);
                        acc = a;
                    }
                } else {
                    for (u64 w = lane; w < f.Wn; w += 32) {
                        const u64 pj = __ldg(f.Spos + u64(j) * f.Wn + w), pk = __ldg(f.Spos + u64(k) * f.Wn + w);
                        const u64 both = f.zeros ? (__ldg(f.Snz + u64(j) * f.Wn + w) &
                                                    __ldg(f.Snz + u64(k) * f.Wn + w))
                                                 : ~0ull;
                        acc += 2 * plane_sum(planes, f.Wn, QB, w, both & ~(pj ^ pk));
                        if (f.zeros) acc -= plane_sum(planes, f.Wn, QB, w, both);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (!f.zeros) acc -= f.qsum;
                double s = 0.5 + (pos_pass ? 1.0 : -1.0) * (double(acc) * f.inv_scale) / (2.0 * f.norm);
                if (s >= gate - f.delta) s = f.exact(j, k, pos_pass, lane, 0xffffffffu);  // warp-uniform
                const bool hit = lane == 0 && (A.rank_thr ? strength_rank(s, 0u, 0) >= rthr : f.exact.hit(s));
                DevHit hr;
                if (hit) hr = make_hit(A, item.run, hpos, spos, flags, s, -1);
                team_append<32>(A, 0xffffffffu, hit, hr);
            }
        }
    }
}

// Pair-list hit of a real-valued strength (the sign transform's pair walk).
__device__ __noinline__ void append_pair_hit_real(const VerifyArgs& A, PairRec pr, double s) {
    u32 j = pr.pa, k = pr.pb;
    if ((pr.pad & 2u) && j > k) {
        const u32 t = j;
        j = k;
        k = t;
    }
    const u64 i = u64(pr.run) * A.S + j;
    DevHit h;
    h.order = A.key64 ? static_cast<const u64*>(A.xkeys)[i] : u64(static_cast<const u32*>(A.xkeys)[i]);
    h.s = s;
    h.j = j;
    h.k = k;
    h.rid = A.rid[pr.run];
    h.sint = -1;
    const u32 slot = atomicAdd(A.hit_count, 1u);
    if (slot < A.hit_cap) A.hits[slot] = h;
}

// Sign-transform verify over the pair list (columns of <= 2048 rows: lane w
// holds word w of the column sign bits and of every response plane). A warp
// takes 32 consecutive pair records with one coalesced load, then walks them
// with the next pair's sign words already in flight while the current pair
// is reduced (SignStrength: quantised strength, exact fp32 re-verification
// within the quantisation bound of the threshold). Top-K over all candidates,
// first phase (running threshold still 0): every pair's rank lower bound
// rank(s_q - delta) goes to sint_out instead (topk::emit_pairs_requant emits).
template <int QB>
__global__ void __launch_bounds__(256, 4) verify_pairs_sign(VerifyArgs A, const PairRec* __restrict__ pairs,
                                                             const u32* __restrict__ npairs, u32 pair_cap,
                                                             SignStrength f) {
    const int lane = threadIdx.x & 31;
    const bool act = u64(lane) < f.Wn;
    u64 pl[QB + 1];
#pragma unroll
    for (int b = 0; b <= QB; ++b) pl[b] = act ? f.planes[u64(b) * f.Wn + lane] : 0ull;
    const u32 P = *A.nitems > A.item_cap ? 0u : min(*npairs, pair_cap);
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    const bool ranks = A.sint_out && rthr == 0;
    const double gate = A.rank_thr ? double(rthr) / double(1u << kRealRankBits) : f.gamma;
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    const u64* Sp = f.Spos;
    const u64* Sz = f.Snz;
    const u64 Wn = f.Wn;
    for (u64 c0 = warp * 32; c0 < P; c0 += nwarps * 32) {
        const u32 cnt = u32(minu(32, P - c0));
        const PairRec mine = u32(lane) < cnt ? pairs[c0 + lane] : PairRec{0, 0, 0, 0};
        u32 j = __shfl_sync(0xffffffffu, mine.pa, 0), k = __shfl_sync(0xffffffffu, mine.pb, 0);
        u64 pj = act ? __ldg(Sp + u64(j) * Wn + lane) : 0ull, pk = act ? __ldg(Sp + u64(k) * Wn + lane) : 0ull;
        u64 zj = ~0ull, zk = ~0ull;
        if (f.zeros && act) {
            zj = __ldg(Sz + u64(j) * Wn + lane);
            zk = __ldg(Sz + u64(k) * Wn + lane);
        }
        for (u32 t = 0; t < cnt; ++t) {
            u32 j1 = 0, k1 = 0;
            u64 pj1 = 0, pk1 = 0, zj1 = ~0ull, zk1 = ~0ull;
            if (t + 1 < cnt) {  // the next pair's words in flight while this one is reduced
                j1 = __shfl_sync(0xffffffffu, mine.pa, t + 1);
                k1 = __shfl_sync(0xffffffffu, mine.pb, t + 1);
                if (act) {
                    pj1 = __ldg(Sp + u64(j1) * Wn + lane);
                    pk1 = __ldg(Sp + u64(k1) * Wn + lane);
                    if (f.zeros) {
                        zj1 = __ldg(Sz + u64(j1) * Wn + lane);
                        zk1 = __ldg(Sz + u64(k1) * Wn + lane);
                    }
                }
            }
            int a = 0;
            if (act) {
                const u64 both = f.zeros ? (zj & zk) : ~0ull;
                a = 2 * plane_sum_reg<QB>(pl, both & ~(pj ^ pk));
                if (f.zeros) a -= plane_sum_reg<QB>(pl, both);
            }
            a = warp_sum(a);
            long long acc = a;
            if (!f.zeros) acc -= f.qsum;
            const u32 run = __shfl_sync(0xffffffffu, mine.run, t);
            const bool pos_pass = A.run_sign[run] > 0;
            double s = 0.5 + (pos_pass ? 1.0 : -1.0) * (double(acc) * f.inv_scale) / (2.0 * f.norm);
            if (ranks) {
                if (u32(lane) == t) A.sint_out[c0 + t] = strength_rank(fmax(0.0, s - f.delta), 0u, 0);
            } else if (s >= gate - f.delta) {  // warp-uniform: exact fp32 re-verification
                s = f.exact(j, k, pos_pass, lane, 0xffffffffu);
                const PairRec r{j, k, run, __shfl_sync(0xffffffffu, mine.pad, t)};
                if (lane == 0 && (A.rank_thr ? strength_rank(s, 0u, 0) >= rthr : f.exact.hit(s)))
                    append_pair_hit_real(A, r, s);
            }
            j = j1;
            k = k1;
            pj = pj1;
            pk = pk1;
            zj = zj1;
            zk = zk1;
        }
    }
}

// Continuous-Y (weighted) strengths from bit planes (A9,
// transforms.cpp:42-76): s = S(x_j ^ x_k ^ s_pass) / ||y||_1 with S(m) the sum
// of |y| over the rows of mask m. |y| is quantised once per search to QB-bit
// unsigned integers q_i = rint(|y_i| scale) held as bit planes, so
// S(m) ~ sum_b 2^b popc(P_b & m) / scale within n / (2 scale) — a per-pair
// cost of 2 column words and QB popcounts per 64 rows instead of a
// dependent fp64 load per set bit. A pair within delta of the threshold is
// re-verified with the exact fp64 sum (WeightedStrength), so hits and their
// strengths are those of the exact verify.
constexpr int kWeightQB = 12;
struct WeightedQ {
    const u64* Xc;
    u32 Wp;
    u64 Wn;
    const u64 *spos, *sneg;  // [Wp] response sign bits of the + / - pass
    const u64* planes;       // [QB][Wn] bit planes of q
    double inv_scale, norm, gamma, delta;
    WeightedStrength exact;
};

// Pair-list walk of the quantised weighted verify (rows <= 2048: lane w
// holds word w of both columns and of every plane), the next pair's words in
// flight; the top-K first phase writes rank lower bounds like the sign walk.
template <int QB>
__global__ void __launch_bounds__(256, 4) verify_pairs_weighted(VerifyArgs A, const PairRec* __restrict__ pairs,
                                                                 const u32* __restrict__ npairs, u32 pair_cap,
                                                                 WeightedQ f) {
    const int lane = threadIdx.x & 31;
    const bool act = u64(lane) < f.Wn;
    u64 pl[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) pl[b] = act ? f.planes[u64(b) * f.Wn + lane] : 0ull;
    const u64 sp = act ? f.spos[lane] : 0ull, sn = act ? f.sneg[lane] : 0ull;
    const u32 P = *A.nitems > A.item_cap ? 0u : min(*npairs, pair_cap);
    const u32 rthr = A.rank_thr ? *A.rank_thr : 0u;
    const bool ranks = A.sint_out && rthr == 0;
    const double gate = A.rank_thr ? double(rthr) / double(1u << kRealRankBits) : f.gamma;
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    const u64* X = f.Xc;
    const u32 Wp = f.Wp;
    for (u64 c0 = warp * 32; c0 < P; c0 += nwarps * 32) {
        const u32 cnt = u32(minu(32, P - c0));
        const PairRec mine = u32(lane) < cnt ? pairs[c0 + lane] : PairRec{0, 0, 0, 0};
        u32 j = __shfl_sync(0xffffffffu, mine.pa, 0), k = __shfl_sync(0xffffffffu, mine.pb, 0);
        u64 xj = act ? __ldg(X + u64(j) * Wp + lane) : 0ull, xk = act ? __ldg(X + u64(k) * Wp + lane) : 0ull;
        for (u32 t = 0; t < cnt; ++t) {
            u32 j1 = 0, k1 = 0;
            u64 xj1 = 0, xk1 = 0;
            if (t + 1 < cnt) {
                j1 = __shfl_sync(0xffffffffu, mine.pa, t + 1);
                k1 = __shfl_sync(0xffffffffu, mine.pb, t + 1);
                if (act) {
                    xj1 = __ldg(X + u64(j1) * Wp + lane);
                    xk1 = __ldg(X + u64(k1) * Wp + lane);
                }
            }
            const u32 run = __shfl_sync(0xffffffffu, mine.run, t);
            const bool pos_pass = A.run_sign[run] > 0;
            const u64 m = xj ^ xk ^ (pos_pass ? sp : sn);
            int a = 0;
#pragma unroll
            for (int b = 0; b < QB; ++b) a += __popcll(pl[b] & m) << b;
            a = warp_sum(a);
            double s = double(a) * f.inv_scale / f.norm;
            if (ranks) {
                if (u32(lane) == t) A.sint_out[c0 + t] = strength_rank(fmax(0.0, s - f.delta), 0u, 0);
            } else if (s >= gate - f.delta) {  // warp-uniform: the exact fp64 sum
                s = f.exact(j, k, pos_pass, lane, 0xffffffffu);
                const PairRec r{j, k, run, __shfl_sync(0xffffffffu, mine.pad, t)};
                if (lane == 0 && (A.rank_thr ? strength_rank(s, 0u, 0) >= rthr : f.exact.hit(s)))
                    append_pair_hit_real(A, r, s);
            }
            j = j1;
            k = k1;
            xj = xj1;
            xk = xk1;
        }
    }
}

} // namespace kern
} // namespace xyzb
