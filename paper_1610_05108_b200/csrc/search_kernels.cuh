// Device kernels of one batch of xyz runs (sm_100a).
//
//   transpose_bits   column-major packed X -> row planes (once per dataset)
//   project_bits     M-bit keys of every column for every run of the batch
//                    (project_keys, projection.cpp:32-57) + the per-run XOR
//                    constant c that turns x-keys into z-keys (A.3)
//   head_table       direct-address table key -> first sorted position
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
    u64 order;     // rid * p^2 + pos_first * p + pos_second  (A.5 order inside a run)
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

// ---------------------------------------------------------------- layout --

// Xc: u64 [p][Wp] column-major words -> Xr: u32 [n][P32] row planes, bit
// (j & 31) of word j >> 5 of row i is X_ij. One warp per (32 columns, word):
// lane l holds word w of column 32c+l; ballot over bit b gives row 64w+b.
__global__ void transpose_bits(const u64* __restrict__ Xc, u64 Wp, u64 W, u64 n, u64 p, u64 P32,
                               u32* __restrict__ Xr) {
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const u64 total = P32 * W;
    if (warp >= total) return;
    const u64 c = warp / W, w = warp % W;
    const u64 col = c * 32 + lane;
    const u64 word = col < p ? Xc[col * Wp + w] : 0ull;
#pragma unroll 8
    for (int b = 0; b < 64; ++b) {
        const u32 bits = __ballot_sync(0xffffffffu, (word >> b) & 1ull);
        const u64 row = w * 64 + b;
        if (lane == (b & 31) && row < n) Xr[row * P32 + c] = bits;
    }
}

// --------------------------------------------------------------- project --

template <class K>
__device__ __forceinline__ K key_mask(int m) {
    return m >= int(sizeof(K) * 8) ? ~K(0) : ((K(1) << m) - 1);
}

// keys[b][j] = sum_s bit(X[rows[b][s], j]) << s; xorc[b] = c of the run.
// Warps read one row-plane word per s for 32 consecutive columns (broadcast).
template <class K>
__global__ void __launch_bounds__(256) project_bits(const u32* __restrict__ Xr, u64 P32, u64 p,
                                                    const u32* __restrict__ rows, int M,
                                                    const u64* __restrict__ ykey_bits,
                                                    const int8_t* __restrict__ run_sign, K* __restrict__ keys,
                                                    K* __restrict__ xorc) {
    __shared__ u32 srow[64];
    const u64 b = blockIdx.y;
    if (threadIdx.x < M) srow[threadIdx.x] = rows[b * M + threadIdx.x];
    __syncthreads();
    const u64 j = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < p) {
        const u32* base = Xr + (j >> 5);
        const int sh = int(j & 31);
        K key = 0;
#pragma unroll 8
        for (int s = 0; s < M; ++s) {
            const u32 w = __ldg(base + u64(srow[s]) * P32);
            key |= K((w >> sh) & 1u) << s;
        }
        keys[b * p + j] = key;
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        const int lane = threadIdx.x;
        u64 yk = 0;
        for (int s0 = 0; s0 < M; s0 += 32) {
            const int s = s0 + lane;
            int bit = 0;
            if (s < M) {
                const u32 r = srow[s];
                bit = int((ykey_bits[r >> 6] >> (r & 63)) & 1ull);
            }
            yk |= u64(__ballot_sync(0xffffffffu, bit)) << s0;
        }
        if (lane == 0) {
            const K mask = key_mask<K>(M);
            const K ykk = K(yk) & mask;
            // z+ = ~(x ^ y) & mask = x ^ (~y & mask); z- = x ^ y  (A.3)
            xorc[b] = run_sign[b] > 0 ? K(~ykk & mask) : ykk;
        }
    }
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

// Direct-address head table for M <= kTableBits: table[b][key] = first sorted
// position of key in run b. Never cleared: a lookup is trusted only if the
// stored position holds the key (stale entries from earlier batches fail it).
constexpr int kTableBits = 22;

template <class K>
__global__ void __launch_bounds__(256) head_table(const K* __restrict__ sk, u64 S, int M, u32* __restrict__ table) {
    const u32 b = blockIdx.y;
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= S) return;
    const K* a = sk + u64(b) * S;
    const K v = a[i];
    if (i == 0 || a[i - 1] != v) table[(u64(b) << M) + u64(v)] = u32(i);
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

// Pass 2: canonical work items of the runs the guard keeps. Item t of a block:
// held chunk t / nsc (<= hmax columns), streamed chunk t % nsc (<=
// kStreamChunk columns), so one big group cannot serialise on one team. The
// item counter keeps counting past `item_cap` so the host can regrow.
template <class K>
__global__ void __launch_bounds__(256) join_emit(const K* __restrict__ sk, u64 S, int M, const K* __restrict__ xorc,
                                                 const u32* __restrict__ table, const u64* __restrict__ tot,
                                                 u64 guard, u32 hmax, Item* __restrict__ items,
                                                 u32* __restrict__ nitems, u32 item_cap,
                                                 u32* __restrict__ npairs) {
    const u32 b = blockIdx.y;
    const bool aborted = tot[b] > guard;
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    HeadBlock hb;
    if (!aborted) hb = head_block(sk + u64(b) * S, i, S, M, xorc[b], table, b);
    u32 nsc = 1, nemit = 0;
    if (hb.work) {
        const bool diag = hb.flags & 2u;
        const u32 slen = diag ? hb.hc - 1 : hb.sc;
        const u32 hlen = diag ? hb.hc - 1 : hb.hc;  // the last diagonal column has no later partner
        nsc = (slen + kStreamChunk - 1) / kStreamChunk;
        nemit = (hlen + hmax - 1) / hmax * nsc;
    }
    // candidate pairs of this head (the diagonal counts only later positions)
    const u32 npair = u32(hb.work);
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
    const u32 wtot = __shfl_sync(0xffffffffu, incl, 31);
    const u32 ptot = __shfl_sync(0xffffffffu, pincl, 31);
    u32 base = 0, pbase = 0;
    if (lane == 31 && wtot) {
        base = atomicAdd(nitems, wtot);
        if (npairs) pbase = atomicAdd(npairs, ptot);
    }
    base = __shfl_sync(0xffffffffu, base, 31) + incl - nemit;
    u32 poff = __shfl_sync(0xffffffffu, pbase, 31) + pincl - npair;  // this head's first pair slot
    const bool diag = hb.flags & 2u;
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
};

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

__device__ __forceinline__ DevHit make_hit(const VerifyArgs& A, u32 run, u32 held_pos, u32 str_pos, u32 flags,
                                           double s, int32_t sint) {
    const u32* svr = A.sv + u64(run) * A.S;
    u32 pa, pb;  // x-side position, z-side position
    if (flags & 2u) {
        pa = min(held_pos, str_pos);
        pb = max(held_pos, str_pos);
    } else if (flags & 1u) {
        pa = held_pos;
        pb = str_pos;
    } else {
        pa = str_pos;
        pb = held_pos;
    }
    DevHit h;
    const u32 r = A.rid[run];
    h.order = (u64(r) * A.p + pa) * A.p + pb;
    h.s = s;
    h.j = svr[pa];  // x side first: its key v < v^c; diagonal: smaller index first (A.8)
    h.k = svr[pb];
    h.rid = r;
    h.sint = sint;
    return h;
}

// Binary: agree = popc(X_j ^ X_k ^ Y) over the padded words (padding is 0 in
// X and Y, packed_matrix.cpp:29-35); pass +1 strength agree/n, pass -1
// (n-agree)/n (search.cpp:25-36,347-349). Integer hit test sint >= astar.
// A team of G lanes owns one item: its <= kHeld held columns (pre-XORed with
// Y) stay in registers, each streamed column is read once and compared with
// all of them. Lane chunk `it` covers 16 B at ulonglong2 index it*G + lane.
template <int G, int NIT, int H>
__global__ void __launch_bounds__(256) verify_binary(VerifyArgs A, const u64* __restrict__ Xc, u32 Wp,
                                                     const u64* __restrict__ Yw, u32 n, u32 astar) {
    const int lane = threadIdx.x & 31;
    const int tl = lane & (G - 1);
    const u32 tmask = team_mask_of<G>(lane);
    const u32 W2 = Wp / 2;  // ulonglong2 per column
    ulonglong2 yv[NIT];
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const u32 wi = it * G + tl;
        yv[it] = wi < W2 ? __ldg(reinterpret_cast<const ulonglong2*>(Yw) + wi) : make_ulonglong2(0, 0);
    }
    const u32 N = min(*A.nitems, A.item_cap);
    const u64 team = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const u64 nteams = (u64(gridDim.x) * blockDim.x) / G;
    const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(Xc);
    for (u64 t = team; t < N; t += nteams) {
        const Item item = A.items[t];
        if (A.tot[item.run] > A.guard) continue;  // aborted run: nothing is evaluated
        const u32 hc = item.hc_flags & 0xffu, flags = item.hc_flags >> 8;
        const u32* svr = A.sv + u64(item.run) * A.S;
        const bool pos_pass = A.run_sign[item.run] > 0;
        ulonglong2 hx[H][NIT];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const u32 col = h < int(hc) ? svr[item.hs + h] : 0u;
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
                const u32 wi = it * G + tl;
                ulonglong2 v = make_ulonglong2(0, 0);
                if (h < int(hc) && wi < W2) {
                    v = __ldg(X2 + u64(col) * W2 + wi);
                    v.x ^= yv[it].x;
                    v.y ^= yv[it].y;
                }
                hx[h][it] = v;
            }
        }
        for (u32 s0 = 0; s0 < item.sc; s0 += G) {
            const u32 my_s = s0 + tl;
            const u32 my_col = my_s < item.sc ? svr[item.ss + my_s] : 0u;
            const u32 cnt = min(u32(G), item.sc - s0);
            for (u32 q = 0; q < cnt; ++q) {
                const u32 col = __shfl_sync(tmask, my_col, q, G);
                ulonglong2 z[NIT];
#pragma unroll
                for (int it = 0; it < NIT; ++it) {
                    const u32 wi = it * G + tl;
                    z[it] = wi < W2 ? __ldg(X2 + u64(col) * W2 + wi) : make_ulonglong2(0, 0);
                }
                u32 acc[H];
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    u32 a = 0;
#pragma unroll
                    for (int it = 0; it < NIT; ++it)
                        a += __popcll(hx[h][it].x ^ z[it].x) + __popcll(hx[h][it].y ^ z[it].y);
                    acc[h] = a;
                }
#pragma unroll
                for (int h = 0; h < H; ++h) {
#pragma unroll
                    for (int o = G / 2; o > 0; o >>= 1) acc[h] += __shfl_xor_sync(tmask, acc[h], o);
                }
                // lane tl of the team tests pairs (held h, streamed s0+q) for h = tl, tl+G, ...
                const u32 spos = item.ss + s0 + q;
#pragma unroll
                for (int h0 = 0; h0 < H; h0 += G) {
                    u32 mine = 0;
#pragma unroll
                    for (int h = 0; h < H; ++h)
                        if (h == h0 + tl) mine = acc[h];
                    const u32 hpos = item.hs + h0 + tl;
                    bool hit = false;
                    u32 si = 0;
                    if (h0 + tl < int(hc) && (!(flags & 2u) || spos > hpos)) {
                        si = pos_pass ? mine : n - mine;
                        hit = si >= astar;
                    }
                    DevHit hr;
                    if (hit) hr = make_hit(A, item.run, hpos, spos, flags, double(si) / double(n), int32_t(si));
                    team_append<G>(A, tmask, hit, hr);
                }
            }
        }
    }
}

// Sum V = 2^k per-lane values across the warp so that lane L ends up with the
// warp total of value index L >> (5 - k): butterfly stages that halve the live
// values (each lane keeps the half selected by its lane bit), then plain
// xor-sums. V - 1 + (5 - k) shuffles for V totals instead of 5 V.
template <int CNT, int O, int V>
__device__ __forceinline__ void butterfly_stage(u32 (&v)[V], int lane) {
    if constexpr (O >= 1) {
        if constexpr (CNT > 1) {
            constexpr int half = CNT / 2;
            const bool up = (lane & O) != 0;
#pragma unroll
            for (int i = 0; i < half; ++i) {
                const u32 send = up ? v[i] : v[i + half];
                const u32 keep = up ? v[i + half] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, O);
            }
            butterfly_stage<half, O / 2>(v, lane);
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], O);
            butterfly_stage<1, O / 2>(v, lane);
        }
    }
}

template <int V>
__device__ __forceinline__ u32 butterfly_sum(u32 (&v)[V], int lane) {
    butterfly_stage<V, 16>(v, lane);
    return v[0];
}

// ------------------------------------------------------- pair list path --

// One canonical candidate: batch-global sorted positions of the x side and
// the z side (oriented: x side first; diagonal blocks: smaller position
// first), and the batch-local run.
struct PairRec {
    u32 pa, pb, run, pad;
};

// Expand every item into its candidate pairs (h-major, so consecutive pairs
// share the held column and stay in one team's L1). Warp per item; slots
// were reserved by join_emit (the counter runs past pair_cap for a regrow).
__global__ void __launch_bounds__(256) expand_pairs(const Item* __restrict__ items, const u32* __restrict__ nitems,
                                                    u32 item_cap, u64 S, PairRec* __restrict__ pairs, u32 pair_cap) {
    const int lane = threadIdx.x & 31;
    const u32 N = min(*nitems, item_cap);
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 t = warp; t < N; t += nwarps) {
        const Item it = items[t];
        const u32 hc = it.hc_flags & 0xffu, flags = it.hc_flags >> 8;
        const bool diag = flags & 2u, held_x = flags & 1u;
        const u32 tot = hc * it.sc;
        const u64 off = u64(it.run) * S;
        const u32 base = it.pad;  // slots reserved by join_emit
        u32 written = 0;
        for (u32 e0 = 0; e0 < tot; e0 += 32) {
            const u32 e = e0 + lane;
            bool ok = e < tot;
            u32 hpos = 0, spos = 0;
            if (ok) {
                const u32 h = e / it.sc, s = e - h * it.sc;
                hpos = it.hs + h;
                spos = it.ss + s;
                if (diag && spos <= hpos) ok = false;
            }
            const u32 bal = __ballot_sync(0xffffffffu, ok);
            if (ok) {
                const u32 slot = base + written + __popc(bal & lanemask_lt());
                if (slot < pair_cap) {
                    PairRec r;
                    const u32 first = (diag || held_x) ? hpos : spos, second = (diag || held_x) ? spos : hpos;
                    r.pa = u32(off + first);
                    r.pb = u32(off + second);
                    r.run = it.run;
                    r.pad = 0;
                    pairs[slot] = r;
                }
            }
            written += __popc(bal);
        }
    }
}

// Binary verify over the pair list: a team of G lanes per pair, NIT x 16 B of
// each column per lane (up to 2 x 64 B in flight per lane), teams walk
// contiguous chunks of kPairChunk pairs so shared columns hit in L1.
constexpr u32 kPairChunk = 32;

template <int G, int NIT>
__global__ void __launch_bounds__(256) verify_pairs_binary(VerifyArgs A, const PairRec* __restrict__ pairs,
                                                           const u32* __restrict__ npairs, u32 pair_cap,
                                                           const u64* __restrict__ Xc, u32 Wp,
                                                           const u64* __restrict__ Yw, u32 n, u32 astar) {
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
    const u32 P = min(*npairs, pair_cap);
    const u64 team = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const u64 nteams = (u64(gridDim.x) * blockDim.x) / G;
    for (u64 c0 = team * kPairChunk; c0 < P; c0 += nteams * kPairChunk) {
        const u32 c1 = u32(minu(P, c0 + kPairChunk));
        for (u32 q = u32(c0); q < c1; ++q) {
            const PairRec pr = pairs[q];
            const u32 j = A.sv[pr.pa], k = A.sv[pr.pb];
            const ulonglong2* xj = X2 + u64(j) * W2;
            const ulonglong2* xk = X2 + u64(k) * W2;
            ulonglong2 a[NIT], b[NIT];
#pragma unroll
            for (int it = 0; it < NIT; ++it) {
                const u32 wi = it * G + tl;
                a[it] = wi < W2 ? __ldg(xj + wi) : make_ulonglong2(0, 0);
                b[it] = wi < W2 ? __ldg(xk + wi) : make_ulonglong2(0, 0);
            }
            u32 acc = 0;
#pragma unroll
            for (int it = 0; it < NIT; ++it)
                acc += __popcll(a[it].x ^ b[it].x ^ yv[it].x) + __popcll(a[it].y ^ b[it].y ^ yv[it].y);
#pragma unroll
            for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(tmask, acc, o);
            const u32 si = A.run_sign[pr.run] > 0 ? acc : n - acc;
            const bool hit = tl == 0 && si >= astar;
            DevHit h;
            if (hit) {
                const u32 r = A.rid[pr.run];
                const u64 base = u64(pr.run) * A.S;
                h.order = (u64(r) * A.p + (pr.pa - base)) * A.p + (pr.pb - base);
                h.s = double(si) / double(n);
                h.j = j;
                h.k = k;
                h.rid = r;
                h.sint = int32_t(si);
            }
            team_append<G>(A, tmask, hit, h);
        }
    }
}

// Binary verify for 33..64-word columns (n in (2048, 4096], e.g. BASELINE
// config 2): one warp per item, 16 B of a column per lane, the <= 8 held
// columns (XORed with Y) in registers, U streamed columns loaded at once
// (U x 512 B in flight per warp) and the 8U popcount partials reduced with
// one butterfly (about one shuffle per pair).
template <int U>
__global__ void __launch_bounds__(256) verify_binary_w32(VerifyArgs A, const u64* __restrict__ Xc, u32 Wp,
                                                         const u64* __restrict__ Yw, u32 n, u32 astar) {
    constexpr int H = 8, V = H * U;
    constexpr int SH = (V == 32) ? 0 : (V == 16) ? 1 : 2;  // lane -> value index shift
    const int lane = threadIdx.x & 31;
    const u32 W2 = Wp / 2;
    const ulonglong2* X2 = reinterpret_cast<const ulonglong2*>(Xc);
    const ulonglong2 y = lane < int(W2) ? __ldg(reinterpret_cast<const ulonglong2*>(Yw) + lane) : make_ulonglong2(0, 0);
    const u32 N = min(*A.nitems, A.item_cap);
    const u64 warp = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const u64 nwarps = (u64(gridDim.x) * blockDim.x) >> 5;
    // this lane's (held, streamed) slot in the butterfly output
    const int my_idx = lane >> SH;
    const int my_u = my_idx / H, my_h = my_idx % H;
    const bool owner = (lane & ((1 << SH) - 1)) == 0;
    for (u64 t = warp; t < N; t += nwarps) {
        const Item item = A.items[t];
        if (A.tot[item.run] > A.guard) continue;  // aborted run: nothing is evaluated
        const u32 hc = item.hc_flags & 0xffu, flags = item.hc_flags >> 8;
        const u32* svr = A.sv + u64(item.run) * A.S;
        const bool pos_pass = A.run_sign[item.run] > 0;
        const u32 my_held = lane < int(hc) ? svr[item.hs + lane] : 0u;
        ulonglong2 hx[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const u32 col = __shfl_sync(0xffffffffu, my_held, h);
            ulonglong2 v = make_ulonglong2(0, 0);
            if (h < int(hc) && lane < int(W2)) {
                v = __ldg(X2 + u64(col) * W2 + lane);
                v.x ^= y.x;
                v.y ^= y.y;
            }
            hx[h] = v;
        }
        for (u32 s0 = 0; s0 < item.sc; s0 += 32) {
            const u32 cnt = min(32u, item.sc - s0);
            const u32 my_col = u32(lane) < cnt ? svr[item.ss + s0 + lane] : 0u;
            for (u32 q0 = 0; q0 < cnt; q0 += U) {
                ulonglong2 z[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const u32 col = __shfl_sync(0xffffffffu, my_col, (q0 + u) & 31);
                    z[u] = (q0 + u < cnt && lane < int(W2)) ? __ldg(X2 + u64(col) * W2 + lane) : make_ulonglong2(0, 0);
                }
                u32 v[V];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int h = 0; h < H; ++h)
                        v[u * H + h] = __popcll(hx[h].x ^ z[u].x) + __popcll(hx[h].y ^ z[u].y);
                const u32 agree = butterfly_sum<V>(v, lane);
                const u32 spos = item.ss + s0 + q0 + my_u;
                const u32 hpos = item.hs + my_h;
                bool hit = false;
                u32 si = 0;
                if (owner && my_h < int(hc) && q0 + my_u < cnt && (!(flags & 2u) || spos > hpos)) {
                    si = pos_pass ? agree : n - agree;
                    hit = si >= astar;
                }
                DevHit hr;
                if (hit) hr = make_hit(A, item.run, hpos, spos, flags, double(si) / double(n), int32_t(si));
                team_append<32>(A, 0xffffffffu, hit, hr);
            }
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
template <int G, bool UNBIASED>
__device__ __forceinline__ double real_pair(const float4* xj, const float4* xk, const double2* yv, u64 n4q, int tl,
                                            u32 tmask) {
    double acc = 0.0;
    for (u64 q = tl; q < n4q; q += G) {
        const float4 a = __ldg(xj + q), b = __ldg(xk + q);
        const double2 y0 = __ldg(yv + 2 * q), y1 = __ldg(yv + 2 * q + 1);
        if (UNBIASED) {
            acc = fma(y0.x, double(a.x) * double(b.x), acc);
            acc = fma(y0.y, double(a.y) * double(b.y), acc);
            acc = fma(y1.x, double(a.z) * double(b.z), acc);
            acc = fma(y1.y, double(a.w) * double(b.w), acc);
        } else {
            auto t = [](float v) { return v > 0.f ? 1.0 : (v < 0.f ? -1.0 : 0.0); };
            acc = fma(y0.x, t(a.x) * t(b.x), acc);
            acc = fma(y0.y, t(a.y) * t(b.y), acc);
            acc = fma(y1.x, t(a.z) * t(b.z), acc);
            acc = fma(y1.y, t(a.w) * t(b.w), acc);
        }
    }
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
                const bool hit = tl == 0 && strength.hit(s);
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
    const double* y;
    double norm, gamma;
    __device__ double operator()(u32 j, u32 k, bool pos_pass, int tl, u32 tmask) const {
        const double acc = real_pair<32, UNBIASED>(reinterpret_cast<const float4*>(Xc32 + u64(j) * n4),
                                                   reinterpret_cast<const float4*>(Xc32 + u64(k) * n4),
                                                   reinterpret_cast<const double2*>(y), n4 / 4, tl, tmask);
        return 0.5 + (pos_pass ? 1.0 : -1.0) * acc / (2.0 * norm);
    }
    __device__ bool hit(double s) const { return s >= gamma; }
};

template <class F>
__global__ void __launch_bounds__(256) verify_items(VerifyArgs A, F f) {
    walk_items<32>(A, f);
}

} // namespace kern
} // namespace xyzb
