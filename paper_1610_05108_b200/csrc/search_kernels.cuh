// Device kernels of one batch of xyz runs (sm_100a).
//
//   transpose_bits   column-major packed X -> row planes (once per dataset)
//   project_bits     M-bit keys of every column for every run of the batch
//                    (project_keys, projection.cpp:32-57) + the per-run XOR
//                    constant c that turns x-keys into z-keys (A.3)
//   join             bucket join over the sorted keys: equal-key runs,
//                    partner run of key^c, |E_r| incl. the diagonal, and one
//                    canonical block per unordered key pair (equal_pairs,
//                    pair_search.cpp:35-53, with the guard of
//                    pair_search.hpp:91-94 applied per run)
//   verify_*         exact strength of every canonical candidate, hit test,
//                    warp-aggregated hit append (filter_strong,
//                    pair_search.hpp:95-109; strengths transforms.cpp:33-76,
//                    search.cpp:477-493)
#pragma once

#include "common.cuh"

namespace xyzb {
namespace kern {

// One canonical block of a run: x-side positions [xs, xs+xc) of the run's
// sorted key array, z-side positions [zs, zs+zc). xs == zs marks the diagonal
// block (c == 0, key paired with itself; canonical pairs a < b only).
struct Block {
    u32 run;  // batch-local run index
    u32 xs, xc, zs, zc;
    u32 pad;
};

// A verified candidate with strength >= gamma (pre-dedup).
struct DevHit {
    u64 order;  // rid * p^2 + pos_first * p + pos_second  (A.5 order inside a run)
    double s;   // strength (binary: exact sint / n)
    u32 j, k;   // oriented as the reference emits it (first in A.5 order)
    u32 rid;    // global run index: pass * L + rep - 1
    int32_t sint;  // binary: integer strength numerator; else -1
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

// first index in [lo, hi) with a[idx] > v, given a[lo] <= v (galloping)
template <class K>
__device__ __forceinline__ u64 run_end(const K* a, u64 lo, u64 hi, K v) {
    u64 step = 1, last_le = lo;
    u64 probe = lo + 1;
    while (probe < hi && a[probe] == v) {
        last_le = probe;
        step <<= 1;
        probe = lo + step;
    }
    u64 l = last_le + 1, h = min(probe, hi);
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

template <class K>
__global__ void __launch_bounds__(256) join(const K* __restrict__ sk, u64 S, const K* __restrict__ xorc,
                                            Block* __restrict__ blocks, u64* __restrict__ bwork,
                                            u32* __restrict__ nblocks, u64* __restrict__ tot) {
    __shared__ u64 red[8];
    const u32 b = blockIdx.y;
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    const K* a = sk + u64(b) * S;
    bool emit = false;
    Block blk{};
    u64 pairs = 0, work = 0;
    if (i < S) {
        const K v = a[i];
        if (i == 0 || a[i - 1] != v) {
            const u64 e = run_end(a, i, S, v);
            const u64 cnt = e - i;
            const K v2 = v ^ xorc[b];
            if (v2 == v) {
                pairs = cnt * cnt;  // the diagonal j == k counts (pair_search.cpp:48-49)
                if (cnt >= 2) {
                    emit = true;
                    blk = {b, u32(i), u32(cnt), u32(i), u32(cnt), 0u};
                    work = cnt * (cnt - 1) / 2;
                }
            } else if (v2 > v) {
                const u64 lo = lower_bound(a, e, S, v2);
                if (lo < S && a[lo] == v2) {
                    const u64 zc = run_end(a, lo, S, v2) - lo;
                    pairs = 2 * cnt * zc;  // (j,k) in block v and (k,j) in block v^c
                    emit = true;
                    blk = {b, u32(i), u32(cnt), u32(lo), u32(zc), 0u};
                    work = cnt * zc;
                }
            }
        }
    }
    // |E_r| per run
    u64 ws = warp_sum(pairs);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ws;
    // warp-aggregated block append
    const u32 ballot = __ballot_sync(0xffffffffu, emit);
    if (ballot) {
        u32 base = 0;
        if ((threadIdx.x & 31) == __ffs(ballot) - 1) base = atomicAdd(nblocks, __popc(ballot));
        base = __shfl_sync(0xffffffffu, base, __ffs(ballot) - 1);
        if (emit) {
            const u32 slot = base + __popc(ballot & lanemask_lt());
            blocks[slot] = blk;
            bwork[slot] = work;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 t = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
        if (t) atomicAdd(reinterpret_cast<unsigned long long*>(tot + b), static_cast<unsigned long long>(t));
    }
}

// Guard (pair_search.hpp:91-94): a run whose |E_r| exceeds the guard is
// aborted, nothing of it is evaluated. Also books per-run counters.
__global__ void guard_blocks(const Block* __restrict__ blocks, u64* __restrict__ bwork, const u32* __restrict__ nblocks,
                             const u64* __restrict__ tot, u64 guard, const u32* __restrict__ rid,
                             u64* __restrict__ verified_by_rid) {
    const u32 nb = *nblocks;
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < nb; i += u64(gridDim.x) * blockDim.x) {
        const u32 r = blocks[i].run;
        if (tot[r] > guard) {
            bwork[i] = 0;
        } else if (bwork[i]) {
            atomicAdd(reinterpret_cast<unsigned long long*>(verified_by_rid + rid[r]),
                      static_cast<unsigned long long>(bwork[i]));
        }
    }
}

__global__ void book_runs(u32 B, const u64* __restrict__ tot, const u32* __restrict__ rid,
                          u64* __restrict__ enumerated_by_rid) {
    const u32 b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < B) enumerated_by_rid[rid[b]] = tot[b];
}

// ---------------------------------------------------------------- verify --

struct PairCursor {
    u64 q, q_end;  // pair range of this chunk
    u32 blk;       // current block
    u64 off, off_next;
};

// Decode canonical pair q of block `bl` with work offset `off` into sorted
// positions (pa: x side, pb: z side). Diagonal block: upper triangle a < b.
__device__ __forceinline__ void decode_pair(const Block& bl, u64 t, u32& pa, u32& pb) {
    if (bl.xs != bl.zs) {
        const u64 a = t / bl.zc;
        pa = bl.xs + u32(a);
        pb = bl.zs + u32(t - a * bl.zc);
    } else {
        // row a holds (c-1-a) pairs; start(a) = a*(2c-a-1)/2
        const double c = double(bl.xc);
        const double disc = (2.0 * c - 1.0) * (2.0 * c - 1.0) - 8.0 * double(t);
        u64 a = u64(floor(((2.0 * c - 1.0) - sqrt(fmax(disc, 0.0))) * 0.5));
        const u64 cc = bl.xc;
        auto start = [&](u64 r) { return r * (2 * cc - r - 1) / 2; };
        while (a > 0 && start(a) > t) --a;
        while (a + 1 < cc && start(a + 1) <= t) ++a;
        pa = bl.xs + u32(a);
        pb = bl.xs + u32(t - start(a) + a + 1);
    }
}

__device__ __forceinline__ u32 find_block(const u64* __restrict__ off, u32 nb, u64 q) {
    // last b with off[b] <= q (off has nb+1 entries, off[nb] = total)
    u32 lo = 0, hi = nb;  // answer in [0, nb)
    while (hi - lo > 1) {
        const u32 mid = (lo + hi) >> 1;
        if (off[mid] <= q) lo = mid; else hi = mid;
    }
    return lo;
}

struct VerifyArgs {
    const Block* blocks;
    const u64* work_off;  // nb+1
    const u32* nblocks;
    const u32* sv;        // sorted column indices [B][S]
    u64 S;                // = p
    const u32* rid;       // batch -> global run id
    const int8_t* run_sign;
    u64 p;
    DevHit* hits;
    u32* hit_count;
    u32 hit_cap;
};

__device__ __forceinline__ void append_hit(const VerifyArgs& A, bool hit, const DevHit& h) {
    const u32 ballot = __ballot_sync(0xffffffffu, hit);
    if (!ballot) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(ballot) - 1;
    u32 base = 0;
    if (lane == leader) base = atomicAdd(A.hit_count, __popc(ballot));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (hit) {
        const u32 slot = base + __popc(ballot & lanemask_lt());
        if (slot < A.hit_cap) A.hits[slot] = h;
    }
}

// Strength kernels share the pair walk: each team of G lanes takes chunks of
// kChunk consecutive canonical pairs (global pair index over all blocks of
// the batch, prefix-summed work), decodes (run, x position, z position), and
// computes the strength cooperatively. Persistent grid.
constexpr u32 kChunk = 64;

template <int G, class Strength>
__device__ __forceinline__ void walk_pairs(const VerifyArgs& A, Strength&& strength) {
    const u32 nb = *A.nblocks;
    if (nb == 0) return;
    const u64 total = A.work_off[nb];
    const int lane = threadIdx.x & 31;
    const int tl = lane & (G - 1);
    const u64 team = (u64(blockIdx.x) * blockDim.x + threadIdx.x) / G;
    const u64 nteams = (u64(gridDim.x) * blockDim.x) / G;
    const u64 nchunks = (total + kChunk - 1) / kChunk;
    // every lane of a warp iterates the same number of times (ballots inside)
    const u64 warp_team0 = (u64(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u)) / G;
    for (u64 c0 = warp_team0; c0 < nchunks; c0 += nteams) {
        const u64 c = c0 + (team - warp_team0);
        const bool active = c < nchunks;
        u64 q = active ? c * kChunk : total;
        const u64 q_end = active ? min(total, q + kChunk) : total;
        u32 bidx = active ? find_block(A.work_off, nb, q) : 0;
        u64 off = A.work_off[bidx], off_next = A.work_off[bidx + 1];
        Block bl = A.blocks[bidx];
        for (u32 it = 0; it < kChunk; ++it) {
            const bool valid = q < q_end;
            u32 pa = 0, pb = 0;
            if (valid) {
                while (q >= off_next) {
                    ++bidx;
                    off = off_next;
                    off_next = A.work_off[bidx + 1];
                    bl = A.blocks[bidx];
                }
                decode_pair(bl, q - off, pa, pb);
            }
            const u64 seg = u64(bl.run) * A.S;
            const u32 j = valid ? A.sv[seg + pa] : 0u;
            const u32 k = valid ? A.sv[seg + pb] : 0u;
            const u32 r = bl.run;
            int32_t sint = -1;
            double s = 0.0;
            bool hit = strength(valid, r, j, k, tl, s, sint);
            DevHit h;
            if (hit) {
                // orientation (A.8): x side first when keys differ; smaller index on the diagonal
                const u32 rid = A.rid[r];
                const bool diag = bl.xs == bl.zs;
                const u32 fj = diag ? min(j, k) : j, fk = diag ? max(j, k) : k;
                const u64 pf = diag ? min(pa, pb) : pa, ps = diag ? max(pa, pb) : pb;
                h.order = (u64(rid) * A.p + pf) * A.p + ps;
                h.s = s;
                h.j = fj;
                h.k = fk;
                h.rid = rid;
                h.sint = sint;
            }
            append_hit(A, hit && tl == 0, h);
            if (valid) ++q;
            // all lanes of the warp keep iterating together; stop when whole warp is done
            if (!__any_sync(0xffffffffu, q < q_end)) break;
        }
    }
}

// Binary: agree = popc(X_j ^ X_k ^ Y) over the padded words (padding is 0 in
// X and Y, packed_matrix.cpp:29-35); pass +1 strength agree/n, pass -1
// (n-agree)/n (search.cpp:25-36,347-349). Integer hit test sint >= astar.
template <int G, int NIT>
__global__ void __launch_bounds__(256) verify_binary(VerifyArgs A, const u64* __restrict__ Xc, u32 Wp,
                                                     const u64* __restrict__ Yw, u32 n, u32 astar) {
    const int tl = threadIdx.x & (G - 1);
    ulonglong2 yv[NIT > 0 ? NIT : 1];
    if (NIT > 0) {
#pragma unroll
        for (int it = 0; it < (NIT > 0 ? NIT : 1); ++it) {
            const u32 wi = 2 * (it * G + tl);
            yv[it] = wi < Wp ? *reinterpret_cast<const ulonglong2*>(Yw + wi) : make_ulonglong2(0, 0);
        }
    }
    walk_pairs<G>(A, [&](bool valid, u32 r, u32 j, u32 k, int tl_, double& s, int32_t& sint) -> bool {
        u32 acc = 0;
        if (valid) {
            const ulonglong2* xj = reinterpret_cast<const ulonglong2*>(Xc + u64(j) * Wp);
            const ulonglong2* xk = reinterpret_cast<const ulonglong2*>(Xc + u64(k) * Wp);
            if (NIT > 0) {
#pragma unroll
                for (int it = 0; it < (NIT > 0 ? NIT : 1); ++it) {
                    const u32 wi = it * G + tl_;
                    if (2 * wi < Wp) {
                        const ulonglong2 a = __ldg(xj + wi), b = __ldg(xk + wi);
                        acc += __popcll(a.x ^ b.x ^ yv[it].x) + __popcll(a.y ^ b.y ^ yv[it].y);
                    }
                }
            } else {
                const ulonglong2* yw = reinterpret_cast<const ulonglong2*>(Yw);
                for (u32 wi = tl_; 2 * wi < Wp; wi += G) {
                    const ulonglong2 a = __ldg(xj + wi), b = __ldg(xk + wi), y = __ldg(yw + wi);
                    acc += __popcll(a.x ^ b.x ^ y.x) + __popcll(a.y ^ b.y ^ y.y);
                }
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (!valid) return false;
        const int8_t sg = A.run_sign[r];
        const u32 si = sg > 0 ? acc : n - acc;
        sint = int32_t(si);
        s = double(si) / double(n);
        return si >= astar;
    });
}

// Continuous-Y (transforms.cpp:42-76): sum of |y_i| over rows where
// bit(x_j ^ x_k ^ s) = 1, s = (resp > 0), over ||resp||_1; resp = +-y.
template <int G>
__global__ void __launch_bounds__(256) verify_weighted(VerifyArgs A, const u64* __restrict__ Xc, u32 Wp,
                                                       const u64* __restrict__ spos, const u64* __restrict__ sneg,
                                                       const double* __restrict__ wabs, double norm, double gamma) {
    walk_pairs<G>(A, [&](bool valid, u32 r, u32 j, u32 k, int tl, double& s, int32_t& sint) -> bool {
        double acc = 0.0;
        if (valid) {
            const u64* xj = Xc + u64(j) * Wp;
            const u64* xk = Xc + u64(k) * Wp;
            const u64* sb = A.run_sign[r] > 0 ? spos : sneg;
            for (u32 wi = tl; wi < Wp; wi += G) {
                u64 m = __ldg(xj + wi) ^ __ldg(xk + wi) ^ __ldg(sb + wi);
                const double* wrow = wabs + u64(wi) * 64;
                while (m) {
                    const int bit = __ffsll(static_cast<long long>(m)) - 1;
                    acc += __ldg(wrow + bit);
                    m &= m - 1;
                }
            }
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (!valid) return false;
        s = acc / norm;
        sint = -1;
        return s >= gamma;
    });
}

// Continuous-XY (search.cpp:477-493): 0.5 + sign * sum_i y_i t(x_ij) t(x_ik) / (2 ||y||_1),
// fp32 columns, products and accumulation in fp64.
template <int G, bool UNBIASED>
__global__ void __launch_bounds__(256) verify_real(VerifyArgs A, const float* __restrict__ Xc32, u64 n4,
                                                   const double* __restrict__ y, double norm, double gamma) {
    walk_pairs<G>(A, [&](bool valid, u32 r, u32 j, u32 k, int tl, double& s, int32_t& sint) -> bool {
        double acc = 0.0;
        if (valid) {
            const float4* xj = reinterpret_cast<const float4*>(Xc32 + u64(j) * n4);
            const float4* xk = reinterpret_cast<const float4*>(Xc32 + u64(k) * n4);
            const double2* yv = reinterpret_cast<const double2*>(y);
            for (u64 q = tl; q < n4 / 4; q += G) {
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
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (!valid) return false;
        const double sg = A.run_sign[r] > 0 ? 1.0 : -1.0;
        s = 0.5 + sg * acc / (2.0 * norm);
        sint = -1;
        return s >= gamma;
    });
}

} // namespace kern
} // namespace xyzb
