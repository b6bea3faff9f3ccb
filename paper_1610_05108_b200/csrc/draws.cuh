// Per-run row draws on the device.
//
// Run r of pass sigma uses std::mt19937_64 seeded through std::seed_seq from
// make_stream(seed, offset + rep) (rng.hpp:18-26), then draws M rows with
// std::uniform_int_distribution<size_t>(0, n-1) (projection.cpp:26-27) or
// WeightedSampler::sample (real_matrix.cpp:49-54). Everything here restates
// those standard-library algorithms bit for bit, as libstdc++ 13 implements
// them (seed_seq::generate, random.tcc:3256-3343; mersenne_twister_engine::
// seed(Sseq&), :351-391, _M_gen_rand :399-425, operator() :455-466;
// uniform_int_distribution::_S_nd, uniform_int_dist.h:252-278, taken with
// unsigned __int128 for a 64-bit engine), so the device draws equal the
// reference's host draws (tests: golden fixtures, draws vs oracle). One warp
// per run; the sequential seed_seq recurrence runs on lane 0 with its chain
// in registers, packing and the first twist on the whole warp, all runs of a
// batch in parallel.
#pragma once

#include "common.cuh"
#include "real_kernels.cuh"

namespace xyzb {
namespace draws {

__device__ __forceinline__ u64 splitmix64(u64& s) {
    u64 z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

struct Mt {
    u64* x;  // 312 words (shared memory)
    int pos;
    __device__ u64 next() {
        if (pos >= real::kMtN) {
            twist_serial();
            pos = 0;
        }
        return real::mt_temper(x[pos++]);
    }
    __device__ void twist_serial() {
        const u64 UM = 0xffffffff80000000ull, LM = 0x7fffffffull, A = 0xb5026f5aa96619e9ull;
        for (int k = 0; k < 156; ++k) {
            const u64 y = (x[k] & UM) | (x[k + 1] & LM);
            x[k] = x[k + 156] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
        }
        for (int k = 156; k < 311; ++k) {
            const u64 y = (x[k] & UM) | (x[k + 1] & LM);
            x[k] = x[k - 156] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
        }
        const u64 y = (x[311] & UM) | (x[0] & LM);
        x[311] = x[155] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
    }
};

// std::seed_seq{v0..v3}.generate(a, a + 624) (random.tcc:3256-3343), lane 0.
// The recurrence is serial through a[k-1]; that value stays in a register
// and the next iteration's a[k+1], a[k+1+p], a[k+1+q] are loaded before this
// iteration's stores (they never alias them: p = 306, q = 317, n = 624), so
// the dependent chain is a few ALU operations per step, not shared-memory
// round trips.
__device__ void seed_seq_624(const u32 v[4], u32* a /*624, filled with 0x8b8b8b8b*/) {
    constexpr u32 n = 624, s = 4, p = 306, q = 317;  // t = 11, p = (n - t) / 2, q = p + t
    u32 prev = a[n - 1], ak = a[0], akp = a[p], akq = a[q];
    for (u32 k = 0; k < n; ++k) {
        const u32 kpn = k + p < n ? k + p : k + p - n, kqn = k + q < n ? k + q : k + q - n;
        const u32 arg = ak ^ akp ^ prev;
        const u32 r1 = 1664525u * (arg ^ (arg >> 27));
        u32 r2 = r1 + k;
        if (k == 0) r2 = r1 + s;
        else if (k <= s) r2 = r1 + k + v[k - 1];
        const u32 k1 = k + 1 < n ? k + 1 : 0;
        const u32 k1p = kpn + 1 < n ? kpn + 1 : 0, k1q = kqn + 1 < n ? kqn + 1 : 0;
        const u32 nk = a[k1], nkp = a[k1p], nkq = a[k1q];
        a[kpn] = akp + r1;
        a[kqn] = akq + r2;
        a[k] = r2;
        prev = r2;
        ak = nk;
        akp = nkp;
        akq = nkq;
    }
    ak = a[0];
    akp = a[p];
    akq = a[q];
    for (u32 k = 0; k < n; ++k) {  // k here is (m + k) % n of the reference loop, m = n
        const u32 kpn = k + p < n ? k + p : k + p - n, kqn = k + q < n ? k + q : k + q - n;
        const u32 arg = ak + akp + prev;
        const u32 r3 = 1566083941u * (arg ^ (arg >> 27));
        const u32 r4 = r3 - k;
        const u32 k1 = k + 1 < n ? k + 1 : 0;
        const u32 k1p = kpn + 1 < n ? kpn + 1 : 0, k1q = kqn + 1 < n ? kqn + 1 : 0;
        const u32 nk = a[k1], nkp = a[k1p], nkq = a[k1q];
        a[kpn] = akp ^ r3;
        a[kqn] = akq ^ r4;
        a[k] = r4;
        prev = r4;
        ak = nk;
        akp = nkp;
        akq = nkq;
    }
}

// mt19937_64::seed(seed_seq&) (random.tcc:351-391) from the 624 words, one
// warp: pack to 312 u64 words, all-zero check.
__device__ void seed_mt_warp(const u32* a, u64* x) {
    const int lane = threadIdx.x & 31;
    bool nz = false;
    for (int i = lane; i < 312; i += 32) {
        x[i] = u64(a[2 * i]) | (u64(a[2 * i + 1]) << 32);
        nz |= i == 0 ? (x[0] & 0xffffffff80000000ull) != 0 : x[i] != 0;
    }
    const bool any = __any_sync(0xffffffffu, nz);
    __syncwarp();
    if (!any && lane == 0) x[0] = 1ull << 63;
    __syncwarp();
}

// _M_gen_rand (random.tcc:399-425) by one warp: the first 156 words depend
// only on old words, the next 155 on old words and phase-1 results, the last
// on phase-1 results.
__device__ void twist_warp(u64* x) {
    const u64 UM = 0xffffffff80000000ull, LM = 0x7fffffffull, A = 0xb5026f5aa96619e9ull;
    const int lane = threadIdx.x & 31;
    u64 v[5];
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int k = lane + 32 * i;
        if (k < 156) {
            const u64 y = (x[k] & UM) | (x[k + 1] & LM);
            v[i] = x[k + 156] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
        }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (lane + 32 * i < 156) x[lane + 32 * i] = v[i];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int k = 156 + lane + 32 * i;
        if (k < 311) {
            const u64 y = (x[k] & UM) | (x[k + 1] & LM);
            v[i] = x[k - 156] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
        }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 5; ++i)
        if (156 + lane + 32 * i < 311) x[156 + lane + 32 * i] = v[i];
    __syncwarp();
    if (lane == 0) {
        const u64 y = (x[311] & UM) | (x[0] & LM);
        x[311] = x[155] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
    }
    __syncwarp();
}

// Lemire nearly-divisionless draw in [0, range) with 128-bit products.
__device__ __forceinline__ u64 lemire(Mt& g, u64 range) {
    u64 v = g.next();
    u64 lo = v * range;
    u64 hi = __umul64hi(v, range);
    if (lo < range) {
        const u64 threshold = (0ull - range) % range;
        while (lo < threshold) {
            v = g.next();
            lo = v * range;
            hi = __umul64hi(v, range);
        }
    }
    return hi;
}

// One warp per run. streams[r] = offset + rep; rows out [R][M]; cum (n
// doubles) selects weighted draws; mt_out [R][313] receives the engine state
// after the draws (continuous-XY transforms consume the stream further).
__global__ void __launch_bounds__(32) draw_runs(u32 R, const u64* __restrict__ streams, u64 seed, u64 n, int M,
                                                const double* __restrict__ cum, u32* __restrict__ rows,
                                                u64* __restrict__ mt_out) {
    __shared__ u32 arr[624];
    __shared__ u64 x[312];
    const u32 r = blockIdx.x;
    if (r >= R) return;
    u32 v[4];
    {
        u64 s = seed;
        const u64 a = splitmix64(s);
        s ^= streams[r] * 0xd1342543de82ef95ull + 0x2545f4914f6cdd1dull;
        const u64 b = splitmix64(s);
        v[0] = u32(a);
        v[1] = u32(a >> 32);
        v[2] = u32(b);
        v[3] = u32(b >> 32);
    }
    for (int i = threadIdx.x; i < 624; i += 32) arr[i] = 0x8b8b8b8bu;
    __syncwarp();
    if (threadIdx.x == 0) seed_seq_624(v, arr);
    __syncwarp();
    seed_mt_warp(arr, x);
    twist_warp(x);  // the first draw regenerates the state: do it with the whole warp
    if (threadIdx.x == 0) {
        Mt g{x, 0};
        for (int t = 0; t < M; ++t) {
            u64 idx;
            if (cum) {
                const double u = double(g.next() >> 11) * 0x1.0p-53;
                u64 lo = 0, hi = n;  // upper_bound
                while (lo < hi) {
                    const u64 mid = (lo + hi) >> 1;
                    if (!(u < cum[mid])) lo = mid + 1; else hi = mid;
                }
                idx = lo < n - 1 ? lo : n - 1;
            } else {
                idx = lemire(g, n);
            }
            rows[u64(r) * M + t] = u32(idx);
        }
        if (mt_out) {
            for (int i = 0; i < 312; ++i) mt_out[u64(r) * 313 + i] = x[i];
            mt_out[u64(r) * 313 + 312] = u64(g.pos);
        }
    }
}

} // namespace draws
} // namespace xyzb
