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
// per run; the sequential seed_seq recurrence runs on lane 0 out of shared
// memory, all runs of a batch in parallel.
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

// std::seed_seq{v0..v3}.generate(a, a + 624) followed by mt19937_64::seed(q).
__device__ void seed_mt(const u32 v[4], u32* a /*624*/, u64* x /*312*/) {
    const u32 n = 624, s = 4, t = 11, p = (n - t) / 2, q = p + t, m = n;  // m = max(s + 1, n)
    for (u32 i = 0; i < n; ++i) a[i] = 0x8b8b8b8bu;
    for (u32 k = 0; k < m; ++k) {
        const u32 kn = k % n, kpn = (k + p) % n, kqn = (k + q) % n;
        const u32 arg = a[kn] ^ a[kpn] ^ a[(k + n - 1) % n];
        const u32 r1 = 1664525u * (arg ^ (arg >> 27));
        u32 r2 = r1 + kn;
        if (k == 0) r2 = r1 + s;
        else if (k <= s) r2 = r1 + kn + v[k - 1];
        a[kpn] += r1;
        a[kqn] += r2;
        a[kn] = r2;
    }
    for (u32 k = m; k < m + n; ++k) {
        const u32 kn = k % n, kpn = (k + p) % n, kqn = (k + q) % n;
        const u32 arg = a[kn] + a[kpn] + a[(k - 1) % n];
        const u32 r3 = 1566083941u * (arg ^ (arg >> 27));
        const u32 r4 = r3 - kn;
        a[kpn] ^= r3;
        a[kqn] ^= r4;
        a[kn] = r4;
    }
    bool zero = true;
    for (int i = 0; i < 312; ++i) {
        x[i] = u64(a[2 * i]) | (u64(a[2 * i + 1]) << 32);
        if (zero) {
            if (i == 0) {
                if ((x[0] & 0xffffffff80000000ull) != 0) zero = false;
            } else if (x[i] != 0) {
                zero = false;
            }
        }
    }
    if (zero) x[0] = 1ull << 63;
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
    if (threadIdx.x == 0) {
        u64 s = seed;
        const u64 a = splitmix64(s);
        s ^= streams[r] * 0xd1342543de82ef95ull + 0x2545f4914f6cdd1dull;
        const u64 b = splitmix64(s);
        const u32 v[4] = {u32(a), u32(a >> 32), u32(b), u32(b >> 32)};
        seed_mt(v, arr, x);
        Mt g{x, 312};
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
