// Continuous-XY projection (search.cpp:440-472) on the device.
//
// The reference binarises X per subsampled entry while it builds the keys,
// consuming its per-run std::mt19937_64 in (j, s) order: one uniform_unit
// per entry for the unbiased transform, one rng() per exact zero for the
// sign transform. The host draws the M rows, then exports the engine state;
// the device resumes the same MT19937-64 stream (libstdc++'s
// mersenne_twister_engine: _M_gen_rand and tempering, random.tcc:399-466)
// with one CTA per run and consumes it in the same order.
#pragma once

#include "common.cuh"

namespace xyzb {
namespace real {

constexpr int kMtN = 312;
constexpr int kMtThreads = 320;

__device__ __forceinline__ u64 mt_temper(u64 z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71d67fffeda60000ull;
    z ^= (z << 37) & 0xfff7eee000000000ull;
    z ^= (z >> 43);
    return z;
}

// fp64 -> fp32 copy (the response for the continuous-XY verify).
__global__ void to_f32(const double* __restrict__ a, u64 n, float* __restrict__ b) {
    for (u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
        b[i] = float(a[i]);
}

// Regenerate the 312-word state in place; all threads of the CTA call it.
__device__ __forceinline__ void mt_twist(u64* x) {
    const u64 UM = 0xffffffff80000000ull, LM = 0x7fffffffull, A = 0xb5026f5aa96619e9ull;
    const int k = threadIdx.x;
    u64 v = 0;
    if (k < 156) {
        const u64 y = (x[k] & UM) | (x[k + 1] & LM);
        v = x[k + 156] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
    }
    __syncthreads();
    if (k < 156) x[k] = v;
    __syncthreads();
    if (k >= 156 && k < 311) {
        const u64 y = (x[k] & UM) | (x[k + 1] & LM);
        v = x[k - 156] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
    }
    __syncthreads();
    if (k >= 156 && k < 311) x[k] = v;
    __syncthreads();
    if (k == 0) {
        const u64 y = (x[311] & UM) | (x[0] & LM);
        x[311] = x[155] ^ (y >> 1) ^ ((y & 1ull) ? A : 0ull);
    }
    __syncthreads();
}

// OR `bits` into word `col` of `keys`, combining lanes that target the same
// column first (consecutive outputs of the stream hit the same column).
template <class K>
__device__ __forceinline__ void or_key(K* keys, u64 col, K bits, bool valid);

template <>
__device__ __forceinline__ void or_key<u32>(u32* keys, u64 col, u32 bits, bool valid) {
    const u32 active = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const u32 peers = __match_any_sync(active, static_cast<unsigned long long>(col));
    const u32 acc = __reduce_or_sync(peers, bits);
    if ((peers & lanemask_lt()) == 0 && acc) atomicOr(keys + col, acc);
}

template <>
__device__ __forceinline__ void or_key<u64>(u64* keys, u64 col, u64 bits, bool valid) {
    const u32 active = __ballot_sync(0xffffffffu, valid);
    if (!valid) return;
    const u32 peers = __match_any_sync(active, static_cast<unsigned long long>(col));
    const u32 lo = __reduce_or_sync(peers, u32(bits));
    const u32 hi = __reduce_or_sync(peers, u32(bits >> 32));
    const u64 acc = (u64(hi) << 32) | lo;
    if ((peers & lanemask_lt()) == 0 && acc)
        atomicOr(reinterpret_cast<unsigned long long*>(keys + col), static_cast<unsigned long long>(acc));
}

// The per-run XOR constant c = ~rp & mask with rp_s = (sign * y[i_s] > 0)
// (resp_positive, search.cpp:444-447); z-key = x-key ^ c.
template <class K>
__global__ void resp_xorc(const u32* __restrict__ rows, int M, const double* __restrict__ y,
                          const int8_t* __restrict__ run_sign, u32 B, K* __restrict__ xorc) {
    const u32 b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    u64 rp = 0;
    for (int s = 0; s < M; ++s) {
        const double v = y[rows[u64(b) * M + s]];
        if ((run_sign[b] > 0 ? v : -v) > 0.0) rp |= 1ull << s;
    }
    const u64 mask = M >= 64 ? ~0ull : ((1ull << M) - 1);
    xorc[b] = K(~rp & mask);
}

template <class K>
__global__ void popc_count(const K* __restrict__ m, u64 count, u32* __restrict__ out) {
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < count; t += u64(gridDim.x) * blockDim.x)
        out[t] = __popcll(static_cast<unsigned long long>(m[t]));
}

// Sign-transform coins: the t-th zero entry of run b in (j, s) order takes
// bit 0 of the t-th output of the run's stream (search.cpp:457-463).
template <class K>
__global__ void __launch_bounds__(kMtThreads) sign_coins(const u64* __restrict__ mt_state, u64 p,
                                                         const K* __restrict__ zmask,
                                                         const u32* __restrict__ zoff /*[B*p+1] global excl scan*/,
                                                         K* __restrict__ keys) {
    __shared__ u64 x[kMtN];
    __shared__ int pos_s;
    const u64 b = blockIdx.x;
    const u64* st = mt_state + b * (kMtN + 1);
    for (int i = threadIdx.x; i < kMtN; i += blockDim.x) x[i] = st[i];
    if (threadIdx.x == 0) pos_s = int(st[kMtN]);
    __syncthreads();
    const u32 base = zoff[b * p];
    const u64 total = u64(zoff[(b + 1) * p]) - base;
    int pos = pos_s;
    for (u64 t0 = 0; t0 < total;) {
        if (pos >= kMtN) {
            mt_twist(x);
            pos = 0;
        }
        const u64 chunk = minu(u64(kMtN - pos), total - t0);
        const bool valid = threadIdx.x < chunk;
        u64 col = 0;
        K bit = 0;
        if (valid) {
            const u64 t = t0 + threadIdx.x;
            const u64 z = mt_temper(x[pos + threadIdx.x]);
            // column: last j with zoff[b*p + j] - base <= t
            u64 lo = 0, hi = p;
            while (hi - lo > 1) {
                const u64 mid = (lo + hi) >> 1;
                if (u64(zoff[b * p + mid] - base) <= t) lo = mid; else hi = mid;
            }
            col = lo;
            u64 m = static_cast<u64>(zmask[b * p + col]);
            u64 r = t - (zoff[b * p + col] - base);
            while (r--) m &= m - 1;
            const int s = __ffsll(static_cast<long long>(m)) - 1;
            bit = K(z & 1ull) << s;
        }
        or_key<K>(keys + b * p, col, bit, valid && bit != 0);
        t0 += chunk;
        pos += int(chunk);
        __syncthreads();
    }
}

// Unbiased transform: output t = j*M + s of the run's stream decides entry
// (j, s): plus = uniform_unit < (v + 1) / 2 in fp64 (search.cpp:455-456).
template <class K>
__global__ void __launch_bounds__(kMtThreads) unbiased_keys(const u64* __restrict__ mt_state, u64 p,
                                                            const u32* __restrict__ rows, int M,
                                                            const double* __restrict__ Xr64, K* __restrict__ keys) {
    __shared__ u64 x[kMtN];
    __shared__ u32 srow[64];
    __shared__ int pos_s;
    const u64 b = blockIdx.x;
    const u64* st = mt_state + b * (kMtN + 1);
    for (int i = threadIdx.x; i < kMtN; i += blockDim.x) x[i] = st[i];
    if (threadIdx.x < M) srow[threadIdx.x] = rows[b * M + threadIdx.x];
    if (threadIdx.x == 0) pos_s = int(st[kMtN]);
    __syncthreads();
    const u64 total = p * u64(M);
    int pos = pos_s;
    K* kb = keys + b * p;
    for (u64 t0 = 0; t0 < total;) {
        if (pos >= kMtN) {
            mt_twist(x);
            pos = 0;
        }
        const u64 chunk = minu(u64(kMtN - pos), total - t0);
        const bool valid = threadIdx.x < chunk;
        u64 col = 0;
        K bit = 0;
        if (valid) {
            const u64 t = t0 + threadIdx.x;
            const u64 z = mt_temper(x[pos + threadIdx.x]);
            col = t / u64(M);
            const int s = int(t - col * u64(M));
            const double v = __ldg(Xr64 + u64(srow[s]) * p + col);
            const double u = double(z >> 11) * 0x1.0p-53;
            if (u < (v + 1.0) / 2.0) bit = K(1) << s;
        }
        or_key<K>(kb, col, bit, valid && bit != 0);
        t0 += chunk;
        pos += int(chunk);
        __syncthreads();
    }
}

// ---- dataset preparation for real X ----

// Column-major sign bits of X (the sign transform's t(x) in {-1, 0, 1},
// search.cpp:456-462): bit i of word w of column j is x[64w + i, j] > 0
// (Spos) / != 0 (Snz), W words per column, for the bit-plane verify; the
// same bits of (x > 0) and (x == 0) with the Wp-word stride of the binary
// layout (Tpos, Tzero; zero padded) for the row-plane transposes the
// projection reads; flags: bit 0 any zero, bit 1 any entry outside [-1, 1]
// (or NaN: the unbiased transform's domain check, search.cpp:417-434).
// One warp per column, ballots per word. T = double (x_real) or float
// (x_real32: double(x) compares the same).
template <class T>
__global__ void sign_cols(const T* __restrict__ X, u64 ld, u64 n, u64 p, u64 Wn, u64 Wp, u64* __restrict__ Spos,
                          u64* __restrict__ Snz, u64* __restrict__ Tpos, u64* __restrict__ Tzero,
                          u32* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const u64 nw = (u64(gridDim.x) * blockDim.x) >> 5;
    u32 fl = 0;
    for (u64 j = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < p; j += nw) {
        const T* col = X + j * ld;
        for (u64 w = 0; w < Wp; ++w) {
            const u64 i0 = 64 * w + lane, i1 = i0 + 32;
            const bool in0 = i0 < n, in1 = i1 < n;
            const double a = in0 ? double(col[i0]) : 1.0, b = in1 ? double(col[i1]) : 1.0;
            const u64 pos = u64(__ballot_sync(0xffffffffu, in0 && a > 0.0)) |
                            (u64(__ballot_sync(0xffffffffu, in1 && b > 0.0)) << 32);
            const u64 zer = u64(__ballot_sync(0xffffffffu, in0 && a == 0.0)) |
                            (u64(__ballot_sync(0xffffffffu, in1 && b == 0.0)) << 32);
            const u64 nz = u64(__ballot_sync(0xffffffffu, in0 && a != 0.0)) |
                           (u64(__ballot_sync(0xffffffffu, in1 && b != 0.0)) << 32);
            const bool out = (in0 && !(a >= -1.0 && a <= 1.0)) || (in1 && !(b >= -1.0 && b <= 1.0));
            if (zer) fl |= 1u;
            if (__any_sync(0xffffffffu, out)) fl |= 2u;
            if (lane == 0) {
                if (w < Wn) {
                    Spos[j * Wn + w] = pos;
                    Snz[j * Wn + w] = nz;
                }
                Tpos[j * Wp + w] = pos;
                Tzero[j * Wp + w] = zer;
            }
        }
    }
    if (lane == 0 && fl) atomicOr(flags, fl);
}

// fp32 columns [p][n] -> [p][n4] (zero padded rows)
__global__ void pad_f32_cols(const float* __restrict__ src, u64 n, u64 p, u64 n4, float* __restrict__ dst) {
    const u64 total = p * n4;
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += u64(gridDim.x) * blockDim.x) {
        const u64 j = t / n4, i = t - j * n4;
        dst[t] = i < n ? src[j * n + i] : 0.f;
    }
}

__global__ void to_f32_cols(const double* __restrict__ Xc64, u64 n, u64 p, u64 n4, float* __restrict__ Xc32) {
    const u64 total = p * n4;
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += u64(gridDim.x) * blockDim.x) {
        const u64 j = t / n4, i = t - j * n4;
        Xc32[t] = i < n ? float(Xc64[j * n + i]) : 0.f;
    }
}

// X [p][ld] column-major (fp64, or fp32 widened exactly) -> Xr64 [n][p]
// (32x32 tiles through shared memory): the unbiased transform's fp64 rows,
// built on the first unbiased search.
template <class T>
__global__ void transpose_f64(const T* __restrict__ Xc, u64 ld, u64 n, u64 p, double* __restrict__ Xr64) {
    __shared__ double tile[32][33];
    const u64 j0 = u64(blockIdx.x) * 32, i0 = u64(blockIdx.y) * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const u64 j = j0 + r, i = i0 + threadIdx.x;
        tile[r][threadIdx.x] = (j < p && i < n) ? double(Xc[j * ld + i]) : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const u64 i = i0 + r, j = j0 + threadIdx.x;
        if (i < n && j < p) Xr64[i * p + j] = tile[threadIdx.x][r];
    }
}

} // namespace real
} // namespace xyzb
