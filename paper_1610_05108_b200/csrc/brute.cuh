// Exhaustive all-pairs strengths on the device: the GPU
// counterpart of oracle::brute_force_search (oracle.hpp:36-41,
// oracle.cpp:24-59, 84-91), which the reference guards at p <= 20000.
//
// agree(j, k) = #rows with y_i == x_ij * x_ik = popc((X_j ^ Z_k) & NZ) over
// the packed words, Z_k = X_k ^ Y (Y bit = y_i > 0) and NZ = rows with
// y_i != 0 (a zero response never agrees, as in scalar_strength). A
// persistent grid walks 64 x 64 tiles of the upper triangle; each thread
// owns a 4 x 4 block of pairs, columns staged in shared memory word-major so
// a warp's loads are contiguous. Two modes:
//   HIST: exact histogram of agree over [0, n] (per-CTA shared counters,
//         flushed once) — the host derives the reference's strength
//         histogram, the gamma cut and the top-K cutoff from it exactly;
//   EMIT: every pair with agree >= cutoff appended as (j, k, agree).
#pragma once

#include "common.cuh"

namespace xyzb {
namespace brute {

constexpr int kTile = 64;      // columns per tile side
constexpr int kChunk = 16;     // words per shared-memory stage
constexpr int kThreads = 256;  // 16 x 16 threads, 4 x 4 pairs each
constexpr u32 kSmemHistMax = 12288;  // agree bins kept in shared memory (n <= this)

// Z = X ^ Y per column word, NZ mask.
__global__ void make_z(const u64* __restrict__ Xc, u64 Wp, u64 W, u64 p, const u64* __restrict__ Yw,
                       u64* __restrict__ Zc) {
    const u64 total = p * Wp;
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += u64(gridDim.x) * blockDim.x) {
        const u64 w = t % Wp;
        Zc[t] = w < W ? Xc[t] ^ Yw[w] : 0ull;
    }
}

struct PairOut {
    u32 j, k, agree, pad;
};

template <bool EMIT>
__global__ void __launch_bounds__(kThreads) all_pairs(const u64* __restrict__ Xc, const u64* __restrict__ Zc,
                                                      const u64* __restrict__ NZ, u64 Wp, u64 W, u32 p, u32 n,
                                                      unsigned long long* __restrict__ hist, u32 cutoff,
                                                      PairOut* __restrict__ out, u32* __restrict__ nout,
                                                      u32 out_cap) {
    __shared__ __align__(16) u64 xs[kChunk][kTile];
    __shared__ __align__(16) u64 zs[kChunk][kTile];
    __shared__ u64 nzs[kChunk];
    extern __shared__ u32 shist[];  // n + 1 bins (HIST with n <= kSmemHistMax)
    const bool smem_hist = !EMIT && n <= kSmemHistMax;
    if (smem_hist)
        for (u32 i = threadIdx.x; i <= n; i += kThreads) shist[i] = 0;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const u32 nb = (p + kTile - 1) / kTile;
    const u64 ntiles = u64(nb) * nb;
    for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const u32 bj = u32(t / nb), bk = u32(t % nb);
        if (bk < bj) continue;  // upper triangle (uniform per CTA)
        const u32 j0 = bj * kTile, k0 = bk * kTile;
        u32 acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = 0;
        for (u64 w0 = 0; w0 < W; w0 += kChunk) {
            __syncthreads();
            // stage kChunk words of 64 + 64 columns, word-major
            for (int i = threadIdx.x; i < kChunk * kTile; i += kThreads) {
                const int c = i / kChunk, w = i % kChunk;
                const u64 wi = w0 + w;
                const u32 jc = j0 + c, kc = k0 + c;
                xs[w][c] = (wi < W && jc < p) ? Xc[u64(jc) * Wp + wi] : 0ull;
                zs[w][c] = (wi < W && kc < p) ? Zc[u64(kc) * Wp + wi] : 0ull;
            }
            if (threadIdx.x < kChunk) nzs[threadIdx.x] = (w0 + threadIdx.x < W) ? NZ[w0 + threadIdx.x] : 0ull;
            __syncthreads();
#pragma unroll 4
            for (int w = 0; w < kChunk; ++w) {
                const u64 m = nzs[w];
                u64 x[4], z[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) x[a] = xs[w][ty * 4 + a];
#pragma unroll
                for (int b = 0; b < 4; ++b) z[b] = zs[w][tx * 4 + b];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b] += __popcll((x[a] ^ z[b]) & m);
            }
        }
        // epilogue: pairs j < k inside [0, p)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const u32 j = j0 + ty * 4 + a;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const u32 k = k0 + tx * 4 + b;
                const bool valid = j < k && k < p;
                if (EMIT) {
                    const bool keep = valid && acc[a][b] >= cutoff;
                    const u32 ball = __ballot_sync(0xffffffffu, keep);
                    if (ball) {
                        const int lane = threadIdx.x & 31, leader = __ffs(ball) - 1;
                        u32 base = 0;
                        if (lane == leader) base = atomicAdd(nout, __popc(ball));
                        base = __shfl_sync(0xffffffffu, base, leader);
                        if (keep) {
                            const u32 slot = base + __popc(ball & lanemask_lt());
                            if (slot < out_cap) out[slot] = PairOut{j, k, acc[a][b], 0u};
                        }
                    }
                } else if (valid) {
                    if (smem_hist) atomicAdd(&shist[acc[a][b]], 1u);
                    else atomicAdd(hist + acc[a][b], 1ull);
                }
            }
        }
    }
    if (smem_hist) {
        __syncthreads();
        for (u32 i = threadIdx.x; i <= n; i += kThreads)
            if (shist[i]) atomicAdd(hist + i, static_cast<unsigned long long>(shist[i]));
    }
}

inline u32 all_pairs_grid() { return kSMs * 4; }

}  // namespace brute
}  // namespace xyzb
