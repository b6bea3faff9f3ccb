// All-pairs agreement counts on the 5th-generation tensor cores (sm_100a).
//
// agree(j, k) over the rows with y != 0 is an inner product of +-1 vectors:
// with A_ij = +1 / -1 for bit(X_ij) = 1 / 0 and B_ik = +1 / -1 for
// bit(X_ik ^ Y_i) = 1 / 0 (0 where y_i = 0 or i >= n),
//     G_jk = sum_i A_ij B_ik = nz - 2 agree(j, k),   nz = #{i : y_i != 0},
// so the exhaustive oracle is one int8 Gram product G = A B^T with exact s32
// accumulation — GEMM-shaped, unlike the sparse candidate verification of
// the search. Per CTA tile of 128 (j) x 256 (k) pairs:
//   - TMA (cp.async.bulk.tensor.2d, 128-byte swizzle) streams 128-byte K
//     slices of A and B into a 3-stage shared-memory ring (mbarrier
//     complete_tx);
//   - one thread issues tcgen05.mma.cta_group::1.kind::i8 (M=128, N=256,
//     K=32 per instruction) with the s32 accumulator in TMEM (256 columns)
//     and releases each stage with tcgen05.commit;
//   - four warps read the accumulator back with tcgen05.ld.32x32b.x32 (warp w
//     owns TMEM lanes 32w..32w+31 = tile rows) and apply the same epilogue
//     as the CUDA-core kernel (histogram of agree or emission above a cut).
// A persistent grid (one CTA per SM, 144 KB of stages) walks the tiles of
// the upper triangle.
#pragma once

#include <cuda.h>

#include "brute.cuh"
#include "common.cuh"

namespace xyzb {
namespace brute {

constexpr int kTcM = 128;
constexpr int kTcN = 256;
constexpr int kTcKB = 128;  // bytes (int8 elements) of K per stage = one 128 B swizzle row
constexpr int kTcStages = 3;
constexpr int kTcThreads = 128;
constexpr u32 kTcStageA = kTcM * kTcKB;
constexpr u32 kTcStageB = kTcN * kTcKB;
// stages (1024-byte aligned, + slack) then the agree histogram
constexpr u32 kTcSmem = kTcStages * (kTcStageA + kTcStageB) + 1024 + (kSmemHistMax + 1) * 4;

__device__ __forceinline__ u32 smem_addr(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// Bounded wait: a pipeline that never completes traps (a kernel error the
// host reports) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(u32 bar, u32 phase) {
    u32 done = 0;
    for (u64 spin = 0; !done; ++spin) {
        if (spin > (u64(1) << 31)) asm volatile("trap;");
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    }
}
__device__ __forceinline__ void tma_load_2d(u32 dst, const CUtensorMap* map, int c0, int c1, u32 bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<u64>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
// K-major operand in the 128-byte-swizzled canonical layout (8-row groups of
// 1024 B): start address, LBO = 1 (unused), SBO = 1024 B, version 1,
// layout SWIZZLE_128B.
__device__ __forceinline__ u64 sw128_desc(u32 saddr) {
    return u64((saddr & 0x3ffffu) >> 4) | (u64(1) << 16) | (u64(1024 >> 4) << 32) | (u64(1) << 46) |
           (u64(2) << 61);
}
// kind::i8 instruction descriptor: D s32, A and B signed int8, both K-major,
// N = 256, M = 128.
constexpr u32 kIdescI8 = (2u << 4) | (1u << 7) | (1u << 10) | (u32(kTcN >> 3) << 17) | (u32(kTcM >> 4) << 24);

__device__ __forceinline__ void mma_i8(u32 tmem_d, u64 adesc, u64 bdesc, u32 accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdescI8), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(u32 bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(u32 taddr, u32 (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// +-1 int8 operands, K-major [p][Kp] (Kp a multiple of 128, zero beyond n).
__global__ void make_pm1(const u64* __restrict__ Xc, u64 Wp, u64 p, u64 n, u64 Kp, const u64* __restrict__ Yw,
                         const u64* __restrict__ NZ, int8_t* __restrict__ A, int8_t* __restrict__ B) {
    const u64 total = p * (Kp / 8);  // 8 rows (one byte of bits) per step
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += u64(gridDim.x) * blockDim.x) {
        const u64 j = t / (Kp / 8), i0 = (t % (Kp / 8)) * 8;
        u64 a8 = 0, b8 = 0;
        if (i0 < n) {
            const u64 w = i0 >> 6, sh = i0 & 63;
            const u32 xb = u32(Xc[j * Wp + w] >> sh) & 0xffu;
            const u32 yb = u32(Yw[w] >> sh) & 0xffu, nz = u32(NZ[w] >> sh) & 0xffu;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const bool in = i0 + q < n;
                const u64 av = in ? ((xb >> q) & 1u ? 0x01ull : 0xffull) : 0ull;
                const u64 bv = in && ((nz >> q) & 1u) ? ((((xb ^ yb) >> q) & 1u) ? 0x01ull : 0xffull) : 0ull;
                a8 |= av << (8 * q);
                b8 |= bv << (8 * q);
            }
        }
        reinterpret_cast<u64*>(A)[t] = a8;
        reinterpret_cast<u64*>(B)[t] = b8;
    }
}

// Warp-specialised persistent kernel: warp 0 = TMA producer, warp 1 = MMA
// issuer, warps 2-5 = epilogue. The accumulator is double-buffered in TMEM
// (2 x 256 columns), so the epilogue of tile i overlaps the MMAs of tile
// i + 1; the stage ring is shared by consecutive tiles.
constexpr int kTcWarps = 6;
constexpr int kTcEpiWarps = 4;
constexpr u32 kTcHistMax = 8192;  // agree bins in shared memory (n <= this), else global atomics
constexpr int kTcStages4 = 4;
constexpr u32 kTcSmem2 = kTcStages4 * (kTcStageA + kTcStageB) + 1024 + (kTcHistMax + 1) * 4;

template <bool EMIT>
__global__ void __launch_bounds__(kTcWarps * 32, 1) all_pairs_tc2(const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmB, u32 p,
                                                                  u32 n, u32 nz, u32 Kp,
                                                                  unsigned long long* __restrict__ hist, u32 cutoff,
                                                                  PairOut* __restrict__ out, u32* __restrict__ nout,
                                                                  u32 out_cap) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ __align__(8) u64 full_bar[kTcStages4], empty_bar[kTcStages4], tfull_bar[2], tempty_bar[2];
    __shared__ u32 tmem_holder;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u32 base = smem_addr(dsm);
    const u32 sbase = (base + 1023u) & ~1023u;
    auto sA = [&](u32 s) { return sbase + s * (kTcStageA + kTcStageB); };
    auto sB = [&](u32 s) { return sA(s) + kTcStageA; };
    u32* shist = reinterpret_cast<u32*>(dsm + (sbase - base) + kTcStages4 * (kTcStageA + kTcStageB));
    const bool smem_hist = !EMIT && n <= kTcHistMax;
    if (smem_hist)
        for (u32 i = threadIdx.x; i <= n; i += kTcWarps * 32) shist[i] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages4; ++s) {
            mbar_init(smem_addr(&full_bar[s]), 1);
            mbar_init(smem_addr(&empty_bar[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_addr(&tfull_bar[b]), 1);
            mbar_init(smem_addr(&tempty_bar[b]), kTcEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<u64>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<u64>(&tmB)) : "memory");
    }
    if (warp == 1) {  // TMEM: two accumulators of 256 s32 columns (whole warp)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_holder)),
                     "r"(u32(2 * kTcN)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const u32 tmem = tmem_holder;
    const u32 nj = (p + kTcM - 1) / kTcM, nk = (p + kTcN - 1) / kTcN;
    const u32 nkb = Kp / kTcKB;
    // tile order: bands of kBand row tiles, row tile fastest inside a band, so
    // the ~148 tiles in flight share a few A and B tiles in L2 (the operands,
    // 2 x p x Kp bytes, do not fit in L2)
    constexpr u32 kBand = 8;
    const u64 ntiles = u64((nj + kBand - 1) / kBand) * kBand * nk;
    auto tile_of = [&](u64 t, u32& tj, u32& tk) {
        const u64 band = t / (u64(kBand) * nk), r = t % (u64(kBand) * nk);
        tk = u32(r / kBand);
        tj = u32(band * kBand + r % kBand);
    };
    auto skip = [&](u64 t) {
        u32 tj, tk;
        tile_of(t, tj, tk);
        return tj >= nj || tk * kTcN + kTcN <= tj * kTcM + 1;  // no pair with k > j
    };
    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer =====
            u32 g = 0;
            for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
                if (skip(t)) continue;
                u32 tj, tk;
                tile_of(t, tj, tk);
                const int j0 = int(tj) * kTcM, k0 = int(tk) * kTcN;
                for (u32 kb = 0; kb < nkb; ++kb, ++g) {
                    const u32 s = g % kTcStages4;
                    if (g >= u32(kTcStages4)) mbar_wait(smem_addr(&empty_bar[s]), ((g / kTcStages4) - 1) & 1);
                    mbar_expect_tx(smem_addr(&full_bar[s]), kTcStageA + kTcStageB);
                    tma_load_2d(sA(s), &tmA, int(kb * kTcKB), j0, smem_addr(&full_bar[s]));
                    tma_load_2d(sB(s), &tmB, int(kb * kTcKB), k0, smem_addr(&full_bar[s]));
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ===== MMA issuer =====
            u32 g = 0, lt = 0;
            for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
                if (skip(t)) continue;
                const u32 b = lt & 1, use = lt >> 1;
                if (use >= 1) mbar_wait(smem_addr(&tempty_bar[b]), (use - 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const u32 acc = tmem + b * kTcN;
                for (u32 kb = 0; kb < nkb; ++kb, ++g) {
                    const u32 s = g % kTcStages4;
                    mbar_wait(smem_addr(&full_bar[s]), (g / kTcStages4) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                    for (int kk = 0; kk < kTcKB / 32; ++kk)
                        mma_i8(acc, sw128_desc(sA(s) + kk * 32), sw128_desc(sB(s) + kk * 32), (kb | kk) != 0);
                    mma_commit(smem_addr(&empty_bar[s]));
                }
                mma_commit(smem_addr(&tfull_bar[b]));
                ++lt;
            }
        }
    } else {  // ===== epilogue: warps 2-5, TMEM lane quarter = warp % 4 =====
        const u32 quarter = u32(warp & 3);
        u32 lt = 0;
        for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
            if (skip(t)) continue;
            const u32 b = lt & 1, use = lt >> 1;
            u32 tj, tk;
            tile_of(t, tj, tk);
            const u32 j0 = tj * kTcM, k0 = tk * kTcN;
            mbar_wait(smem_addr(&tfull_bar[b]), use & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const u32 j = j0 + quarter * 32 + u32(lane);
#pragma unroll 1
            for (int c = 0; c < kTcN / 32; ++c) {
                u32 v[32];
                tmem_ld32(tmem + ((quarter * 32) << 16) + b * kTcN + u32(c * 32), v);
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const u32 k = k0 + u32(c * 32 + q);
                    const u32 agree = (nz - v[q]) >> 1;  // G = nz - 2 agree
                    const bool valid = j < k && k < p;
                    if (EMIT) {
                        const bool keep = valid && agree >= cutoff;
                        const u32 ball = __ballot_sync(0xffffffffu, keep);
                        if (ball) {
                            const int leader = __ffs(ball) - 1;
                            u32 b0 = 0;
                            if (lane == leader) b0 = atomicAdd(nout, __popc(ball));
                            b0 = __shfl_sync(0xffffffffu, b0, leader);
                            if (keep) {
                                const u32 slot = b0 + __popc(ball & lanemask_lt());
                                if (slot < out_cap) out[slot] = PairOut{j, k, agree, 0u};
                            }
                        }
                    } else if (valid) {
                        if (smem_hist) atomicAdd(&shist[agree], 1u);
                        else atomicAdd(hist + agree, 1ull);
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&tempty_bar[b])) : "memory");
            ++lt;
        }
    }
    __syncthreads();
    if (smem_hist)
        for (u32 i = threadIdx.x; i <= n; i += kTcWarps * 32)
            if (shist[i]) atomicAdd(hist + i, static_cast<unsigned long long>(shist[i]));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(u32(2 * kTcN)));
}

}  // namespace brute
}  // namespace xyzb
