// libxyzb.so — the B200 xyz interaction-search engine behind include/xyzb.h.
//
// Host orchestration of one search (the three xyz::xyz_search overloads,
// proj/core/src/search.cpp:325-506, with run_search / run_pass,
// search.cpp:65-111,295-321):
//   1. validate (SearchConfig::validate, search.cpp:119-134, plus the
//      per-overload checks) before any device work, same messages;
//   2. host draws per run (make_stream(seed, offset + rep), draw_subsample);
//   3. batches of runs: project -> segmented radix sort -> bucket join +
//      guard -> canonical-work scan -> verify (device, one stream);
//   4. device merge: first-occurrence dedup, reference order, top-K;
//   5. counters and the optional complexity estimate.
// No CPU fallback: every stage runs on the GPU; without a device the calls
// fail with XYZB_E_CUDA.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <condition_variable>
#include <thread>
#include <string>
#include <vector>

#include "../../include/xyzb.h"
#include "../../include/xyzb_testing.h"
#include "brute.cuh"
#include "brute_tc.cuh"
#include "cta_group.cuh"
#include "common.cuh"
#include "draws.cuh"
#include "host_rng.hpp"
#include "merge_kernels.cuh"
#include "msplit_group.cuh"
#include "part_group.cuh"
#include "topk_kernels.cuh"
#include "radix_sort.cuh"
#include "run_sort.cuh"
#include "real_kernels.cuh"
#include "scan.cuh"
#include "search_kernels.cuh"
#include "binned_verify.cuh"

using namespace xyzb;

namespace {

// ------------------------------------------------------------ test options --
// Process-wide options the unit tests set through xyzb_test_set_option
// (include/xyzb_testing.h) to force rare paths — buffer regrowth, multi-batch
// runs, a grouping path outside its default range, the multi-kernel merge,
// the fp32 verify beside the sign-bit one. 0 = the engine's own choice.
struct TestOptions {
    std::atomic<long long> batch_entries{0}, hit_cap{0}, item_cap{0}, pair_cap{0}, grouping{0}, merge_large{0},
        sign_verify_off{0}, trace{0}, brute_cuda{0}, binned{0}, binned_wshift{0}, binned_cap{0}, one_pass_join{0}, part_fixed{0};
};
TestOptions& topt() {
    static TestOptions* o = new TestOptions();  // leaked on purpose (outlives static destructors)
    return *o;
}
enum { kGroupAuto = 0, kGroupSort = 1, kGroupPart = 2, kGroupMsplit = 3 };

// ------------------------------------------------------------ buffers --

// Caching allocator: device blocks (per device) and pinned host blocks are
// returned to a free list instead of cudaFree / cudaFreeHost, so datasets
// created per call (the end-to-end path) and regrown scratch do not pay
// cudaMalloc latency. On allocation failure the cache is trimmed and retried.
struct BlockPool {
    std::mutex mu;
    std::multimap<size_t, std::pair<int, void*>> free_;  // size -> (device or -1 host, ptr)
    static size_t granule(size_t b) { return b <= (1u << 20) ? round_pow2(b) : (b + (1u << 20) - 1) & ~size_t((1u << 20) - 1); }
    static size_t round_pow2(size_t b) {
        size_t r = 256;
        while (r < b) r <<= 1;
        return r;
    }
    void* take(size_t& b, int dev) {
        b = granule(b);
        {
            std::lock_guard<std::mutex> lk(mu);
            // a cached block at most 1/8 (+ 1 MiB) larger: a 50 MB request must not take the 80 MB block
            // another buffer of the next search needs (a pool miss costs a synchronising cudaMalloc)
            for (auto it = free_.lower_bound(b); it != free_.end() && it->first <= b + b / 8 + (1u << 20); ++it) {
                if (it->second.first == dev) {
                    void* p = it->second.second;
                    b = it->first;
                    free_.erase(it);
                    return p;
                }
            }
        }
        void* p = nullptr;
        if (topt().trace.load()) std::fprintf(stderr, "[xyzb] pool miss: %s %zu bytes\n", dev >= 0 ? "cudaMalloc" : "cudaMallocHost", b);
        cudaError_t err = dev >= 0 ? cudaMalloc(&p, b) : cudaMallocHost(&p, b);
        if (err != cudaSuccess) {
            cudaGetLastError();
            trim(dev);
            err = dev >= 0 ? cudaMalloc(&p, b) : cudaMallocHost(&p, b);
        }
        if (err != cudaSuccess)
            throw cuda_error(std::string(dev >= 0 ? "cudaMalloc(" : "cudaMallocHost(") + std::to_string(b) +
                             "): " + cudaGetErrorString(err));
        return p;
    }
    void give(void* p, size_t b, int dev) {
        std::lock_guard<std::mutex> lk(mu);
        free_.emplace(b, std::make_pair(dev, p));
    }
    void trim(int dev) {
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = free_.begin(); it != free_.end();) {
            if (it->second.first == dev) {
                if (dev >= 0) cudaFree(it->second.second); else cudaFreeHost(it->second.second);
                it = free_.erase(it);
            } else {
                ++it;
            }
        }
    }
};

BlockPool& pool() {
    static BlockPool* p = new BlockPool();  // intentionally leaked: outlives static destructors
    return *p;
}

// The stream the calling thread's current API call issues its work on
// (StreamScope): device buffers remember it, so returning a block to the pool
// waits for that stream only, and calls on different datasets from different
// host threads do not serialise on a device-wide synchronisation.
thread_local cudaStream_t tl_stream = nullptr;
thread_local cudaStream_t tl_drained = nullptr;  // a stream already synchronised (dataset teardown)
struct StreamScope {
    cudaStream_t prev;
    explicit StreamScope(cudaStream_t s) : prev(tl_stream) { tl_stream = s; }
    ~StreamScope() { tl_stream = prev; }
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int dev = 0;
    cudaStream_t st = nullptr;  // the stream that used the block last (null: unknown)
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            // the block may still be in use by queued work: wait for its stream
            // (or the whole device when unknown) before the pool hands it out again
            if (!st || st != tl_drained) {
                int cur = 0;
                cudaGetDevice(&cur);
                cudaSetDevice(dev);
                if (st) {
                    cudaStreamSynchronize(st);
                } else {
                    if (topt().trace.load()) std::fprintf(stderr, "[xyzb] device-wide sync on release (%zu bytes)\n", bytes);
                    cudaDeviceSynchronize();
                }
                cudaSetDevice(cur);
            }
            pool().give(p, bytes, dev);
        }
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t b) {
        if (b <= bytes) {
            if (tl_stream) st = tl_stream;
            return;
        }
        release();
        XYZB_CUDA(cudaGetDevice(&dev));
        size_t got = std::max<size_t>(b, 256);
        p = pool().take(got, dev);
        bytes = got;
        st = tl_stream;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

struct HostBuf {  // pinned
    void* p = nullptr;
    size_t bytes = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() {
        if (p) pool().give(p, bytes, -1);
    }
    void ensure(size_t b) {
        if (b <= bytes) return;
        if (p) pool().give(p, bytes, -1);
        size_t got = std::max<size_t>(b, 256);
        p = pool().take(got, -1);
        bytes = got;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

u64 round_up(u64 a, u64 m) { return (a + m - 1) / m * m; }


// NVTX range over a host-side region (search, batch, stage launches): the
// engine's phases on an Nsight Systems timeline; free without a tool attached.
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// event-timed stage accounting on the dataset stream
struct StageClock {
    cudaStream_t st;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> spans;
    std::vector<cudaEvent_t> pool;
    size_t used = 0;
    cudaEvent_t get() {
        if (used == pool.size()) {
            cudaEvent_t e;
            XYZB_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[used++];
    }
    cudaEvent_t mark() {
        cudaEvent_t e = get();
        XYZB_CUDA(cudaEventRecord(e, st));
        return e;
    }
    void span(int stage, cudaEvent_t a, cudaEvent_t b) { spans.push_back({stage, {a, b}}); }
    void reset() {
        spans.clear();
        used = 0;
    }
    ~StageClock() {
        for (auto e : pool) cudaEventDestroy(e);
    }
};

} // namespace

// ------------------------------------------------------------ dataset --

struct xyzb_dataset {
    int device = 0;
    cudaStream_t stream = nullptr;
    u64 n = 0, p = 0;
    bool binary = true;
    u64 W = 0, Wp = 0, P32 = 0, n4 = 0;
    // binary
    DevBuf Xc;  // u64 [p][Wp]
    DevBuf Xr;  // u32 [n][P32]
    // real
    DevBuf Xc32;    // f32 [p][n4]
    DevBuf Xsrc64;  // f64 [p][n]: the caller's fp64 values (x_real), source of the unbiased transform's rows
    DevBuf Xr64;    // f64 [n][p]: built on the first unbiased search (ensure_xr64)
    bool f32_src = false;  // created from x_real32 (Xc32 holds the exact values)
    DevBuf Xpos, Xzero;  // u32 [n][P32]
    DevBuf Spos, Snz;    // u64 [p][W] column sign bits (x > 0, x != 0): the sign transform's bit-plane verify
    bool has_zero = false, in_unit = true;
    // response (per search)
    DevBuf yk_bits, spos, sneg, wabs, yreal, yreal32;
    // batch scratch
    DevBuf keys[2], vals[2], keys_x, hist, items, table, partial, rows, rid, rsign, streams, xorc, tot, work_run, nblocks, cum;
    DevBuf pairs, npairs, table_end, perm, gtab, slots, pgrp, pent, povf, yplanes;
    DevBuf zmask, zcount, zoff, zcnt_n, mt_state;
    // search scratch
    DevBuf enumerated, verified, sign_by_rid, hits, hit_count, rmin;
    DevBuf tkeys, tvals, keep, kpos, kept, kept_order, fin, fin_order, tie, kbufA, kbufB, vbufA, vbufB, topidx, hcount;
    DevBuf pairs_dev, strengths_dev;
    // top-K over all candidates (topk_kernels.cuh)
    DevBuf tk_state, tk_hist, tk_dhist, tk_sint, tk_table, hits2, tk_cnt2;
    // binned verify (binned_verify.cuh): per-window regions, bins by x-side tile, cursors
    DevBuf bin_xy, bin_s, bin_wcnt, bin_b, bin_d, bin_cnt, bin_start, bin_fill, bin_boff, bin_ovf, bin_ovfn, bin_zero;
    u64 bin_hint = 0;      // mean bucket fill of the last binned search on this dataset (sizes the buckets)
    u64 bin_ovf_hint = 0;  // overflow-list size that last sufficed
    HostBuf h_rows, h_state, h_small, h_merge, h_status, h_planes;
    StageClock clock;
    u32 hit_cap = 1u << 16;
    int part_fixed_fails = 0;  // searches of this dataset whose fixed-capacity partition pass overflowed
    // X replicated on further devices (xyzb_problem.devices[1..]): the search shards its runs over them
    std::vector<std::unique_ptr<xyzb_dataset>> replicas;
    ~xyzb_dataset();
};

namespace {

void set_err(char* err, size_t errlen, const std::string& msg) {
    if (err && errlen) std::snprintf(err, errlen, "%s", msg.c_str());
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        return XYZB_OK;
    } catch (const data_error& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_DATA;
    } catch (const std::invalid_argument& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_DATA;
    } catch (const cuda_error& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_CUDA;
    } catch (const guard_error& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_GUARD;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_INTERNAL;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d) {
        XYZB_CUDA(cudaGetDevice(&prev));
        XYZB_CUDA(cudaSetDevice(d));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

void require_device() {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw cuda_error(std::string("libxyzb: no CUDA device available (") + cudaGetErrorString(e) +
                         "); the engine has no CPU fallback");
}

u32 grid_for(u64 n, u32 block, u32 cap = kSMs * 16) {
    return static_cast<u32>(std::max<u64>(1, std::min<u64>(ceil_div(n, block), cap)));
}

// SearchConfig::validate (search.cpp:119-134)
void validate_params(const xyzb_params* q) {
    if (q->m < 1 || q->m > 64) throw data_error("SearchConfig: M = " + std::to_string(q->m) + " outside [1,64]");
    if (q->l < 1) throw data_error("SearchConfig: L must be >= 1");
    if (!(q->gamma > 0.0 && q->gamma <= 1.0)) throw data_error("SearchConfig: gamma must lie in (0,1]");
    const bool wants = q->mode == XYZB_MODE_CONTINUOUS_XY;
    if (wants && q->transform == XYZB_TRANSFORM_NONE)
        throw data_error("SearchConfig: continuous-XY mode requires a binarize transform");
    if (!wants && q->transform != XYZB_TRANSFORM_NONE)
        throw data_error("SearchConfig: binarize transform is only valid in continuous-XY mode");
    if (q->mode < 0 || q->mode > 2) throw data_error("SearchConfig: unknown mode");
}

// ------------------------------------------------------------ dataset creation --

// XYZB_TRACE=1: host-side phase times of dataset creation on stderr (device
// drained at each mark, so only for diagnosis).
struct Trace {
    bool on = topt().trace.load() != 0;
    cudaStream_t st;
    bool sync;  // false: host-side times only (the stream keeps running)
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    explicit Trace(cudaStream_t s, bool sync_ = true) : st(s), sync(sync_) {}
    void mark(const char* what) {
        if (!on) return;
        if (sync) cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[xyzb] %-14s %8.1f us\n", what,
                     std::chrono::duration<double, std::micro>(now - t).count());
        t = now;
    }
};

// Persistent host worker pool for parallel staging copies (the single-thread
// memcpy into pinned memory, not PCIe, bounds the upload otherwise).
class CopyPool {
public:
    CopyPool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned n = std::min(8u, hw);
        for (unsigned t = 0; t < n; ++t) workers_.emplace_back([this] { loop(); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& w : workers_) w.join();
    }
    // memcpy(dst, src, len) split over the workers and the calling thread
    // (one copy at a time: concurrent callers queue on call_mu_)
    void copy(void* dst, const void* src, size_t len) {
        std::lock_guard<std::mutex> call(call_mu_);
        const size_t parts = workers_.size() + 1;
        const size_t slice = (len + parts - 1) / parts;
        std::unique_lock<std::mutex> lk(mu_);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        len_ = len;
        slice_ = slice;
        next_ = 1;
        pending_ = workers_.size();
        ++gen_;
        lk.unlock();
        cv_.notify_all();
        std::memcpy(dst, src, std::min(slice, len));
        lk.lock();
        done_cv_.wait(lk, [this] { return pending_ == 0; });
    }
    static CopyPool& get() {
        static CopyPool* p = new CopyPool();  // leaked on purpose (outlives static destructors)
        return *p;
    }

private:
    void loop() {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> lk(mu_);
        while (true) {
            cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            const size_t part = next_++;
            char* d = dst_;
            const char* s = src_;
            const size_t len = len_, slice = slice_;
            lk.unlock();
            const size_t b0 = std::min(len, part * slice), b1 = std::min(len, b0 + slice);
            if (b1 > b0) std::memcpy(d + b0, s + b0, b1 - b0);
            lk.lock();
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    bool stop_ = false;
    uint64_t gen_ = 0;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t len_ = 0, slice_ = 0, next_ = 0, pending_ = 0;
};

// Host -> device through two pooled pinned staging buffers: the (parallel)
// host copy of chunk i+1 overlaps the DMA of chunk i (pageable copies and 2-D
// copies with 504-byte rows are several times slower).
// Page-locked caller memory (cudaHostAlloc / cudaHostRegister / torch
// pin_memory) is copied by DMA directly.
bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Small transfers between page-locked host memory and the device as a kernel
// (zero-copy through UVA: the SMs read or write the pinned host buffer over
// PCIe). They do not queue on the copy engines behind other jobs' large X
// uploads: with several (X, y) jobs in flight a search's few-KB response,
// plan and status copies otherwise wait out another job's 400 MB - 1.3 GB
// upload (e2e traces: 1.4 ms searches taking 4-25 ms).
__global__ void zc_copy_kernel(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, size_t n) {
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x, nt = size_t(gridDim.x) * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const size_t n16 = n / 16;
        for (size_t i = tid; i < n16; i += nt)
            reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
        for (size_t i = n16 * 16 + tid; i < n; i += nt) dst[i] = src[i];
    } else {
        for (size_t i = tid; i < n; i += nt) dst[i] = src[i];
    }
}

// dst / src: one side device memory, the other page-locked host memory.
void small_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    if (bytes > (size_t(4) << 20)) {
        XYZB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
        return;
    }
    const u32 grid = static_cast<u32>(std::min<u64>(64, ceil_div(bytes, 256 * 16)));
    zc_copy_kernel<<<grid, 256, 0, st>>>(static_cast<const unsigned char*>(src), static_cast<unsigned char*>(dst),
                                         bytes);
    XYZB_LAUNCH_CHECK();
}

void upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    constexpr size_t kChunk = size_t(16) << 20;
    if (bytes <= (size_t(1) << 20) || is_pinned(src)) {
        XYZB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        return;
    }
    HostBuf stage[2];
    cudaEvent_t done[2];
    for (int i = 0; i < 2; ++i) {
        stage[i].ensure(kChunk);
        XYZB_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    bool used[2] = {false, false};
    for (size_t off = 0, i = 0; off < bytes; off += kChunk, i ^= 1) {
        const size_t len = std::min(kChunk, bytes - off);
        if (used[i]) XYZB_CUDA(cudaEventSynchronize(done[i]));
        CopyPool::get().copy(stage[i].p, static_cast<const char*>(src) + off, len);
        XYZB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage[i].p, len, cudaMemcpyHostToDevice, st));
        XYZB_CUDA(cudaEventRecord(done[i], st));
        used[i] = true;
    }
    XYZB_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < 2; ++i) cudaEventDestroy(done[i]);
}

// First column whose last word has a bit set above row n - 1 (PackedMatrix
// invariant, packed_matrix.hpp:10-14); *bad stays ~0 when every column is clean.
__global__ void check_padding(const u64* __restrict__ src, u64 W, u64 p, u32 tail, unsigned long long* bad) {
    for (u64 j = u64(blockIdx.x) * blockDim.x + threadIdx.x; j < p; j += u64(gridDim.x) * blockDim.x)
        if (src[j * W + W - 1] >> tail) atomicMin(bad, static_cast<unsigned long long>(j));
}

__global__ void pad_words(const u64* __restrict__ src, u64 W, u64 p, u64 Wp, u64* __restrict__ dst) {
    const u64 total = p * Wp;
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += u64(gridDim.x) * blockDim.x) {
        const u64 j = t / Wp, w = t - j * Wp;
        dst[t] = w < W ? src[j * W + w] : 0ull;
    }
}

// Raw column-major X lands in a device buffer through `fill(dev, bytes)`:
// an upload from caller memory (xyzb_dataset_create) or a stream from an
// XYZ1 file (xyzb_dataset_open).
using Fill = std::function<void(void*, size_t)>;

// check_pad: verify the padding bits on the device (caller memory) and throw
// data_error naming the first bad column, as the host check did.
void create_binary(xyzb_dataset* ds, const Fill& fill, bool check_pad = false) {
    Trace tr(ds->stream);
    ds->binary = true;
    ds->W = ceil_div(ds->n, 64);
    ds->Wp = round_up(ds->W, 4);
    ds->P32 = ceil_div(ds->p, 32);
    ds->Xc.ensure(ds->p * ds->Wp * 8);
    {
        DevBuf raw;
        raw.ensure(ds->p * ds->W * 8);
        tr.mark("alloc");
        fill(raw.p, ds->p * ds->W * 8);
        tr.mark("fill");
        const u32 tail = static_cast<u32>(ds->n & 63);
        if (check_pad && tail) {
            DevBuf bad;
            bad.ensure(8);
            XYZB_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, ds->stream));
            check_padding<<<grid_for(ds->p, 256, 1024), 256, 0, ds->stream>>>(raw.as<u64>(), ds->W, ds->p, tail,
                                                                                 bad.as<unsigned long long>());
            XYZB_LAUNCH_CHECK();
            u64 first = 0;
            XYZB_CUDA(cudaMemcpyAsync(&first, bad.p, 8, cudaMemcpyDeviceToHost, ds->stream));
            XYZB_CUDA(cudaStreamSynchronize(ds->stream));
            if (first != ~0ull)
                throw data_error("xyzb_dataset_create: padding bits of column " + std::to_string(first) +
                                 " are not zero");
            tr.mark("check_pad");
        }
        pad_words<<<grid_for(ds->p * ds->Wp, 256, 4096), 256, 0, ds->stream>>>(raw.as<u64>(), ds->W, ds->p, ds->Wp,
                                                                                ds->Xc.as<u64>());
        XYZB_LAUNCH_CHECK();
        tr.mark("pad");
        XYZB_CUDA(cudaStreamSynchronize(ds->stream));  // raw returns to the pool
    }
    tr.mark("raw_release");
    ds->Xr.ensure(ds->n * ds->P32 * 4);
    dim3 tg(static_cast<u32>(ceil_div(ds->P32, 32)), static_cast<u32>(ceil_div(ds->W, kern::kTrWords)));
    kern::transpose_bits<<<tg, 1024, 0, ds->stream>>>(ds->Xc.as<u64>(), ds->Wp, ds->W, ds->n, ds->p, ds->P32,
                                                      ds->Xr.as<u32>());
    XYZB_LAUNCH_CHECK();
    tr.mark("transpose");
}

// Real X: fp32 columns for the verify, column sign bits for the sign
// transform's bit-plane verify, row planes of (x > 0) / (x == 0) for the
// projection (bit transposes of the column bits), and the [-1, 1] / zero
// flags. f32: the caller's values are floats (x_real32; half the upload).
void create_real(xyzb_dataset* ds, const Fill& fill, bool f32) {
    ds->binary = false;
    ds->f32_src = f32;
    ds->n4 = round_up(ds->n, 4);
    ds->P32 = ceil_div(ds->p, 32);
    ds->W = ceil_div(ds->n, 64);
    ds->Wp = round_up(ds->W, 4);
    const u64 n = ds->n, p = ds->p;
    ds->Xc32.ensure(p * ds->n4 * 4);
    ds->Spos.ensure(p * ds->W * 8);
    ds->Snz.ensure(p * ds->W * 8);
    DevBuf tpos, tzero, flags;
    tpos.ensure(p * ds->Wp * 8);
    tzero.ensure(p * ds->Wp * 8);
    flags.ensure(4);
    XYZB_CUDA(cudaMemsetAsync(flags.p, 0, 4, ds->stream));
    const u32 sgrid = static_cast<u32>(std::min<u64>(ceil_div(p * 32, 256), u64(kSMs) * 16));
    if (f32) {
        if (n == ds->n4) {
            fill(ds->Xc32.p, n * p * 4);
        } else {
            DevBuf raw;
            raw.ensure(n * p * 4);
            fill(raw.p, n * p * 4);
            real::pad_f32_cols<<<grid_for(p * ds->n4, 256, 4096), 256, 0, ds->stream>>>(raw.as<float>(), n, p, ds->n4,
                                                                                         ds->Xc32.as<float>());
            XYZB_LAUNCH_CHECK();
            XYZB_CUDA(cudaStreamSynchronize(ds->stream));  // raw returns to the pool
        }
        real::sign_cols<float><<<sgrid, 256, 0, ds->stream>>>(ds->Xc32.as<float>(), ds->n4, n, p, ds->W, ds->Wp,
                                                              ds->Spos.as<u64>(), ds->Snz.as<u64>(), tpos.as<u64>(),
                                                              tzero.as<u64>(), flags.as<u32>());
    } else {
        ds->Xsrc64.ensure(n * p * 8);
        fill(ds->Xsrc64.p, n * p * 8);
        real::to_f32_cols<<<grid_for(p * ds->n4, 256, 4096), 256, 0, ds->stream>>>(ds->Xsrc64.as<double>(), n, p,
                                                                                     ds->n4, ds->Xc32.as<float>());
        XYZB_LAUNCH_CHECK();
        real::sign_cols<double><<<sgrid, 256, 0, ds->stream>>>(ds->Xsrc64.as<double>(), n, n, p, ds->W, ds->Wp,
                                                               ds->Spos.as<u64>(), ds->Snz.as<u64>(), tpos.as<u64>(),
                                                               tzero.as<u64>(), flags.as<u32>());
    }
    XYZB_LAUNCH_CHECK();
    ds->Xpos.ensure(n * ds->P32 * 4);
    ds->Xzero.ensure(n * ds->P32 * 4);
    dim3 tg(static_cast<u32>(ceil_div(ds->P32, 32)), static_cast<u32>(ceil_div(ds->W, kern::kTrWords)));
    kern::transpose_bits<<<tg, 1024, 0, ds->stream>>>(tpos.as<u64>(), ds->Wp, ds->W, n, p, ds->P32, ds->Xpos.as<u32>());
    XYZB_LAUNCH_CHECK();
    kern::transpose_bits<<<tg, 1024, 0, ds->stream>>>(tzero.as<u64>(), ds->Wp, ds->W, n, p, ds->P32,
                                                      ds->Xzero.as<u32>());
    XYZB_LAUNCH_CHECK();
    u32 hf = 0;
    XYZB_CUDA(cudaMemcpyAsync(&hf, flags.p, 4, cudaMemcpyDeviceToHost, ds->stream));
    XYZB_CUDA(cudaStreamSynchronize(ds->stream));
    ds->has_zero = (hf & 1u) != 0;
    ds->in_unit = (hf & 2u) == 0;
}

// The unbiased transform's fp64 rows [n][p], built on the first unbiased
// search from the caller's fp64 values (or the exact fp32 ones).
void ensure_xr64(xyzb_dataset* ds) {
    if (ds->Xr64.p) return;
    ds->Xr64.ensure(ds->n * ds->p * 8);
    dim3 tg(static_cast<u32>(ceil_div(ds->p, 32)), static_cast<u32>(ceil_div(ds->n, 32)));
    if (ds->f32_src)
        real::transpose_f64<float><<<tg, dim3(32, 8), 0, ds->stream>>>(ds->Xc32.as<float>(), ds->n4, ds->n, ds->p,
                                                                       ds->Xr64.as<double>());
    else
        real::transpose_f64<double><<<tg, dim3(32, 8), 0, ds->stream>>>(ds->Xsrc64.as<double>(), ds->n, ds->n, ds->p,
                                                                        ds->Xr64.as<double>());
    XYZB_LAUNCH_CHECK();
}

// A copy of a dataset's device-resident X on another device (or the same
// one): peer copies of the column / row layouts, over NVLink between GPUs.
std::unique_ptr<xyzb_dataset> replicate(xyzb_dataset* src, int dev) {
    std::unique_ptr<xyzb_dataset> r(new xyzb_dataset());
    r->device = dev;
    r->n = src->n;
    r->p = src->p;
    r->binary = src->binary;
    r->W = src->W;
    r->Wp = src->Wp;
    r->P32 = src->P32;
    r->n4 = src->n4;
    r->has_zero = src->has_zero;
    r->in_unit = src->in_unit;
    r->f32_src = src->f32_src;
    r->hit_cap = src->hit_cap;
    DeviceGuard dg(dev);
    XYZB_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    StreamScope ss(r->stream);
    DevBuf xyzb_dataset::*bufs[] = {&xyzb_dataset::Xc,  &xyzb_dataset::Xr,   &xyzb_dataset::Xc32,
                                    &xyzb_dataset::Xsrc64, &xyzb_dataset::Xpos, &xyzb_dataset::Xzero,
                                    &xyzb_dataset::Spos, &xyzb_dataset::Snz};
    for (auto m : bufs) {
        const DevBuf& s = src->*m;
        if (!s.p) continue;
        DevBuf& d = r.get()->*m;
        d.ensure(s.bytes);
        XYZB_CUDA(cudaMemcpyPeerAsync(d.p, dev, s.p, src->device, s.bytes, r->stream));
    }
    XYZB_CUDA(cudaStreamSynchronize(r->stream));
    return r;
}

// Stream an XYZ1 payload (dataset_io.cpp:91-129) from `f` to the device
// through pinned staging, validating column padding (binary) on the way.
void stream_file(void* dst, std::FILE* f, size_t bytes, bool binary, u64 W, u64 n, const std::string& path,
                 cudaStream_t st) {
    constexpr size_t kChunk = size_t(16) << 20;  // a multiple of 8 bytes
    HostBuf stage[2];
    cudaEvent_t done[2];
    for (int i = 0; i < 2; ++i) {
        stage[i].ensure(kChunk);
        XYZB_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    const u64 tail = n & 63;
    const u64 mask = tail == 0 ? ~0ull : ((1ull << tail) - 1);
    bool used[2] = {false, false};
    std::string fail;
    for (size_t off = 0, i = 0; off < bytes && fail.empty(); off += kChunk, i ^= 1) {
        const size_t len = std::min(kChunk, bytes - off);
        if (used[i]) XYZB_CUDA(cudaEventSynchronize(done[i]));
        if (std::fread(stage[i].p, 1, len, f) != len) {
            fail = "read_dataset: truncated payload in " + path;
            break;
        }
        if (binary && mask != ~0ull) {
            const u64* w = stage[i].as<u64>();
            const u64 w0 = off / 8;
            for (u64 t = (W - 1 + W - w0 % W) % W; t < len / 8; t += W)  // last word of each column
                if (w[t] & ~mask) {
                    fail = "read_dataset: nonzero padding bits in " + path;
                    break;
                }
        }
        if (!fail.empty()) break;
        XYZB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage[i].p, len, cudaMemcpyHostToDevice, st));
        XYZB_CUDA(cudaEventRecord(done[i], st));
        used[i] = true;
    }
    XYZB_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < 2; ++i) cudaEventDestroy(done[i]);
    if (!fail.empty()) throw data_error(fail);
    if (std::fgetc(f) != EOF) throw data_error("read_dataset: trailing bytes in " + path);
}

// ------------------------------------------------------------ the search --

struct RunPlan {
    u64 L = 0;
    int npass = 1;
    std::vector<u32> rid;             // global run ids in execution order
    std::vector<int8_t> sign;         // per run
    std::vector<u64> stream;          // per run: make_stream stream id = offset + rep
    std::vector<u32> rows;            // [R][M], only for caller-supplied draws
    std::vector<int8_t> sign_by_rid;  // [npass * L]
};

struct SearchCtx {
    xyzb_dataset* ds;
    const xyzb_params* q;
    int mode;
    u64 n, p, M, guard;
    double gamma;
    u32 astar = 0;        // binary integer threshold
    double norm = 0.0;    // ||y||_1 (continuous)
    bool weighted = false;
    u64 item_cap = 0, nbatches = 0, pair_cap = 0;
    u64 item_scale = 1;  // grows when a batch overflows its item buffer
    u64 pair_scale = 1;  // grows when a batch overflows its pair list
    // the sign transform's quantised response (bit planes, SignStrength)
    int qB = kern::kSignQB;
    double qinv = 0.0, qdelta = 0.0;
    // the weighted verify's quantised |y| (continuous-Y, WeightedQ)
    double wqinv = 0.0, wqdelta = 0.0;
    long long qsum = 0;
    bool sign_verify = false;  // the bit-plane verify ran
    bool no_hash = false;  // a hashed partition overflowed: the sparse grouping runs on the sorted path
    bool pairs_in_sort = false;  // the fused group + join kernel writes the pair list (its stage is SORT)
    // top-K over all verified candidates (XYZB_TOPK_CANDIDATES): running rank threshold per batch
    bool topk_all = false;
    int tk_level = 0;      // 0: emission target 4K + 256; 1: 64K + 4096; 2: emit everything >= thr
    int tk_shift = 0;      // rank bin shift
    u64 tk_table = 0;      // dedup table slots (power of two)
    // binned verify (X >> L2): pairs of all batches bucketed by (z window, x tile), verified at the end
    bool binned = false;
    bool tk_all_windows = false;  // binned top-K: a phase after every window (the redo when the first window's
                                  // phase left the threshold at 0)
    u64 attempts = 0;            // device passes over the search (redos after an outgrown capacity)
    bool no_fixed_part = false;  // a fixed-capacity partition overflowed: the redo counts the partitions first
    bool no_one_pass = false;  // a one-pass join overflowed the pair list: the redo counts first
    int wshift = 0, nkt = 0;
    u64 nbj = 0, nbh = 0, cap_kt = 0, cap_bucket = 0, ovf_cap = 0;
    RunPlan plan;
    xyzb_result* out;
    u64 launches[XYZB_NUM_STAGES] = {};
    u64 bytes[XYZB_NUM_STAGES] = {};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> verify_spans;
};

// smallest a with double(a)/double(n) >= gamma (A.7)
u32 integer_threshold(u64 n, double gamma) {
    u64 lo = 0, hi = n + 1;
    while (lo < hi) {
        const u64 mid = (lo + hi) / 2;
        if (double(mid) / double(n) >= gamma) hi = mid; else lo = mid + 1;
    }
    return static_cast<u32>(lo);
}

// Response-derived device vectors, staged through the dataset's pinned buffer
// (asynchronous; the search synchronises before the buffer is reused).
void upload_response(SearchCtx& c, const xyzb_response* resp) {
    xyzb_dataset* ds = c.ds;
    cudaStream_t st = ds->stream;
    const u64 n = c.n, Wp = ds->Wp, nb = Wp * 64;
    if (c.mode == XYZB_MODE_BINARY) {
        ds->h_small.ensure(Wp * 8);
        u64* bits = ds->h_small.as<u64>();
        std::memset(bits, 0, Wp * 8);
        for (u64 i = 0; i < n; ++i) {
            const int8_t v = resp->y_sign[i];
            if (v != 1 && v != -1) throw data_error("xyz_search: binary response must be +-1");
            if (v > 0) bits[i >> 6] |= 1ull << (i & 63);
        }
        ds->yk_bits.ensure(Wp * 8);
        small_copy(ds->yk_bits.p, bits, Wp * 8, st);
        return;
    }
    const double* y = resp->y_real;
    double norm = 0.0;
    for (u64 i = 0; i < n; ++i) norm += std::abs(y[i]);
    if (norm <= 0.0) throw data_error("xyz_search: zero response vector");
    c.norm = norm;
    // WeightedSampler::from_magnitudes cumulative table (real_matrix.cpp:36-47), host fp64 in order
    host::WeightedSampler ws(y, n);
    c.weighted = true;
    const u64 n4 = ds->n4 ? ds->n4 : round_up(n, 4);
    const size_t need = n * 8 /*cum*/ + (c.mode == XYZB_MODE_CONTINUOUS_Y ? 3 * Wp * 8 + nb * 8 : n4 * 8);
    ds->h_small.ensure(need);
    char* hp = ds->h_small.as<char>();
    double* cum = reinterpret_cast<double*>(hp);
    ws.copy_cumulative(cum);
    ds->cum.ensure(n * 8);
    small_copy(ds->cum.p, cum, n * 8, st);
    hp += n * 8;
    if (c.mode == XYZB_MODE_CONTINUOUS_Y) {
        u64* bits = reinterpret_cast<u64*>(hp);
        u64* sp = bits + Wp;
        u64* sn = sp + Wp;
        double* w = reinterpret_cast<double*>(sn + Wp);
        std::memset(hp, 0, 3 * Wp * 8 + nb * 8);
        for (u64 i = 0; i < n; ++i) {
            if (y[i] >= 0.0) bits[i >> 6] |= 1ull << (i & 63);  // y_sign for the keys (search.cpp:377-378)
            if (y[i] > 0.0) sp[i >> 6] |= 1ull << (i & 63);
            if (y[i] < 0.0) sn[i >> 6] |= 1ull << (i & 63);
            w[i] = std::abs(y[i]);
        }
        ds->yk_bits.ensure(Wp * 8);
        ds->spos.ensure(Wp * 8);
        ds->sneg.ensure(Wp * 8);
        ds->wabs.ensure(nb * 8);
        small_copy(ds->yk_bits.p, bits, Wp * 8, st);
        small_copy(ds->spos.p, sp, Wp * 8, st);
        small_copy(ds->sneg.p, sn, Wp * 8, st);
        small_copy(ds->wabs.p, w, nb * 8, st);
        // |y| quantised to kWeightQB-bit unsigned planes (WeightedQ): q_i = rint(|y_i| scale)
        double ymax = 0.0;
        for (u64 i = 0; i < n; ++i) ymax = std::max(ymax, std::abs(y[i]));
        constexpr int QB = kern::kWeightQB;
        const double scale = (std::ldexp(1.0, QB) - 1.0) / ymax;
        const u64 W = ds->W;
        ds->h_planes.ensure(u64(QB) * W * 8);
        u64* pl = ds->h_planes.as<u64>();
        std::memset(pl, 0, u64(QB) * W * 8);
        for (u64 i = 0; i < n; ++i) {
            const u64 q = static_cast<u64>(std::llrint(std::abs(y[i]) * scale));
            for (int b = 0; b < QB; ++b)
                if ((q >> b) & 1ull) pl[u64(b) * W + (i >> 6)] |= 1ull << (i & 63);
        }
        c.wqinv = 1.0 / scale;
        // |quantised - exact| <= n / (2 scale) over ||y||_1; + slack for the fp64 sums
        c.wqdelta = double(n) / (2.0 * scale * norm) + 1e-9;
        ds->yplanes.ensure(u64(QB) * W * 8);
        small_copy(ds->yplanes.p, pl, u64(QB) * W * 8, st);
        return;
    }
    double* yp = reinterpret_cast<double*>(hp);
    std::memset(yp, 0, n4 * 8);
    std::copy(y, y + n, yp);
    ds->yreal.ensure(n4 * 8);
    small_copy(ds->yreal.p, yp, n4 * 8, st);
    if (c.q->transform == XYZB_TRANSFORM_SIGN) {
        // q_i = rint(y_i * scale) as two's-complement bit planes 0..B over the row words (SignStrength)
        double ymax = 0.0;
        for (u64 i = 0; i < n; ++i) ymax = std::max(ymax, std::abs(y[i]));
        const int B = c.qB;
        const double scale = (std::ldexp(1.0, B) - 1.0) / ymax;  // |q| <= 2^B - 1: B + 1 two's-complement bits
        const u64 W = ds->W;
        ds->h_planes.ensure(u64(B + 1) * W * 8);
        u64* pl = ds->h_planes.as<u64>();
        std::memset(pl, 0, u64(B + 1) * W * 8);
        long long qs = 0;
        for (u64 i = 0; i < n; ++i) {
            const long long q = std::llrint(y[i] * scale);
            qs += q;
            const unsigned long long u = static_cast<unsigned long long>(q);
            for (int b = 0; b <= B; ++b)
                if ((u >> b) & 1ull) pl[u64(b) * W + (i >> 6)] |= 1ull << (i & 63);
        }
        c.qinv = 1.0 / scale;
        c.qsum = qs;
        // |quantised - exact| <= 1.5 n / (2 scale norm); + 1e-6 for the fp32 columns of RealStrength
        c.qdelta = 1.5 * double(n) / (2.0 * scale * norm) + 1e-6;
        ds->yplanes.ensure(u64(B + 1) * W * 8);
        small_copy(ds->yplanes.p, pl, u64(B + 1) * W * 8, st);
    }
}

// Runs of the search in execution order (pass +1 then -1, reps ascending;
// PassPlan stream offsets 0 and L, search.cpp:353-358).
void plan_runs(SearchCtx& c, const uint32_t* draws) {
    const xyzb_params* q = c.q;
    RunPlan& pl = c.plan;
    pl.L = q->l;
    pl.npass = q->search_negatives ? 2 : 1;
    u64 rb = 1, re = q->l + 1;
    if (q->rep_begin || q->rep_end) {
        rb = q->rep_begin;
        re = q->rep_end;
        if (rb < 1 || re > q->l + 1 || rb > re) throw data_error("xyzb: rep shard outside [1, L]");
    }
    pl.sign_by_rid.resize(pl.npass * pl.L);
    for (int ps = 0; ps < pl.npass; ++ps)
        for (u64 r = 0; r < pl.L; ++r) pl.sign_by_rid[ps * pl.L + r] = ps == 0 ? 1 : -1;
    if (draws && c.mode == XYZB_MODE_CONTINUOUS_XY)
        throw data_error("xyzb: caller-supplied draws are not supported for continuous-XY transforms");
    for (int ps = 0; ps < pl.npass; ++ps) {
        const u64 offset = ps == 0 ? 0 : q->l;
        for (u64 rep = rb; rep < re; ++rep) {
            pl.rid.push_back(static_cast<u32>(ps * pl.L + rep - 1));
            pl.sign.push_back(ps == 0 ? 1 : -1);
            pl.stream.push_back(offset + rep);
            if (draws) {
                const size_t at = pl.rows.size();
                pl.rows.resize(at + c.M);
                std::memcpy(pl.rows.data() + at, draws + ((ps * pl.L) + rep - 1) * c.M, c.M * 4);
                for (u64 s = 0; s < c.M; ++s)
                    if (pl.rows[at + s] >= c.n) throw data_error("project_keys: draw index out of range");
            }
        }
    }
}

// The sign transform's verify functor (bit planes + the exact fp32 fallback);
// converts the response to fp32 on the dataset stream first.
kern::SignStrength sign_strength(SearchCtx& c) {
    xyzb_dataset* ds = c.ds;
    ds->yreal32.ensure(ds->n4 * 4);
    real::to_f32<<<grid_for(ds->n4, 256, 256), 256, 0, ds->stream>>>(ds->yreal.as<double>(), ds->n4,
                                                                     ds->yreal32.as<float>());
    XYZB_LAUNCH_CHECK();
    kern::RealStrength<false> f{ds->Xc32.as<float>(), ds->n4, ds->yreal32.as<float>(), c.norm, c.gamma};
    return kern::SignStrength{ds->Spos.as<u64>(), ds->Snz.as<u64>(), ds->W, ds->yplanes.as<u64>(), c.qsum,
                              ds->has_zero, c.qinv, c.norm, c.gamma, c.qdelta, f};
}

// Top-K over all candidates, after a batch's verify (topk_kernels.cuh): the
// pair-list path picks an emission threshold from the batch's rank histogram
// and appends the pairs at or above it; then the hit buffer is pruned to the
// occurrences at or above the K-th distinct key's rank bin.
void topk_prune(SearchCtx& c, const kern::VerifyArgs& A, u64* launches);

void topk_after_batch(SearchCtx& c, bool pair_path, const kern::VerifyArgs& A, const u32* np, u64* launches,
                      const kern::SignStrength* sg = nullptr, const kern::WeightedQ* wq = nullptr) {
    Nvtx nv("xyzb:topk");
    xyzb_dataset* ds = c.ds;
    cudaStream_t st = ds->stream;
    auto* S = ds->tk_state.as<topk::State>();
    if (pair_path) {
        const u64 K = c.q->top_k;
        const u32 target = c.tk_level == 0 ? u32(std::min<u64>(4 * K + 256, 0x7fffffffull))
                                           : u32(std::min<u64>(64 * K + 4096, 0x7fffffffull));
        topk::rank_hist<<<kSMs * 2, 512, 0, st>>>(ds->tk_sint.as<u32>(), np, static_cast<u32>(c.pair_cap), A.nitems,
                                                  A.item_cap, S, c.tk_shift, ds->tk_hist.as<u32>());
        XYZB_LAUNCH_CHECK();
        topk::emit_select<<<1, 1024, 0, st>>>(ds->tk_hist.as<u32>(), c.tk_shift, target, S, c.tk_level >= 2);
        XYZB_LAUNCH_CHECK();
        if (sg)  // sign transform: exact re-verification of the pairs that may reach E
            topk::emit_pairs_requant<<<kSMs * 8, 256, 0, st>>>(A, ds->pairs.as<kern::PairRec>(), np,
                                                               static_cast<u32>(c.pair_cap), *sg, S);
        else if (wq)  // weighted: likewise
            topk::emit_pairs_requant<<<kSMs * 8, 256, 0, st>>>(A, ds->pairs.as<kern::PairRec>(), np,
                                                               static_cast<u32>(c.pair_cap), *wq, S);
        else
            topk::emit_pairs<<<kSMs * 8, 256, 0, st>>>(ds->pairs.as<kern::PairRec>(), ds->tk_sint.as<u32>(), np,
                                                       static_cast<u32>(c.pair_cap), A.nitems, A.item_cap, S,
                                                       A.xkeys, A.key64, A.S, A.rid, A.hits, A.hit_count, A.hit_cap,
                                                       static_cast<u32>(c.n));
        XYZB_LAUNCH_CHECK();
        *launches += 3;
    } else {
        topk::emit_all<<<1, 1, 0, st>>>(S);
        XYZB_LAUNCH_CHECK();
        *launches += 1;
    }
    topk_prune(c, A, launches);
}

// prune: distinct keys by rank bin, raise the threshold, keep the occurrences at or above it
void topk_prune(SearchCtx& c, const kern::VerifyArgs& A, u64* launches) {
    xyzb_dataset* ds = c.ds;
    cudaStream_t st = ds->stream;
    auto* S = ds->tk_state.as<topk::State>();
    const int binary = c.mode == XYZB_MODE_BINARY ? 1 : 0;
    XYZB_CUDA(cudaMemsetAsync(ds->tk_table.p, 0xff, c.tk_table * 8, st));
    XYZB_CUDA(cudaMemsetAsync(ds->tk_cnt2.p, 0, 4, st));
    topk::prune_insert<<<grid_for(ds->hit_cap, 256, kSMs * 4), 256, 0, st>>>(
        A.hits, A.hit_count, A.hit_cap, ds->sign_by_rid.as<int8_t>(), ds->tk_table.as<u64>(), c.tk_table - 1,
        c.tk_shift, static_cast<u32>(c.n), binary, ds->tk_dhist.as<u32>(), S);
    XYZB_LAUNCH_CHECK();
    topk::prune_select<<<1, 1024, 0, st>>>(ds->tk_dhist.as<u32>(), c.tk_shift, static_cast<u32>(c.q->top_k), S);
    XYZB_LAUNCH_CHECK();
    topk::prune_compact<<<grid_for(ds->hit_cap, 256, kSMs * 4), 256, 0, st>>>(
        A.hits, A.hit_count, A.hit_cap, static_cast<u32>(c.n), binary, S, ds->hits2.as<kern::DevHit>(),
        ds->tk_cnt2.as<u32>());
    XYZB_LAUNCH_CHECK();
    topk::copy_back<<<grid_for(ds->hit_cap, 256, kSMs * 4), 256, 0, st>>>(ds->hits2.as<kern::DevHit>(),
                                                                          ds->tk_cnt2.as<u32>(), A.hits, A.hit_count);
    XYZB_LAUNCH_CHECK();
    *launches += 4;
}

// Binned verify (binned_verify.cuh), after every batch's pairs sit in their
// z-side windows: bins by x-side tile (counting sort), then one persistent
// verify per window; top-K over all candidates treats each window like a
// batch (the first window writes ranks, emits at E, prunes; later windows
// append at or above the running threshold).
void binned_verify(SearchCtx& c) {
    xyzb_dataset* ds = c.ds;
    cudaStream_t st = ds->stream;
    StageClock& clk = ds->clock;
    const u32 nbj = static_cast<u32>(c.nbj);
    const int nkt = c.nkt;
    cudaEvent_t e0 = clk.mark();
    const u32 nbuckets = static_cast<u32>(u64(nkt) * c.nbh);
    const u32 cpk = static_cast<u32>(ceil_div(kSMs * 4, nkt));  // CTAs per window
    func_smem(bins::bin_split, bins::step_stage_smem());
    bins::bin_split<<<cpk * nkt, bins::kPartThreads, bins::step_stage_smem(), st>>>(
        ds->bin_s.as<u64>(), static_cast<u32>(c.cap_kt), ds->bin_wcnt.as<u32>(), cpk, static_cast<u32>(c.nbh),
        ds->bin_b.as<u64>(), static_cast<u32>(c.cap_bucket), ds->bin_cnt.as<u32>(), ds->bin_ovf.as<u64>(),
        static_cast<u32>(c.ovf_cap), ds->bin_ovfn.as<u32>());
    XYZB_LAUNCH_CHECK();
    XYZB_CUDA(cudaMemsetAsync(ds->bin_fill.p, 0, u64(nkt) * nbj * 4, st));
    func_smem(bins::bin_sort, bins::step_stage_smem());
    bins::bin_sort<<<nbuckets, bins::kPartThreads, bins::step_stage_smem(), st>>>(ds->bin_b.as<u64>(), static_cast<u32>(c.cap_bucket), ds->bin_cnt.as<u32>(),
                                              static_cast<u32>(c.nbh), nbj, ds->bin_d.as<u64>(), ds->bin_start.as<u32>(),
                                              ds->bin_fill.as<u32>(), ds->bin_ovf.as<u64>(),
                                              static_cast<u32>(c.ovf_cap), ds->bin_ovfn.as<u32>());
    XYZB_LAUNCH_CHECK();
    bins::tile_sort<<<static_cast<u32>(u64(nkt) * nbj), bins::kTileSortThreads, 0, st>>>(
        ds->bin_d.as<u64>(), static_cast<u32>(c.cap_bucket), static_cast<u32>(c.nbh), nbj, ds->bin_start.as<u32>(),
        ds->bin_fill.as<u32>());
    XYZB_LAUNCH_CHECK();
    bins::bin_scan<<<nkt, 1024, 0, st>>>(ds->bin_fill.as<u32>(), nbj, ds->bin_boff.as<u32>());
    XYZB_LAUNCH_CHECK();
    c.launches[XYZB_STAGE_JOIN] += 4;
    clk.span(XYZB_STAGE_JOIN, e0, clk.mark());
    bins::BinVerifyArgs A;
    A.Xc = ds->Xc.as<u64>();
    A.Wp = static_cast<u32>(ds->Wp);
    A.Yw = ds->yk_bits.as<u64>();
    A.n = static_cast<u32>(c.n);
    A.astar = c.astar;
    A.p = c.p;
    A.nbj = nbj;
    A.rid = ds->rid.as<u32>();
    A.hits = ds->hits.as<kern::DevHit>();
    A.hit_count = ds->hit_count.as<u32>();
    A.hit_cap = ds->hit_cap;
    A.krows = ds->rows.as<u32>();
    A.kM = static_cast<int>(c.M);
    A.sint_out = c.topk_all ? ds->tk_sint.as<u32>() : nullptr;
    A.rank_thr = c.topk_all ? &ds->tk_state.as<topk::State>()->thr : nullptr;
    A.rank_fail = c.topk_all ? &ds->tk_state.as<topk::State>()->fail : nullptr;
    A.phase_follows = 1;
    const int ns = static_cast<int>(ceil_div(ds->Wp / 2, 16));
    const size_t smem = bins::verify_smem(A.Wp);
    const bool full = ds->Wp / 2 == u64(16 * ns);  // every lane's slices inside the column
    auto* vk = ns <= 1 ? (full ? bins::verify_binned<1, true> : bins::verify_binned<1, false>)
             : ns == 2 ? (full ? bins::verify_binned<2, true> : bins::verify_binned<2, false>)
             : ns == 3 ? (full ? bins::verify_binned<3, true> : bins::verify_binned<3, false>)
             : ns == 4 ? (full ? bins::verify_binned<4, true> : bins::verify_binned<4, false>)
                       : (full ? bins::verify_binned<5, true> : bins::verify_binned<5, false>);
    func_smem(vk, smem);
    // the x tiles of this search: X ^ Y (the response XORed in once, so the tiles need no pass of their own)
    cudaEvent_t ex0 = clk.mark();
    ds->bin_xy.ensure(c.p * ds->Wp * 8);
    bins::xor_response<<<kSMs * 16, 256, 0, st>>>(ds->Xc.as<ulonglong2>(), ds->yk_bits.as<ulonglong2>(),
                                                  static_cast<u32>(ds->Wp / 2), c.p * (ds->Wp / 2),
                                                  ds->bin_xy.as<ulonglong2>());
    XYZB_LAUNCH_CHECK();
    c.launches[XYZB_STAGE_VERIFY] += 1;
    clk.span(XYZB_STAGE_VERIFY, ex0, clk.mark());
    // the prune reads the hit buffer through VerifyArgs
    kern::VerifyArgs PA{};
    PA.hits = A.hits;
    PA.hit_count = A.hit_count;
    PA.hit_cap = A.hit_cap;
    auto topk_phase = [&](cudaEvent_t ev1, const u32* cnt, u32 cap, const u64* list, const u32* boff) {
        Nvtx nv("xyzb:topk");
        auto* S = ds->tk_state.as<topk::State>();
        const u64 K = c.q->top_k;
        const u32 target = c.tk_level == 0 ? u32(std::min<u64>(4 * K + 256, 0x7fffffffull))
                                           : u32(std::min<u64>(64 * K + 4096, 0x7fffffffull));
        topk::rank_hist<<<kSMs * 2, 512, 0, st>>>(ds->tk_sint.as<u32>(), cnt, cap, ds->bin_zero.as<u32>(), 1u, S,
                                                  c.tk_shift, ds->tk_hist.as<u32>());
        XYZB_LAUNCH_CHECK();
        topk::emit_select<<<1, 1024, 0, st>>>(ds->tk_hist.as<u32>(), c.tk_shift, target, S, c.tk_level >= 2);
        XYZB_LAUNCH_CHECK();
        if (list)
            bins::emit_list<<<kSMs * 8, 256, 0, st>>>(list, ds->tk_sint.as<u32>(), cnt, cap, S, A.rid, A.krows, A.kM,
                                                      A.Xc, A.Wp, A.hits, A.hit_count, A.hit_cap, A.n);
        else
            bins::emit_bins<<<kSMs * 8, 256, 0, st>>>(A.F, A.bstart, boff, nbj, ds->tk_sint.as<u32>(), S, A.rid,
                                                      A.krows, A.kM, A.Xc, A.Wp, A.hits, A.hit_count, A.hit_cap,
                                                      A.n);
        XYZB_LAUNCH_CHECK();
        c.launches[XYZB_STAGE_MERGE] += 3;
        topk_prune(c, PA, &c.launches[XYZB_STAGE_MERGE]);
        clk.span(XYZB_STAGE_MERGE, ev1, clk.mark());
    };
    for (int kt = 0; kt < nkt; ++kt) {
        Nvtx nv_verify("xyzb:verify");
        A.F = ds->bin_d.as<u64>() + u64(kt) * c.nbh * c.cap_bucket;
        A.bstart = ds->bin_start.as<u32>() + u64(kt) * nbj;
        A.boff = ds->bin_boff.as<u32>() + u64(kt) * (nbj + 1);
        // top-K: the first window's phase sets the threshold, later windows append at or above it and the
        // last phase (after the overflow list) prunes; a later window that still finds the threshold at 0
        // flags the search, which is then redone with a phase after every window
        const bool phase = c.topk_all && (kt == 0 || c.tk_all_windows);
        A.phase_follows = phase ? 1u : 0u;
        cudaEvent_t ev0 = clk.mark();
        vk<<<kSMs, bins::kVerifyThreads, smem, st>>>(A, ds->bin_xy.as<u64>());
        XYZB_LAUNCH_CHECK();
        c.launches[XYZB_STAGE_VERIFY] += 1;
        cudaEvent_t ev1 = clk.mark();
        clk.span(XYZB_STAGE_VERIFY, ev0, ev1);
        c.verify_spans.push_back({ev0, ev1});
        if (phase) topk_phase(ev1, A.boff + nbj, 0xffffffffu, nullptr, A.boff);  // the window's pairs held in bins
    }
    // pairs whose bin was full
    A.phase_follows = 1;
    cudaEvent_t ev0 = clk.mark();
    bins::verify_list<<<kSMs * 8, 256, 0, st>>>(A, ds->bin_ovf.as<u64>(), ds->bin_ovfn.as<u32>(),
                                                static_cast<u32>(c.ovf_cap));
    XYZB_LAUNCH_CHECK();
    c.launches[XYZB_STAGE_VERIFY] += 1;
    cudaEvent_t ev1 = clk.mark();
    clk.span(XYZB_STAGE_VERIFY, ev0, ev1);
    if (c.topk_all)
        topk_phase(ev1, ds->bin_ovfn.as<u32>(), static_cast<u32>(c.ovf_cap), ds->bin_ovf.as<u64>(), nullptr);
}

template <class K>
void run_batches(SearchCtx& c) {
    xyzb_dataset* ds = c.ds;
    cudaStream_t st = ds->stream;
    const u64 p = c.p, M = c.M;
    const u64 R = c.plan.rid.size();
    const u64 Rall = c.plan.sign_by_rid.size();
    StageClock& clk = ds->clock;
    // per-search counters
    ds->enumerated.ensure(Rall * 8);
    ds->verified.ensure(Rall * 8);
    ds->sign_by_rid.ensure(Rall);
    XYZB_CUDA(cudaMemsetAsync(ds->enumerated.p, 0, Rall * 8, st));
    XYZB_CUDA(cudaMemsetAsync(ds->verified.p, 0, Rall * 8, st));
    ds->hit_count.ensure(8);
    XYZB_CUDA(cudaMemsetAsync(ds->hit_count.p, 0, 4, st));
    ds->povf.ensure(8);
    XYZB_CUDA(cudaMemsetAsync(ds->povf.p, 0, 8, st));  // [0] hashed partition overflow, [1] fixed partition overflow
    ds->hits.ensure(sizeof(kern::DevHit) * u64(ds->hit_cap));
    if (c.topk_all) {
        ds->hits2.ensure(sizeof(kern::DevHit) * u64(ds->hit_cap));
        c.tk_table = 64;
        while (c.tk_table < 2ull * ds->hit_cap) c.tk_table <<= 1;
        ds->tk_table.ensure(c.tk_table * 8);
        ds->tk_state.ensure(sizeof(topk::State));
        ds->tk_hist.ensure(topk::kBins * 4);
        ds->tk_dhist.ensure(topk::kBins * 4);
        ds->tk_cnt2.ensure(8);
        XYZB_CUDA(cudaMemsetAsync(ds->tk_state.p, 0, sizeof(topk::State), st));
        XYZB_CUDA(cudaMemsetAsync(ds->tk_hist.p, 0, topk::kBins * 4, st));
        XYZB_CUDA(cudaMemsetAsync(ds->tk_dhist.p, 0, topk::kBins * 4, st));
        const u64 max_rank = c.mode == XYZB_MODE_BINARY ? c.n : (u64(1) << kern::kRealRankBits);
        c.tk_shift = topk::bin_shift(max_rank);
    }
    // batch size: B*p entries under the budget (about 64 B of scratch each)
    u64 budget = u64(1) << 26;  // the batch_entries test option forces multi-batch runs
    if (const long long e = topt().batch_entries.load()) budget = std::max<u64>(1, u64(e));
    const u64 B = std::max<u64>(1, std::min<u64>({R, budget / std::max<u64>(p, 1), u64(bins::kMaxRunsPerBatch)}));
    const u64 cap = B * p;
    for (int i = 0; i < 2; ++i) {
        ds->keys[i].ensure(cap * sizeof(K));
        ds->vals[i].ensure(cap * 4);
    }
    ds->hist.ensure(rsort::hist_words(B, p) * 4);
    u64 item_cap = std::min<u64>(0xffffffffull, B * (p / 2 + 64) * c.item_scale);  // regrows on overflow
    if (const long long e = topt().item_cap.load())  // tests force the item-buffer regrow path
        item_cap = std::min<u64>(item_cap, std::max<u64>(1, u64(e)) * c.item_scale);
    if (item_cap > 0xffffffffull) throw internal_error("xyzb: batch too large for 32-bit item indices");
    ds->items.ensure(item_cap * sizeof(kern::Item));
    // host plan -> pinned -> device
    const bool host_rows = !c.plan.rows.empty();
    // per-batch counters live in their own pinned slots: a later batch must not
    // overwrite a value an earlier, still-queued copy has not read yet
    const size_t hbytes = R * 4 + R + R * 8 + (host_rows ? R * M * 4 : 0) + 2 * R * 4 + 96 + Rall;
    ds->h_rows.ensure(hbytes);
    char* hp = ds->h_rows.as<char>();
    std::memcpy(hp, c.plan.rid.data(), R * 4);
    std::memcpy(hp + R * 4, c.plan.sign.data(), R);
    std::memcpy(hp + R * 5, c.plan.stream.data(), R * 8);
    if (host_rows) std::memcpy(hp + R * 13, c.plan.rows.data(), R * M * 4);
    char* hsr = hp + hbytes - Rall;  // the signs by run id, staged in the pinned block too
    std::memcpy(hsr, c.plan.sign_by_rid.data(), Rall);
    small_copy(ds->sign_by_rid.p, hsr, Rall, st);
    ds->rid.ensure(R * 4);
    ds->rsign.ensure(R);
    ds->streams.ensure(R * 8);
    ds->rows.ensure(R * M * 4);
    small_copy(ds->rid.p, hp, R * 4, st);
    small_copy(ds->rsign.p, hp + R * 4, R, st);
    small_copy(ds->streams.p, hp + R * 5, R * 8, st);
    const bool xy = c.mode == XYZB_MODE_CONTINUOUS_XY;
    const bool unbiased = xy && c.q->transform == XYZB_TRANSFORM_UNBIASED;
    const bool coins = xy && !unbiased && ds->has_zero;
    if (unbiased || coins) ds->mt_state.ensure(R * 313 * 8);
    // ---- draws (device RNG, or the caller's rows) ----
    cudaEvent_t ed0 = clk.mark();
    if (host_rows) {
        small_copy(ds->rows.p, hp + R * 13, R * M * 4, st);
    } else {
        draws::draw_runs<<<static_cast<u32>(R), 32, 0, st>>>(
            static_cast<u32>(R), ds->streams.as<u64>(), c.q->seed, c.n, int(M), c.weighted ? ds->cum.as<double>() : nullptr,
            ds->rows.as<u32>(), (unbiased || coins) ? ds->mt_state.as<u64>() : nullptr);
        XYZB_LAUNCH_CHECK();
        c.launches[XYZB_STAGE_DRAWS] += 1;
    }
    clk.span(XYZB_STAGE_DRAWS, ed0, clk.mark());
    c.bytes[XYZB_STAGE_DRAWS] += R * M * 4;
    if (coins) {
        ds->zmask.ensure(cap * sizeof(K));
        ds->zcount.ensure(cap * 4);
        ds->zoff.ensure((cap + 1) * 4);
        ds->zcnt_n.ensure(8);
        ds->partial.ensure(scan::kGrid * 8);
    }
    ds->xorc.ensure(B * sizeof(K));
    ds->tot.ensure(B * 8);
    ds->work_run.ensure(B * 8);
    const u64 nbatches = ceil_div(R, B);
    ds->nblocks.ensure(nbatches * 4);  // items per batch (may exceed item_cap: regrow)
    XYZB_CUDA(cudaMemsetAsync(ds->nblocks.p, 0, nbatches * 4, st));
    c.item_cap = item_cap;
    c.nbatches = nbatches;
    // the sign transform's bit-plane verify over the pair list: columns of <= 2048 rows (lane w holds
    // word w of the sign bits and of the response planes)
    const bool sign_pairs = xy && !unbiased && ds->Spos.p && ds->W <= 32 && !topt().sign_verify_off.load();
    // the weighted (continuous-Y) verify over the pair list: rows <= 2048, |y| as bit planes
    const bool weighted_pairs = c.mode == XYZB_MODE_CONTINUOUS_Y && ds->W <= 32 && !topt().sign_verify_off.load();
    const bool pair_path = (c.mode == XYZB_MODE_BINARY && ds->Wp / 2 <= 128) || sign_pairs || weighted_pairs;
    if (pair_path) {
        c.pair_cap = std::min<u64>(0xffffffffull, std::max<u64>(u64(1) << 20, B * p) * c.pair_scale);
        if (const long long e = topt().pair_cap.load())  // tests force the pair-list regrow path
            c.pair_cap = std::min<u64>(c.pair_cap, std::max<u64>(1, u64(e)) * c.pair_scale);
        ds->pairs.ensure(c.pair_cap * sizeof(kern::PairRec));
        if (c.topk_all) ds->tk_sint.ensure(c.pair_cap * 4);
        ds->npairs.ensure(nbatches * 4);
        XYZB_CUDA(cudaMemsetAsync(ds->npairs.p, 0, nbatches * 4, st));
    }
    // binned verify (binned_verify.cuh): binary columns of <= 80 16-byte slices, X much larger than L2
    {
        const long long bsel = topt().binned.load();  // 1 forces it (tests), -1 disables it
        const bool ok = c.mode == XYZB_MODE_BINARY && pair_path && !sign_pairs && !weighted_pairs &&
                        ds->Wp / 2 <= 80 && p <= (u64(1) << 20) && R < (u64(1) << bins::kRunBits);
        c.binned = ok && (bsel == 1 || (bsel == 0 && p * ds->Wp * 8 >= (u64(512) << 20)));
    }
    if (c.binned) {
        int ws = 20;  // z-side windows of ~84 MB (L2-resident while their bins are verified)
        while (ws > 10 && (u64(1) << ws) * ds->Wp * 8 > (u64(88) << 20)) --ws;
        if (const long long w = topt().binned_wshift.load()) ws = static_cast<int>(w);
        while (ceil_div(p, u64(1) << ws) > bins::kMaxRegions) ++ws;
        c.wshift = ws;
        c.nkt = static_cast<int>(ceil_div(p, u64(1) << ws));
        c.nbj = ceil_div(p, bins::kBinJT);
        c.nbh = ceil_div(c.nbj, u64(1) << bins::kHiBits);
        const u64 nbk = u64(c.nkt) * c.nbh;
        // capacities: 1.25x the last search's mean fills (+ slack), else the batches' pair capacity spread evenly
        const u64 mean = ds->bin_hint ? ds->bin_hint : ceil_div(nbatches * c.pair_cap, 2 * nbk);
        c.cap_bucket = std::min<u64>(0xffffffffull / nbk, mean + mean / 4 + 4096);
        c.cap_kt = std::min<u64>(0xffffffffull / u64(c.nkt), c.nbh * mean + c.nbh * mean / 4 + 65536);
        c.ovf_cap = std::min<u64>(0xffffffffull,
                                  std::max<u64>({u64(1) << 20, nbk * c.cap_bucket / 16, ds->bin_ovf_hint}));
        if (const long long cap = topt().binned_cap.load()) {  // tests: tiny regions and overflow list (redo path)
            c.cap_bucket = std::max<u64>(1, u64(cap));
            c.cap_kt = c.cap_bucket * c.nbh;
            c.ovf_cap = std::max<u64>(c.cap_bucket, ds->bin_ovf_hint);
        }
        ds->bin_s.ensure(u64(c.nkt) * c.cap_kt * 8);
        ds->bin_wcnt.ensure(u64(c.nkt) * 4);
        XYZB_CUDA(cudaMemsetAsync(ds->bin_wcnt.p, 0, u64(c.nkt) * 4, st));
        ds->bin_b.ensure(nbk * c.cap_bucket * 8);
        ds->bin_d.ensure(nbk * c.cap_bucket * 8);
        ds->bin_cnt.ensure(nbk * 4);
        ds->bin_start.ensure(u64(c.nkt) * c.nbj * 4);
        ds->bin_fill.ensure(u64(c.nkt) * c.nbj * 4);
        ds->bin_boff.ensure(u64(c.nkt) * (c.nbj + 1) * 4);
        ds->bin_ovf.ensure(c.ovf_cap * 8);
        ds->bin_ovfn.ensure(4);
        ds->bin_zero.ensure(4);
        XYZB_CUDA(cudaMemsetAsync(ds->bin_cnt.p, 0, nbk * 4, st));
        XYZB_CUDA(cudaMemsetAsync(ds->bin_ovfn.p, 0, 4, st));
        XYZB_CUDA(cudaMemsetAsync(ds->bin_zero.p, 0, 4, st));
        if (c.topk_all) ds->tk_sint.ensure(std::max(c.nbh * c.cap_bucket, c.ovf_cap) * 4);
    }
    const u32 hmax = 8u;  // held columns per item (pair expansion chunks)
    // Grouping + join, by the run's bucket space 2^M against p:
    //   4 <= M <= 16, dense: two CTAs per run splitting a 16-bit shared bucket table (split_group_join);
    //   M = 17, 18, dense:   a 2^(M-16)-CTA cluster of such tables (msplit_group_join);
    //   19 <= M <= 24, dense: partition pass + one CTA per (run, partition) (part_group.cuh);
    //   sparse (2^M > 4p + 1024), M <= 31: the same partition pass with shared hash tables (a partition
    //     above its capacity raises povf: the search is redone on the sorted path);
    //   otherwise (M < 4, M > 31, a hashed overflow): per-run cluster radix sorts of symmetric keys.
    // The grouping test option forces the sorted path (1), the partition path for any M <= 24 (2) or the
    // cluster of 16-bit tables for M = 19, 20 and sparse spaces (3).
    const long long gsel = topt().grouping.load();
    const bool dense = (u64(1) << M) <= 4 * p + 1024;
    const bool part_hash = sizeof(K) == 4 && M >= 2 && M <= 31 && !dense && !c.no_hash &&
                           (gsel == kGroupAuto || gsel == kGroupPart);
    const bool part_path = part_hash || (sizeof(K) == 4 && M >= 2 && M <= 24 && dense &&
                                         (gsel == kGroupPart || (gsel == kGroupAuto && M >= 19)));
    const int pk = part_hash ? kern::part_digits_hash(int(M), p) : kern::part_digits(int(M), p);
    if (part_path) {
        ds->pgrp.ensure(kern::part_scratch_words(pk, B) * 4);
        ds->pent.ensure(cap * 8);
    }
    const bool ms_path = !part_path && sizeof(K) == 4 && M >= 17 && M <= 20 &&
                         ((gsel == kGroupAuto && M <= 18 && dense) || gsel == kGroupMsplit) &&
                         kern::msplit_schedulable(int(M));
    const bool split_path = !part_path && !ms_path && sizeof(K) == 4 && M >= 4 && M <= 16 && dense &&
                            gsel == kGroupAuto;
    if (ms_path) {
        if (kern::msplit_group_scratch(int(M), p)) ds->gtab.ensure(kern::msplit_group_scratch(int(M), p) * 4);
        ds->slots.ensure(kSMs * 4);
        XYZB_CUDA(cudaMemsetAsync(ds->slots.p, 0, kSMs * 4, st));
    }
    if (split_path) {
        if (kern::split_group_scratch(int(M), p)) ds->gtab.ensure(kern::split_group_scratch(int(M), p) * 4);
        ds->slots.ensure(kSMs * 4);
        XYZB_CUDA(cudaMemsetAsync(ds->slots.p, 0, kSMs * 4, st));
    }
    // the binned verify bins the pairs after the join, so a dense partition join can emit in the same pass
    // as it counts |E_r| when the runs are expected far below the guard (p^2 / 2^M <= guard / 8): a run that
    // still turns out over the guard has its pairs dropped by bin_window
    // binary keys of the partition path: the projection counts the partition sizes itself
    const bool fused_count = part_path && !xy && sizeof(K) == 4 && M <= 31;
    // ... and with the binned verify nothing reads the keys afterwards (hits recompute a key from the draws):
    // the partition records come from the row planes directly
    const bool keyless = fused_count && c.binned;
    // keyless: 4-byte records (local bucket | column) where both fit 32 bits ...
    const bool packed = keyless && kern::part_packed_ok(int(M) - pk, p, part_hash);
    // ... and no count pass at all: every partition owns a fixed region of 2.5 x its mean size (+ 64) — a run
    // that drew a row twice has two equal key bits, and when both are partition digits half of its partitions
    // hold twice the mean (about two of config 4's 800 runs; their sizes spread by a few percent more where
    // neighbouring columns are correlated). An overflow (three equal digit bits, or keys far from uniform)
    // is flagged on the device and the search redone with counted partitions; after two such searches the
    // dataset counts from then on
    const long long fsel = topt().part_fixed.load();
    const bool fixed_part = packed && !c.no_fixed_part && ds->part_fixed_fails < 2 && fsel >= 0;
    const u64 pmean = ceil_div(p, u64(1) << pk);
    const u32 fixed_cap = !fixed_part ? 0u : fsel > 0 ? static_cast<u32>(fsel) : static_cast<u32>(2 * pmean + pmean / 2 + 64);
    if (fixed_part) ds->pent.ensure(std::max<u64>(cap * 8, (B << pk) * u64(fixed_cap) * 4 + 16));
    const bool one_pass_join = c.binned && part_path && !part_hash && !c.no_one_pass &&
                               (double(p) * double(p) / std::ldexp(1.0, int(M)) <= double(c.guard) / 8.0 ||
                                topt().one_pass_join.load() == 1);
    const int bits = static_cast<int>(M);
    for (u64 b0 = 0, batch_idx = 0; b0 < R; b0 += B, ++batch_idx) {
        const u64 nb = std::min(B, R - b0);
        Nvtx nv_batch("xyzb:batch");
        const u32* rows = ds->rows.as<u32>() + b0 * M;
        const u32* rid = ds->rid.as<u32>() + b0;
        const int8_t* rsign = ds->rsign.as<int8_t>() + b0;
        K* k0 = ds->keys[0].as<K>();
        cudaEvent_t e0 = clk.mark();
        // ---- project ----
        if (!xy && fused_count) {  // xorc first, then the keys with the partition sizes counted on the fly
            if constexpr (sizeof(K) == 4) {
                kern::ykey_xorc<K><<<static_cast<u32>(ceil_div(nb, 128)), 128, 0, st>>>(
                    rows, int(M), ds->yk_bits.as<u64>(), rsign, static_cast<u32>(nb), ds->xorc.as<K>());
                XYZB_LAUNCH_CHECK();
                XYZB_CUDA(cudaMemsetAsync(ds->pgrp.p, 0, (nb << pk) * 4, st));
                dim3 g(static_cast<u32>(ceil_div(ds->P32, 128)), static_cast<u32>(nb));
                if (!fixed_part) {
                    auto* pc = keyless ? kern::project_count<false> : kern::project_count<true>;
                    pc<<<g, 128, 0, st>>>(ds->Xr.as<u32>(), ds->P32, p, rows, int(M), k0, ds->xorc.as<K>(),
                                          int(M) - pk, part_hash ? 1 : 0, ds->pgrp.as<u32>());
                    XYZB_LAUNCH_CHECK();
                }
                c.launches[XYZB_STAGE_PROJECT] += fixed_part ? 1 : 2;
            }
        } else if (!xy) {
            dim3 g(static_cast<u32>(ceil_div(ds->P32, 128)), static_cast<u32>(nb));
            kern::project_bits_t<K><<<g, 128, 0, st>>>(ds->Xr.as<u32>(), ds->P32, p, rows, int(M), k0);
            XYZB_LAUNCH_CHECK();
            kern::ykey_xorc<K><<<static_cast<u32>(ceil_div(nb, 128)), 128, 0, st>>>(
                rows, int(M), ds->yk_bits.as<u64>(), rsign, static_cast<u32>(nb), ds->xorc.as<K>());
            XYZB_LAUNCH_CHECK();
            c.launches[XYZB_STAGE_PROJECT] += 2;
        } else {
            real::resp_xorc<K><<<static_cast<u32>(ceil_div(nb, 128)), 128, 0, st>>>(rows, int(M), ds->yreal.as<double>(),
                                                                                 rsign, static_cast<u32>(nb),
                                                                                 ds->xorc.as<K>());
            XYZB_LAUNCH_CHECK();
            const u64* mts = (unbiased || coins) ? ds->mt_state.as<u64>() + b0 * 313 : nullptr;
            if (unbiased) {
                XYZB_CUDA(cudaMemsetAsync(k0, 0, nb * p * sizeof(K), st));
                real::unbiased_keys<K><<<static_cast<u32>(nb), real::kMtThreads, 0, st>>>(mts, p, rows, int(M),
                                                                                        ds->Xr64.as<double>(), k0);
                XYZB_LAUNCH_CHECK();
                c.launches[XYZB_STAGE_PROJECT] += 2;
            } else {
                // sign transform: key bits from the (v > 0) planes, coin mask from the (v == 0) planes
                dim3 g(static_cast<u32>(ceil_div(ds->P32, 128)), static_cast<u32>(nb));
                kern::project_bits_t<K><<<g, 128, 0, st>>>(ds->Xpos.as<u32>(), ds->P32, p, rows, int(M), k0);
                XYZB_LAUNCH_CHECK();
                c.launches[XYZB_STAGE_PROJECT] += 2;
                if (coins) {
                    kern::project_bits_t<K><<<g, 128, 0, st>>>(ds->Xzero.as<u32>(), ds->P32, p, rows, int(M),
                                                               ds->zmask.as<K>());
                    XYZB_LAUNCH_CHECK();
                    real::popc_count<K><<<grid_for(nb * p, 256, 4096), 256, 0, st>>>(ds->zmask.as<K>(), nb * p,
                                                                                     ds->zcount.as<u32>());
                    XYZB_LAUNCH_CHECK();
                    c.launches[XYZB_STAGE_PROJECT] += 2;
                }
                if (coins) {
                    u32* cnt = reinterpret_cast<u32*>(hp + hbytes - 96 - 2 * R * 4) + 2 * batch_idx + 1;
                    *cnt = static_cast<u32>(nb * p);
                    small_copy(ds->zcnt_n.p, cnt, 4, st);
                    scan::exclusive<u32>(ds->zcount.as<u32>(), ds->zcnt_n.as<u32>(), ds->zoff.as<u32>(),
                                         reinterpret_cast<u32*>(ds->partial.p), st, &c.launches[XYZB_STAGE_PROJECT]);
                    real::sign_coins<K><<<static_cast<u32>(nb), real::kMtThreads, 0, st>>>(
                        mts, p, ds->zmask.as<K>(), ds->zoff.as<u32>(), k0);
                    XYZB_LAUNCH_CHECK();
                    c.launches[XYZB_STAGE_PROJECT] += 1;
                }
            }
        }
        cudaEvent_t e1 = clk.mark();
        clk.span(XYZB_STAGE_PROJECT, e0, e1);
        c.bytes[XYZB_STAGE_PROJECT] += nb * (unbiased ? 8 * M * p : ceil_div(M * p, 8)) + nb * p * sizeof(K);
        K* kb[2] = {ds->keys[0].as<K>(), ds->keys[1].as<K>()};
        u32* vb[2] = {ds->vals[0].as<u32>(), ds->vals[1].as<u32>()};
        u32* nitems = ds->nblocks.as<u32>() + batch_idx;
        u32* npairs_b = pair_path ? ds->npairs.as<u32>() + batch_idx : nullptr;
        const u32* sv = nullptr;
        const K* sorted_keys = nullptr;
        int vshift = 0;
        cudaEvent_t e2;
        if (part_path) {
            // ---- group: partition pass (per-run partitions that hold both sides of every block) ----
            if constexpr (sizeof(K) == 4) {
                auto scatter_records = [&](u32* cursor) {  // the records straight from the row planes (no key array)
                    dim3 g(static_cast<u32>(ceil_div(ds->P32, 128)), static_cast<u32>(nb));
                    auto* ps = packed ? kern::project_scatter<true> : kern::project_scatter<false>;
                    ps<<<g, 128, kern::project_scatter_smem(pk), st>>>(ds->Xr.as<u32>(), ds->P32, p, rows, int(M), ds->xorc.as<K>(), int(M) - pk,
                                          part_hash ? 1 : 0, cursor, ds->pent.as<uint2>(), fixed_cap,
                                          ds->povf.as<u32>() + 1);
                    XYZB_LAUNCH_CHECK();
                };
                // fixed regions: the scatter's cursors (zeroed above) end as the partition sizes, scanned after
                if (fixed_part) scatter_records(ds->pgrp.as<u32>());
                kern::part_partition_launch(k0, nb, p, int(M), pk, part_hash, ds->xorc.as<K>(), ds->tot.as<u64>(),
                                            ds->work_run.as<u64>(), ds->pgrp.as<u32>(), ds->pent.as<uint2>(), st,
                                            fused_count, !keyless);
                c.launches[XYZB_STAGE_SORT] += fused_count ? 2 : 3;
                if (keyless && !fixed_part) scatter_records(ds->pgrp.as<u32>() + (nb << pk));
                e2 = clk.mark();
                clk.span(XYZB_STAGE_SORT, e1, e2);
                const u64 rec_bytes = packed ? 4 : 8;
                if (keyless)  // M row-plane words per 32 columns (twice with a count pass), records written
                    c.bytes[XYZB_STAGE_SORT] += nb * ((fixed_part ? 1 : 2) * M * ds->P32 * 4 + p * rec_bytes);
                else  // keys read twice, records written
                    c.bytes[XYZB_STAGE_SORT] += nb * p * (2 * sizeof(K) + 8);
                c.bytes[XYZB_STAGE_JOIN] += nb * p * rec_bytes * (one_pass_join ? 1 : 2);  // records read per join pass
                // ---- join: per (run, partition) bucket tables in shared memory; |E_r|, guard, blocks ----
                kern::part_join_launch(nb, p, int(M), pk, part_hash, ds->xorc.as<K>(), c.guard, hmax, vb[0],
                                       ds->tot.as<u64>(), ds->work_run.as<u64>(), ds->items.as<kern::Item>(), nitems,
                                       static_cast<u32>(item_cap), npairs_b, ds->pairs.as<kern::PairRec>(),
                                       static_cast<u32>(c.pair_cap), ds->pgrp.as<u32>(), ds->pent.as<uint2>(),
                                       ds->povf.as<u32>(), st, one_pass_join, packed, fixed_cap);
                c.launches[XYZB_STAGE_JOIN] += one_pass_join ? 1 : 2;
            } else {
                throw internal_error("xyzb: partitioned grouping needs 32-bit keys");
            }
            sv = vb[0];
        } else if (ms_path) {
            // ---- group + join fused: 2^(M-16) CTAs per run, 16-bit tables split by parities of c's zero bits ----
            if constexpr (sizeof(K) == 4) {
                if (!kern::msplit_group_join_launch(k0, nb, p, int(M), ds->xorc.as<K>(), c.guard, hmax, vb[0],
                                                    ds->tot.as<u64>(), ds->work_run.as<u64>(),
                                                    ds->items.as<kern::Item>(), nitems, static_cast<u32>(item_cap),
                                                    npairs_b, ds->pairs.as<kern::PairRec>(),
                                                    static_cast<u32>(c.pair_cap), ds->gtab.as<u32>(),
                                                    ds->slots.as<u32>(), st))
                    throw internal_error("xyzb: the grouping cluster could not be launched");
            }
            XYZB_LAUNCH_CHECK();
            c.launches[XYZB_STAGE_SORT] += 1;
            sv = vb[0];
            e2 = clk.mark();
            clk.span(XYZB_STAGE_SORT, e1, e2);
            c.bytes[XYZB_STAGE_SORT] += nb * p * (2 * sizeof(K) + 4);  // keys read twice, indices written
            c.pairs_in_sort = true;
        } else if (split_path) {
            // ---- group + join fused: two CTAs per run, each half of the 16-bit bucket table ----
            if constexpr (sizeof(K) == 4) {  // M <= 16 always runs with u32 keys
                kern::split_group_join_launch<K>(k0, nb, p, int(M), ds->xorc.as<K>(), c.guard, hmax, vb[0],
                                                 ds->tot.as<u64>(), ds->work_run.as<u64>(),
                                                 ds->items.as<kern::Item>(), nitems, static_cast<u32>(item_cap),
                                                 npairs_b, ds->pairs.as<kern::PairRec>(),
                                                 static_cast<u32>(c.pair_cap), ds->gtab.as<u32>(),
                                                 ds->slots.as<u32>(), st);
            } else {
                throw internal_error("xyzb: split grouping needs 32-bit keys");
            }
            XYZB_LAUNCH_CHECK();
            c.launches[XYZB_STAGE_SORT] += 1;
            sv = vb[0];
            e2 = clk.mark();
            clk.span(XYZB_STAGE_SORT, e1, e2);
            c.bytes[XYZB_STAGE_SORT] += nb * p * (2 * sizeof(K) + 4);  // keys read twice, indices written
            c.pairs_in_sort = true;
        } else {
            // symmetric keys (u = min(v, v^c), side bit): the join needs no lookups;
            // M = 64 keeps plain keys and binary-search partner lookups
            const bool ukeys = M + 1 <= sizeof(K) * 8;
            const int sbits = ukeys ? bits + 1 : bits;
            if (pair_path) {  // pair-list hits look keys up by column: keep the unsorted keys
                ds->keys_x.ensure(nb * p * sizeof(K));
                XYZB_CUDA(cudaMemcpyAsync(ds->keys_x.p, k0, nb * p * sizeof(K), cudaMemcpyDeviceToDevice, st));
            }
            if (ukeys) {
                kern::ukey_transform<K><<<grid_for(nb * p, 256, 4096), 256, 0, st>>>(k0, p, nb * p, ds->xorc.as<K>());
                XYZB_LAUNCH_CHECK();
                c.launches[XYZB_STAGE_SORT] += 1;
            }
            // ---- sort: one cluster per run (DSMEM histogram exchange) ----
            const int res = rsort::sort_runs_launch<K>(kb[0], vb[0], kb[1], vb[1], nb, p, sbits, st);
            XYZB_LAUNCH_CHECK();
            c.launches[XYZB_STAGE_SORT] += 1;
            e2 = clk.mark();
            clk.span(XYZB_STAGE_SORT, e1, e2);
            c.bytes[XYZB_STAGE_SORT] += nb * p * (2 * sizeof(K) + 8) * u64((sbits + 7) / 8);
            sv = vb[res];
            sorted_keys = kb[res];
            vshift = ukeys ? 1 : 0;
            // ---- join (+ guard bookkeeping) ----
            XYZB_CUDA(cudaMemsetAsync(ds->tot.p, 0, nb * 8, st));
            XYZB_CUDA(cudaMemsetAsync(ds->work_run.p, 0, nb * 8, st));
            dim3 gj(static_cast<u32>(ceil_div(p, 256)), static_cast<u32>(nb));
            if (ukeys) {
                kern::ujoin_count<K><<<gj, 256, 0, st>>>(kb[res], p, ds->xorc.as<K>(), ds->tot.as<u64>(),
                                                         ds->work_run.as<u64>());
                XYZB_LAUNCH_CHECK();
                kern::ujoin_emit<K><<<gj, 256, 0, st>>>(kb[res], p, ds->xorc.as<K>(), ds->tot.as<u64>(), c.guard, hmax,
                                                        ds->items.as<kern::Item>(), nitems, static_cast<u32>(item_cap),
                                                        npairs_b, ds->pairs.as<kern::PairRec>(),
                                                        static_cast<u32>(c.pair_cap), sv);
                XYZB_LAUNCH_CHECK();
            } else {
                kern::join_count<K><<<gj, 256, 0, st>>>(kb[res], p, int(M), ds->xorc.as<K>(), nullptr,
                                                        ds->tot.as<u64>(), ds->work_run.as<u64>());
                XYZB_LAUNCH_CHECK();
                kern::join_emit<K><<<gj, 256, 0, st>>>(kb[res], p, int(M), ds->xorc.as<K>(), nullptr, ds->tot.as<u64>(),
                                                       c.guard, hmax, ds->items.as<kern::Item>(), nitems,
                                                       static_cast<u32>(item_cap), npairs_b,
                                                       ds->pairs.as<kern::PairRec>(), static_cast<u32>(c.pair_cap), sv);
                XYZB_LAUNCH_CHECK();
            }
            c.launches[XYZB_STAGE_JOIN] += 2;
        }
        kern::book_runs<<<static_cast<u32>(ceil_div(nb, 256)), 256, 0, st>>>(
            static_cast<u32>(nb), ds->tot.as<u64>(), ds->work_run.as<u64>(), c.guard, rid, ds->enumerated.as<u64>(),
            ds->verified.as<u64>());
        XYZB_LAUNCH_CHECK();
        c.launches[XYZB_STAGE_JOIN] += 1;
        cudaEvent_t e3 = clk.mark();
        clk.span(XYZB_STAGE_JOIN, e2, e3);
        if (!part_path && !c.pairs_in_sort)  // sorted / bucket paths: sorted keys + indices read by count and emit
            c.bytes[XYZB_STAGE_JOIN] += nb * p * (sizeof(K) + 4) * 2;
        // ---- verify ----
        Nvtx nv_verify("xyzb:verify");
        kern::VerifyArgs A;
        A.items = ds->items.as<kern::Item>();
        A.nitems = nitems;
        A.item_cap = static_cast<u32>(item_cap);
        A.tot = ds->tot.as<u64>();
        A.guard = c.guard;
        A.sv = sv;
        A.S = p;
        const bool unsorted = split_path || ms_path || part_path;
        A.vkeys = unsorted ? static_cast<const void*>(k0) : static_cast<const void*>(sorted_keys);
        A.vkeys_by_pos = unsorted ? 0 : 1;
        A.xkeys = unsorted ? static_cast<const void*>(k0) : ds->keys_x.p;
        A.key64 = sizeof(K) == 8;
        A.vshift = vshift;
        A.rid = rid;
        A.run_sign = rsign;
        A.p = p;
        A.hits = ds->hits.as<kern::DevHit>();
        A.hit_count = ds->hit_count.as<u32>();
        A.hit_cap = ds->hit_cap;
        A.krows = nullptr;
        A.kM = 0;
        A.kXc = nullptr;
        A.kWp = 0;
        A.sint_out = nullptr;
        A.rank_thr = nullptr;
        A.rank_binary = c.mode == XYZB_MODE_BINARY ? 1 : 0;
        A.rank_n = static_cast<u32>(c.n);
        if (c.topk_all) {
            if (pair_path) A.sint_out = ds->tk_sint.as<u32>();
            A.rank_thr = &ds->tk_state.as<topk::State>()->thr;
        }
        const u32 vgrid = kSMs * 8;
        if (pair_path) {
            u32* np = ds->npairs.as<u32>() + batch_idx;
            kern::expand_pairs<<<vgrid, 256, 0, st>>>(A.items, A.nitems, A.item_cap, p, ds->pairs.as<kern::PairRec>(),
                                                      static_cast<u32>(c.pair_cap), sv);
            XYZB_LAUNCH_CHECK();
            c.launches[XYZB_STAGE_JOIN] += 1;
            cudaEvent_t ev0 = clk.mark();
            clk.span(XYZB_STAGE_JOIN, e3, ev0);  // pair expansion belongs to the join
            if (c.binned) {  // the batch's pairs go to their z-side windows; verified after the last batch
                func_smem(bins::bin_window, bins::bin_window_smem());
                bins::bin_window<<<kSMs * 4, bins::kPartThreads, bins::bin_window_smem(), st>>>(
                    ds->pairs.as<kern::PairRec>(), np, static_cast<u32>(c.pair_cap), A.nitems, A.item_cap,
                    static_cast<u32>(b0), rsign, static_cast<u32>(nb), ds->tot.as<u64>(), c.guard, c.wshift,
                    static_cast<u32>(c.nkt),
                    ds->bin_s.as<u64>(), static_cast<u32>(c.cap_kt), ds->bin_wcnt.as<u32>(), ds->bin_ovf.as<u64>(),
                    static_cast<u32>(c.ovf_cap), ds->bin_ovfn.as<u32>());
                XYZB_LAUNCH_CHECK();
                c.launches[XYZB_STAGE_JOIN] += 1;
                clk.span(XYZB_STAGE_JOIN, ev0, clk.mark());
                continue;
            }
            if (sign_pairs) {
                const kern::SignStrength g = sign_strength(c);
                kern::verify_pairs_sign<kern::kSignQB><<<vgrid, 256, 0, st>>>(A, ds->pairs.as<kern::PairRec>(), np,
                                                                              static_cast<u32>(c.pair_cap), g);
                XYZB_LAUNCH_CHECK();
                c.sign_verify = true;
                c.launches[XYZB_STAGE_VERIFY] += 1;
                cudaEvent_t ev1 = clk.mark();
                clk.span(XYZB_STAGE_VERIFY, ev0, ev1);
                c.verify_spans.push_back({ev0, ev1});
                if (c.topk_all) {
                    topk_after_batch(c, true, A, np, &c.launches[XYZB_STAGE_MERGE], &g);
                    clk.span(XYZB_STAGE_MERGE, ev1, clk.mark());
                }
                continue;
            }
            if (weighted_pairs) {
                const kern::WeightedQ g{ds->Xc.as<u64>(), static_cast<u32>(ds->Wp), ds->W, ds->spos.as<u64>(),
                                        ds->sneg.as<u64>(), ds->yplanes.as<u64>(), c.wqinv, c.norm, c.gamma, c.wqdelta,
                                        kern::WeightedStrength{ds->Xc.as<u64>(), static_cast<u32>(ds->Wp),
                                                               ds->spos.as<u64>(), ds->sneg.as<u64>(),
                                                               ds->wabs.as<double>(), c.norm, c.gamma}};
                kern::verify_pairs_weighted<kern::kWeightQB><<<vgrid, 256, 0, st>>>(
                    A, ds->pairs.as<kern::PairRec>(), np, static_cast<u32>(c.pair_cap), g);
                XYZB_LAUNCH_CHECK();
                c.launches[XYZB_STAGE_VERIFY] += 1;
                cudaEvent_t ev1 = clk.mark();
                clk.span(XYZB_STAGE_VERIFY, ev0, ev1);
                c.verify_spans.push_back({ev0, ev1});
                if (c.topk_all) {
                    topk_after_batch(c, true, A, np, &c.launches[XYZB_STAGE_MERGE], nullptr, &g);
                    clk.span(XYZB_STAGE_MERGE, ev1, clk.mark());
                }
                continue;
            }
            const u64 W2 = ds->Wp / 2;
            // team of G lanes, NIT 16-byte chunks of each column per lane, measured on B200
            // (tools/sweep_verify.py, tools/l2_window2.cu): long columns (>= 512 B) take 8..32-lane
            // teams with up to 64 B per lane and column walking one pair at a time, short ones
            // full-column teams with the next pair's columns prefetched
            const u64 chunks = W2 >= 32 ? 4 : 1;
            const bool simple = W2 >= 32;
            int G = 1;
            while (G < 32 && u64(G) * chunks < W2) G <<= 1;
            const int nit = static_cast<int>(ceil_div(W2, G));
            const auto* PR = ds->pairs.as<kern::PairRec>();
            const u32 pc = static_cast<u32>(c.pair_cap);
            const u64* X = ds->Xc.as<u64>();
            const u32 Wp = static_cast<u32>(ds->Wp);
            const u64* Y = ds->yk_bits.as<u64>();
            const u32 n32 = static_cast<u32>(c.n);
#define XYZB_VP(GG, NN)                                                                                          \
    do {                                                                                                         \
        if (simple)                                                                                              \
            kern::verify_pairs_simple<GG, NN><<<vgrid, 256, 0, st>>>(A, PR, np, pc, X, Wp, Y, n32, c.astar);     \
        else                                                                                                     \
            kern::verify_pairs_binary<GG, NN><<<vgrid, 256, 0, st>>>(A, PR, np, pc, X, Wp, Y, n32, c.astar);     \
    } while (0)
#define XYZB_VP4(GG) \
    switch (nit) { case 1: XYZB_VP(GG, 1); break; case 2: XYZB_VP(GG, 2); break; case 3: XYZB_VP(GG, 3); break; default: XYZB_VP(GG, 4); }
            switch (G) {
                case 1: XYZB_VP4(1); break;
                case 2: XYZB_VP4(2); break;
                case 4: XYZB_VP4(4); break;
                case 8: XYZB_VP4(8); break;
                case 16: XYZB_VP4(16); break;
                default: XYZB_VP4(32); break;
            }
#undef XYZB_VP4
#undef XYZB_VP
            XYZB_LAUNCH_CHECK();
            c.launches[XYZB_STAGE_VERIFY] += 1;
            cudaEvent_t ev1 = clk.mark();
            clk.span(XYZB_STAGE_VERIFY, ev0, ev1);
            c.verify_spans.push_back({ev0, ev1});
            if (c.topk_all) {
                topk_after_batch(c, true, A, np, &c.launches[XYZB_STAGE_MERGE]);
                clk.span(XYZB_STAGE_MERGE, ev1, clk.mark());
            }
            continue;
        } else if (c.mode == XYZB_MODE_BINARY) {  // long columns (n > 8192): warp per pair
            kern::BinaryStrength f{ds->Xc.as<u64>(), static_cast<u32>(ds->Wp), ds->yk_bits.as<u64>(),
                                   static_cast<u32>(c.n), c.astar};
            kern::verify_items<<<vgrid, 256, 0, st>>>(A, f);
        } else if (c.mode == XYZB_MODE_CONTINUOUS_Y) {
            kern::WeightedStrength f{ds->Xc.as<u64>(), static_cast<u32>(ds->Wp), ds->spos.as<u64>(), ds->sneg.as<u64>(),
                                     ds->wabs.as<double>(), c.norm, c.gamma};
            kern::verify_items<<<vgrid, 256, 0, st>>>(A, f);
        } else {
            // the fp32 response in shared memory when it fits (n <= 49152), else through L1
            ds->yreal32.ensure(ds->n4 * 4);
            real::to_f32<<<grid_for(ds->n4, 256, 256), 256, 0, st>>>(ds->yreal.as<double>(), ds->n4,
                                                                     ds->yreal32.as<float>());
            XYZB_LAUNCH_CHECK();
            const size_t ysm = ds->n4 * 4;
            const bool ysmem = ysm <= (size_t(192) << 10);
            if (ysmem && ysm > (size_t(48) << 10)) {
                func_smem(kern::verify_items_real<true>, ysm);
                func_smem(kern::verify_items_real<false>, ysm);
            }
            if (unbiased) {
                kern::RealStrength<true> f{ds->Xc32.as<float>(), ds->n4, ds->yreal32.as<float>(), c.norm, c.gamma};
                if (ysmem) kern::verify_items_real<true><<<vgrid, 256, ysm, st>>>(A, f);
                else kern::verify_items<<<vgrid, 256, 0, st>>>(A, f);
            } else {
                kern::RealStrength<false> f{ds->Xc32.as<float>(), ds->n4, ds->yreal32.as<float>(), c.norm, c.gamma};
                if (!topt().sign_verify_off.load() && ds->Spos.p) {
                    // sign transform: strengths from column sign bits and the response's bit planes
                    kern::SignStrength g{ds->Spos.as<u64>(), ds->Snz.as<u64>(), ds->W, ds->yplanes.as<u64>(),
                                         c.qsum, ds->has_zero, c.qinv, c.norm, c.gamma, c.qdelta, f};
                    const size_t psm = size_t(c.qB + 1) * ds->W * 8;
                    kern::verify_items_sign<kern::kSignQB>
                        <<<vgrid, 256, (ds->W > 32 && psm <= (size_t(48) << 10)) ? psm : 0, st>>>(A, g);
                    c.sign_verify = true;
                } else if (ysmem) {
                    kern::verify_items_real<false><<<vgrid, 256, ysm, st>>>(A, f);
                } else {
                    kern::verify_items<<<vgrid, 256, 0, st>>>(A, f);
                }
            }
        }
        XYZB_LAUNCH_CHECK();
        c.launches[XYZB_STAGE_VERIFY] += 1;
        cudaEvent_t e4 = clk.mark();
        clk.span(XYZB_STAGE_VERIFY, e3, e4);
        c.verify_spans.push_back({e3, e4});
        if (c.topk_all) {
            topk_after_batch(c, false, A, nullptr, &c.launches[XYZB_STAGE_MERGE]);
            clk.span(XYZB_STAGE_MERGE, e4, clk.mark());
        }
    }
    if (c.binned) binned_verify(c);
}

// Top-K over all candidates: the merged list holds every first occurrence at
// or above the final rank threshold (a bin edge); keep those at or above the
// K-th ranked strength — the reference's A.8 list at that gamma — and remap
// the top-K indices. Returns gamma_effective.
double topk_filter(std::vector<xyzb_hit>& hits, std::vector<u64>& order, std::vector<u64>& topk) {
    if (topk.empty()) return 0.0;
    const double sK = hits[topk.back()].strength;
    std::vector<u64> remap(hits.size(), ~0ull);
    size_t w = 0;
    for (size_t i = 0; i < hits.size(); ++i) {
        if (!(hits[i].strength >= sK)) continue;
        remap[i] = w;
        hits[w] = hits[i];
        order[w] = order[i];
        ++w;
    }
    hits.resize(w);
    order.resize(w);
    for (u64& t : topk) t = remap[t];
    return sK;
}

// Keep the first occurrence of each (min, max, sign), order by (run, A.5),
// rank for top-K; copy the report arrays to the host.
void merge_hits(SearchCtx& c, u32 H, u32 rmax, std::vector<xyzb_hit>& hits_out, std::vector<u64>& order_out,
                std::vector<u64>& topk_out) {
    Nvtx nv("xyzb:merge");
    xyzb_dataset* ds = c.ds;
    cudaStream_t st = ds->stream;
    hits_out.clear();
    order_out.clear();
    topk_out.clear();
    if (H == 0) return;
    u64& L = c.launches[XYZB_STAGE_MERGE];
    if (H <= u32(merge::kSmallMerge) && !topt().merge_large.load()) {
        // short lists: one CTA dedups, orders and ranks in shared memory
        const size_t smem = merge::small_merge_smem(merge::kSmallMerge);
        func_smem(merge::merge_small, smem);
        ds->fin.ensure(u64(H) * sizeof(xyzb_hit));
        ds->fin_order.ensure(u64(H) * 8);
        ds->topidx.ensure(u64(H) * 8 + 16);
        u64* top = ds->topidx.as<u64>();
        u32* counts = reinterpret_cast<u32*>(top + H);
        merge::merge_small<<<1, merge::kSmallThreads, smem, st>>>(
            ds->hits.as<kern::DevHit>(), H, ds->sign_by_rid.as<int8_t>(), rmax, c.plan.L, c.q->top_k,
            ds->fin.as<xyzb_hit>(), ds->fin_order.as<u64>(), top, counts);
        XYZB_LAUNCH_CHECK();
        L += 1;
        const size_t hb = u64(H) * sizeof(xyzb_hit), ob = u64(H) * 8, tb = u64(H) * 8 + 16;
        ds->h_merge.ensure(hb + ob + tb);
        char* hp = ds->h_merge.as<char>();
        XYZB_CUDA(cudaMemcpyAsync(hp, ds->fin.p, hb, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaMemcpyAsync(hp + hb, ds->fin_order.p, ob, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaMemcpyAsync(hp + hb + ob, top, tb, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        const u32* cnt = reinterpret_cast<const u32*>(hp + hb + ob + u64(H) * 8);
        const u32 K = cnt[0], kk = cnt[1];
        hits_out.assign(reinterpret_cast<const xyzb_hit*>(hp), reinterpret_cast<const xyzb_hit*>(hp) + K);
        order_out.assign(reinterpret_cast<const u64*>(hp + hb), reinterpret_cast<const u64*>(hp + hb) + K);
        topk_out.assign(reinterpret_cast<const u64*>(hp + hb + ob), reinterpret_cast<const u64*>(hp + hb + ob) + kk);
        return;
    }
    // dedup table
    u64 T = 64;
    while (T < 2ull * H) T <<= 1;
    ds->tkeys.ensure(T * 8);
    ds->tvals.ensure(T * 8);
    merge::fill_u64<<<grid_for(T, 256), 256, 0, st>>>(ds->tkeys.as<u64>(), T, merge::kEmpty);
    merge::fill_u64<<<grid_for(T, 256), 256, 0, st>>>(ds->tvals.as<u64>(), T, merge::kEmpty);
    ds->rmin.ensure(8);
    XYZB_CUDA(cudaMemcpyAsync(ds->rmin.p, &rmax, 4, cudaMemcpyHostToDevice, st));
    const kern::DevHit* h = ds->hits.as<kern::DevHit>();
    merge::hash_insert<<<grid_for(H, 256), 256, 0, st>>>(h, H, ds->sign_by_rid.as<int8_t>(), ds->tkeys.as<u64>(),
                                                          ds->tvals.as<u64>(), T - 1);
    ds->keep.ensure(u64(H) * 4);
    ds->kpos.ensure((u64(H) + 1) * 4);
    merge::hash_mark<<<grid_for(H, 256), 256, 0, st>>>(h, H, ds->sign_by_rid.as<int8_t>(), ds->tkeys.as<u64>(),
                                                        ds->tvals.as<u64>(), T - 1, ds->rmin.as<u32>(),
                                                        ds->keep.as<u32>());
    ds->hcount.ensure(8);
    ds->partial.ensure(scan::kGrid * 8);
    XYZB_CUDA(cudaMemcpyAsync(ds->hcount.p, &H, 4, cudaMemcpyHostToDevice, st));
    scan::exclusive<u32>(ds->keep.as<u32>(), ds->hcount.as<u32>(), ds->kpos.as<u32>(),
                         reinterpret_cast<u32*>(ds->partial.p), st, &L);
    ds->kept.ensure(u64(H) * sizeof(kern::DevHit));
    ds->kbufA.ensure(u64(H) * 8);
    ds->kbufB.ensure(u64(H) * 8);
    ds->vbufA.ensure(u64(H) * 4);
    ds->vbufB.ensure(u64(H) * 4);
    merge::compact<<<grid_for(H, 256), 256, 0, st>>>(h, H, ds->keep.as<u32>(), ds->kpos.as<u32>(),
                                                      ds->kept.as<kern::DevHit>(), ds->kbufA.as<u64>());
    L += 6;
    u32 K = 0;
    XYZB_CUDA(cudaMemcpyAsync(&K, ds->kpos.as<u32>() + H, 4, cudaMemcpyDeviceToHost, st));
    XYZB_CUDA(cudaStreamSynchronize(st));
    if (K == 0) return;
    // reference order (run, v, j, k): stable LSD sorts by (j, k), then v, then run
    ds->hist.ensure(rsort::hist_words(1, K) * 4);
    ds->perm.ensure(u64(K) * 8);
    u64* kb[2] = {ds->kbufA.as<u64>(), ds->kbufB.as<u64>()};
    u32* vb[2] = {ds->vbufA.as<u32>(), ds->vbufB.as<u32>()};
    u32* perm = ds->perm.as<u32>();
    u32* perm2 = perm + K;
    int r1 = rsort::sort_segments<u64>(kb, vb, 1, K, 64, ds->hist.as<u32>(), st, &L);  // jk keys from compact
    XYZB_CUDA(cudaMemcpyAsync(perm, vb[r1], u64(K) * 4, cudaMemcpyDeviceToDevice, st));
    int vbits = 1;
    while (vbits < 64 && (c.M >= 64 || (u64(1) << vbits) < (u64(1) << c.M))) ++vbits;
    int rbits = 1;
    while (rbits < 32 && (u64(1) << rbits) < c.plan.sign_by_rid.size()) ++rbits;
    for (int which = 0; which < 2; ++which) {
        merge::order_key<<<grid_for(K, 256), 256, 0, st>>>(ds->kept.as<kern::DevHit>(), perm, K, which, kb[0]);
        const int rr = rsort::sort_segments<u64>(kb, vb, 1, K, which == 0 ? vbits : rbits, ds->hist.as<u32>(), st, &L);
        merge::compose_perm<<<grid_for(K, 256), 256, 0, st>>>(perm, vb[rr], K, perm2);
        XYZB_CUDA(cudaMemcpyAsync(perm, perm2, u64(K) * 4, cudaMemcpyDeviceToDevice, st));
        L += 2;
    }
    r1 = 0;
    XYZB_CUDA(cudaMemcpyAsync(vb[0], perm, u64(K) * 4, cudaMemcpyDeviceToDevice, st));
    ds->fin.ensure(u64(K) * sizeof(xyzb_hit));
    ds->fin_order.ensure(u64(K) * 8);
    ds->tie.ensure(u64(K) * 8);
    int bp = 1;
    while (bp < 32 && (1ull << bp) < c.p) ++bp;
    merge::gather_final<<<grid_for(K, 256), 256, 0, st>>>(ds->kept.as<kern::DevHit>(), vb[r1], K,
                                                           ds->sign_by_rid.as<int8_t>(), c.plan.L, bp,
                                                           ds->fin.as<xyzb_hit>(), ds->fin_order.as<u64>(),
                                                           ds->tie.as<u64>());
    L += 1;
    hits_out.resize(K);
    order_out.resize(K);
    XYZB_CUDA(cudaMemcpyAsync(hits_out.data(), ds->fin.p, u64(K) * sizeof(xyzb_hit), cudaMemcpyDeviceToHost, st));
    XYZB_CUDA(cudaMemcpyAsync(order_out.data(), ds->fin_order.p, u64(K) * 8, cudaMemcpyDeviceToHost, st));
    if (c.q->top_k > 0) {
        // A.10: stable LSD — tie key (min, max, sign) first, then strength desc
        XYZB_CUDA(cudaMemcpyAsync(kb[0], ds->tie.p, u64(K) * 8, cudaMemcpyDeviceToDevice, st));
        const int r2 = rsort::sort_segments<u64>(kb, vb, 1, K, 2 * bp + 1, ds->hist.as<u32>(), st, &L);
        // tie-sorted index list lives in vb[r2]; copy it aside
        ds->topidx.ensure(u64(K) * 12);
        u32* tie_idx = reinterpret_cast<u32*>(ds->topidx.p);
        XYZB_CUDA(cudaMemcpyAsync(tie_idx, vb[r2], u64(K) * 4, cudaMemcpyDeviceToDevice, st));
        const bool bin = c.mode == XYZB_MODE_BINARY;
        merge::primary_key<<<grid_for(K, 256), 256, 0, st>>>(ds->fin.as<xyzb_hit>(), nullptr, tie_idx, K, bin ? 1 : 0,
                                                              static_cast<u32>(c.n), kb[0]);
        int pbits = 64;
        if (bin) {
            pbits = 1;
            while (pbits < 64 && (1ull << pbits) <= c.n) ++pbits;
        }
        const int r3 = rsort::sort_segments<u64>(kb, vb, 1, K, pbits, ds->hist.as<u32>(), st, &L);
        const u64 kk = std::min<u64>(c.q->top_k, K);
        u64* top = reinterpret_cast<u64*>(ds->tvals.p);  // reuse scratch (T >= 2H >= K)
        merge::compose_idx<<<grid_for(kk, 256), 256, 0, st>>>(tie_idx, vb[r3], static_cast<u32>(kk), top);
        L += 2;
        topk_out.resize(kk);
        XYZB_CUDA(cudaMemcpyAsync(topk_out.data(), top, kk * 8, cudaMemcpyDeviceToHost, st));
    }
    XYZB_CUDA(cudaStreamSynchronize(st));
}

// sample_strengths + expected_complexity (search.cpp:136-188,229-291,313-317):
// host-drawn pairs on stream 0, device strengths, fp64 mean in draw order.
template <class Fn>
double estimate_complexity(SearchCtx& c, Fn&& device_strengths) {
    const u64 p = c.p;
    const u64 cnt = c.q->strength_sample_size ? c.q->strength_sample_size : std::min<u64>(100000, 10 * p);
    std::mt19937_64 rng = host::make_stream(c.q->seed, 0);
    std::uniform_int_distribution<size_t> dist(0, p - 1);
    std::vector<u32> pairs(2 * cnt);
    for (u64 t = 0; t < cnt; ++t) {
        size_t j = dist(rng), k = dist(rng);
        while (p > 1 && k == j) k = dist(rng);
        pairs[2 * t] = static_cast<u32>(j);
        pairs[2 * t + 1] = static_cast<u32>(k);
    }
    std::vector<double> s(cnt);
    device_strengths(pairs.data(), cnt, s.data());
    double acc = 0.0;
    for (double v : s) acc += std::pow(v, double(c.M));
    const double mp = acc / double(s.size());
    const double np = double(c.n) * double(p), pd = double(p);
    const double e1 = pd * pd * mp;
    return np + double(c.q->l) * (double(c.M) * pd + pd * std::log(pd) + double(c.n) * e1);
}

// Pass-+1 strengths of explicit pairs on the device (the complexity
// estimate, xyzb_pair_strengths, the drop-in's sample_strengths), one thread
// per pair in the reference's own evaluation order so every strength is
// bit-identical to the host's:
//   binary:        agree / n (interaction_strength, transforms.cpp:33-40);
//   continuous-Y:  sum of |y_i| over the set bits of x_j ^ x_k ^ s, words and
//                  bits ascending, / ||y||_1 (transforms.cpp:42-76);
//   continuous-XY: 0.5 + sum_i y_i t(x_ij) t(x_ik) / (2 ||y||_1), rows
//                  ascending, each product rounded left to right with no
//                  fused multiply-add (search.cpp:477-493 and :273-287, built
//                  without -march, i.e. no FMA contraction on the host).
template <class T>
__global__ void pair_strengths_exact(const u32* __restrict__ pairs, u64 cnt, int mode, int unbiased,
                                     const u64* __restrict__ Xc, u32 Wp, u32 W, const u64* __restrict__ yk,
                                     const u64* __restrict__ spos, const double* __restrict__ wabs,
                                     const T* __restrict__ Xr, u64 ld, const double* __restrict__ y, u32 n,
                                     double norm, double* __restrict__ out) {
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < cnt; t += u64(gridDim.x) * blockDim.x) {
        const u32 j = pairs[2 * t], k = pairs[2 * t + 1];
        if (mode == XYZB_MODE_BINARY) {
            const u64 *a = Xc + u64(j) * Wp, *b = Xc + u64(k) * Wp;
            u32 agree = 0;
            for (u32 w = 0; w < W; ++w) agree += __popcll(a[w] ^ b[w] ^ yk[w]);
            out[t] = double(agree) / double(n);
        } else if (mode == XYZB_MODE_CONTINUOUS_Y) {
            const u64 *a = Xc + u64(j) * Wp, *b = Xc + u64(k) * Wp;
            double acc = 0.0;
            for (u32 w = 0; w < W; ++w) {
                u64 m = a[w] ^ b[w] ^ spos[w];
                while (m) {
                    const int bit = __ffsll(static_cast<long long>(m)) - 1;
                    acc = __dadd_rn(acc, wabs[u64(w) * 64 + bit]);
                    m &= m - 1;
                }
            }
            out[t] = acc / norm;
        } else {
            const T *a = Xr + u64(j) * ld, *b = Xr + u64(k) * ld;
            double acc = 0.0;
            for (u32 i = 0; i < n; ++i) {
                const double u = double(a[i]), v = double(b[i]);
                if (unbiased) {
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(y[i], u), v));
                } else {
                    const double tu = u > 0.0 ? 1.0 : (u < 0.0 ? -1.0 : 0.0);
                    const double tv = v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0);
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(y[i], tu), tv));
                }
            }
            out[t] = __dadd_rn(0.5, acc / (2.0 * norm));
        }
    }
}

// agree(z_j, x_k) of two binary datasets (count_agreements, packed_matrix.cpp:37-47)
__global__ void pair_agreements_kernel(const u32* __restrict__ pairs, u64 cnt, const u64* __restrict__ Z, u32 Wz,
                                       const u64* __restrict__ X, u32 Wx, u32 W, u64 n, u64* __restrict__ out) {
    for (u64 t = u64(blockIdx.x) * blockDim.x + threadIdx.x; t < cnt; t += u64(gridDim.x) * blockDim.x) {
        const u64 *a = Z + u64(pairs[2 * t]) * Wz, *b = X + u64(pairs[2 * t + 1]) * Wx;
        u64 dis = 0;
        for (u32 w = 0; w < W; ++w) dis += __popcll(a[w] ^ b[w]);
        out[t] = n - dis;
    }
}

void device_pair_strengths(SearchCtx& c, const u32* pairs, u64 cnt, double* out) {
    xyzb_dataset* ds = c.ds;
    cudaStream_t st = ds->stream;
    if (cnt == 0) return;
    for (u64 t = 0; t < cnt; ++t)
        if (pairs[2 * t] >= c.p || pairs[2 * t + 1] >= c.p) throw data_error("interaction_strength: index out of range");
    ds->pairs_dev.ensure(cnt * 8);
    ds->strengths_dev.ensure(cnt * 8);
    XYZB_CUDA(cudaMemcpyAsync(ds->pairs_dev.p, pairs, cnt * 8, cudaMemcpyHostToDevice, st));
    const u32 grid = grid_for(cnt, 128, kSMs * 32);
    const int unb = c.q->transform == XYZB_TRANSFORM_UNBIASED;
    if (ds->binary || ds->f32_src)
        pair_strengths_exact<float><<<grid, 128, 0, st>>>(
            ds->pairs_dev.as<u32>(), cnt, c.mode, unb, ds->Xc.as<u64>(), static_cast<u32>(ds->Wp),
            static_cast<u32>(ds->W), ds->yk_bits.as<u64>(), ds->spos.as<u64>(), ds->wabs.as<double>(),
            ds->Xc32.as<float>(), ds->n4, ds->yreal.as<double>(), static_cast<u32>(c.n), c.norm,
            ds->strengths_dev.as<double>());
    else  // the caller's fp64 values
        pair_strengths_exact<double><<<grid, 128, 0, st>>>(
            ds->pairs_dev.as<u32>(), cnt, c.mode, unb, ds->Xc.as<u64>(), static_cast<u32>(ds->Wp),
            static_cast<u32>(ds->W), ds->yk_bits.as<u64>(), ds->spos.as<u64>(), ds->wabs.as<double>(),
            ds->Xsrc64.as<double>(), ds->n, ds->yreal.as<double>(), static_cast<u32>(c.n), c.norm,
            ds->strengths_dev.as<double>());
    XYZB_LAUNCH_CHECK();
    c.launches[XYZB_STAGE_ESTIMATE] += 1;
    XYZB_CUDA(cudaMemcpyAsync(out, ds->strengths_dev.p, cnt * 8, cudaMemcpyDeviceToHost, st));
    XYZB_CUDA(cudaStreamSynchronize(st));
}

void check_mode(const xyzb_dataset* ds, const xyzb_params* q, const xyzb_response* resp, bool unit_check = true) {
    if (q->mode == XYZB_MODE_BINARY) {
        if (!ds->binary) throw data_error("xyz_search: real X requires continuous-XY mode");
        if (!resp || !resp->y_sign) throw data_error("xyz_search: packed X with sign Y requires binary mode");
    } else if (q->mode == XYZB_MODE_CONTINUOUS_Y) {
        if (!ds->binary) throw data_error("xyz_search: real X requires continuous-XY mode");
        if (!resp || !resp->y_real) throw data_error("xyz_search: packed X with real Y requires continuous-Y mode");
    } else {
        if (ds->binary) throw data_error("xyz_search: packed X with real Y requires continuous-Y mode");
        if (!resp || !resp->y_real) throw data_error("xyz_search: real X requires continuous-XY mode");
        if (unit_check && q->transform == XYZB_TRANSFORM_UNBIASED && !ds->in_unit)
            throw data_error(
                "xyz_search: unbiased transform needs entries in [-1,1]; apply rescale_rows or cap_entries first");
    }
}

// The binned verify (binned_verify.cuh) sizes its z windows to stay resident
// in L2 and keeps one CTA per SM: two such searches interleaving on a device
// evict each other's windows. They take the device in turn (uploads, dataset
// creation and every other search still overlap them).
bool binned_eligible(const xyzb_dataset* ds, const xyzb_params* q) {
    const long long bsel = topt().binned.load();
    if (bsel < 0 || q->mode != XYZB_MODE_BINARY || !ds->binary || ds->Wp / 2 > 80 || ds->p > (u64(1) << 20))
        return false;
    return bsel == 1 || ds->p * ds->Wp * 8 >= (u64(512) << 20);
}
std::mutex& device_search_mutex(int dev) {
    static std::mutex mu[64];
    return mu[dev & 63];
}

void do_search(xyzb_dataset* ds, const xyzb_response* resp, const xyzb_params* q, const uint32_t* draws,
               xyzb_result* out) {
    Nvtx nv("xyzb_search");
    const auto t0 = std::chrono::steady_clock::now();
    validate_params(q);
    std::unique_lock<std::mutex> turn;  // taken just before the first kernel, released once the results are home
    DeviceGuard dg(ds->device);
    StreamScope ss(ds->stream);
    Trace tr(ds->stream, false);
    check_mode(ds, q, resp);
    SearchCtx c;
    c.ds = ds;
    c.q = q;
    c.mode = q->mode;
    c.n = ds->n;
    c.p = ds->p;
    c.M = q->m;
    c.gamma = q->gamma;
    c.guard = q->max_candidates_per_rep ? q->max_candidates_per_rep : 16 * ds->p;  // search.cpp:303-304
    c.out = out;
    if (ds->p > 0x7fffffffull) throw data_error("xyzb: more than 2^31-1 columns");
    if (c.mode == XYZB_MODE_BINARY) c.astar = integer_threshold(c.n, c.gamma);
    if (q->stop_after_first_hit && (q->rep_begin || q->rep_end))
        throw data_error("xyzb: stop_after_first_hit cannot be combined with a rep shard");
    if (q->top_k_mode != XYZB_TOPK_HITS && q->top_k_mode != XYZB_TOPK_CANDIDATES)
        throw data_error("xyzb: unknown top_k_mode");
    c.topk_all = q->top_k_mode == XYZB_TOPK_CANDIDATES;
    if (c.topk_all) c.astar = 0;  // every candidate is ranked; the running threshold gates the appends
    if (c.topk_all && q->top_k == 0) throw data_error("xyzb: top-K over all candidates needs top_k >= 1");
    if (c.topk_all && q->stop_after_first_hit)
        throw data_error("xyzb: top-K over all candidates cannot be combined with stop_after_first_hit");
    if (c.topk_all && q->top_k > 0x7fffffffull) throw data_error("xyzb: top_k too large");
    std::memset(out, 0, sizeof(*out));
    ds->clock.st = ds->stream;
    ds->clock.reset();
    cudaEvent_t ev_start = ds->clock.mark();
    upload_response(c, resp);
    if (c.mode == XYZB_MODE_CONTINUOUS_XY && q->transform == XYZB_TRANSFORM_UNBIASED) ensure_xr64(ds);
    tr.mark("search:y");
    plan_runs(c, draws);
    tr.mark("search:plan");
    cudaEvent_t ev_draw = ds->clock.mark();
    ds->clock.span(XYZB_STAGE_OTHER, ev_start, ev_draw);
    u32 H = 0;
    const size_t spans0 = ds->clock.spans.size();
    const u64 Rall = c.plan.sign_by_rid.size();
    std::vector<u64> enumerated(Rall), verified(Rall);
    // the single-CTA merge is queued right behind the search (hit count read on
    // the device); one host round trip then returns every counter at once
    const bool fused_merge = !q->stop_after_first_hit && !topt().merge_large.load();
    u32 fusedK = 0xffffffffu, fusedKK = 0;
    u32 fcap = 0;
    cudaEvent_t ev_dev_end = nullptr;  // end of the device work (results resident in HBM)
    if (binned_eligible(ds, q)) turn = std::unique_lock<std::mutex>(device_search_mutex(ds->device));
    for (int attempt = 0; attempt < 8; ++attempt) {
        ds->clock.spans.resize(spans0);
        c.attempts += 1;
        if (c.M <= 31) run_batches<u32>(c); else run_batches<u64>(c);  // u32 holds M bits + the side bit
        const u64 nbt = c.nbatches;
        u32* top_counts = nullptr;
        if (fused_merge) {
            fcap = std::min<u32>(ds->hit_cap, u32(merge::kSmallMerge));
            const size_t smem = merge::small_merge_smem(merge::kSmallMerge);
            func_smem(merge::merge_small, smem);
            ds->fin.ensure(u64(fcap) * sizeof(xyzb_hit));
            ds->fin_order.ensure(u64(fcap) * 8);
            ds->topidx.ensure(u64(fcap) * 8 + 16);
            top_counts = reinterpret_cast<u32*>(ds->topidx.as<u64>() + fcap);
            cudaEvent_t m0 = ds->clock.mark();
            merge::merge_small<<<1, merge::kSmallThreads, smem, ds->stream>>>(
                ds->hits.as<kern::DevHit>(), 0, ds->sign_by_rid.as<int8_t>(), 0xffffffffu, c.plan.L, q->top_k,
                ds->fin.as<xyzb_hit>(), ds->fin_order.as<u64>(), ds->topidx.as<u64>(), top_counts,
                ds->hit_count.as<u32>(), fcap);
            XYZB_LAUNCH_CHECK();
            cudaEvent_t m1 = ds->clock.mark();
            ds->clock.span(XYZB_STAGE_MERGE, m0, m1);
            ev_dev_end = m1;
        }
        // status block (pinned): H, merge counts, items and pairs per batch, per-run counters
        const size_t o_cnt = 8, o_items = 16, o_pairs = o_items + 4 * nbt, o_enum = round_up(o_pairs + 4 * nbt, 8),
                     o_ver = o_enum + 8 * Rall, o_ovf = o_ver + 8 * Rall, o_tk = o_ovf + 8,
                     o_bin = round_up(o_tk + sizeof(topk::State), 8), sbytes = o_bin + 8;
        ds->h_status.ensure(sbytes);
        char* hs = ds->h_status.as<char>();
        small_copy(hs, ds->hit_count.p, 4, ds->stream);
        if (top_counts) small_copy(hs + o_cnt, top_counts, 8, ds->stream);
        small_copy(hs + o_items, ds->nblocks.p, nbt * 4, ds->stream);
        if (c.pair_cap)
            small_copy(hs + o_pairs, ds->npairs.p, nbt * 4, ds->stream);
        small_copy(hs + o_enum, ds->enumerated.p, Rall * 8, ds->stream);
        small_copy(hs + o_ver, ds->verified.p, Rall * 8, ds->stream);
        small_copy(hs + o_ovf, ds->povf.p, 8, ds->stream);
        if (c.topk_all)
            small_copy(hs + o_tk, ds->tk_state.p, sizeof(topk::State), ds->stream);
        if (c.binned)
            small_copy(hs + o_bin, ds->bin_ovfn.p, 4, ds->stream);
        tr.mark("search:launch");
        XYZB_CUDA(cudaStreamSynchronize(ds->stream));
        tr.mark("search:device");
        H = *reinterpret_cast<const u32*>(hs);
        if (top_counts) {
            fusedK = reinterpret_cast<const u32*>(hs + o_cnt)[0];
            fusedKK = reinterpret_cast<const u32*>(hs + o_cnt)[1];
        }
        const u32* nitems = reinterpret_cast<const u32*>(hs + o_items);
        const u64 need = nbt ? *std::max_element(nitems, nitems + nbt) : 0;
        u64 pneed = 0;
        if (c.pair_cap) {
            const u32* np = reinterpret_cast<const u32*>(hs + o_pairs);
            pneed = *std::max_element(np, np + nbt);
            if (pneed > c.pair_cap) {
                c.no_one_pass = true;  // an aborted run's pairs (a one-pass join) may be what overflowed
                if (c.pair_cap == 0xffffffffull) throw internal_error("xyzb: candidate pairs exceed 2^32 in one batch");
                c.pair_scale *= std::max<u64>(2, ceil_div(pneed, c.pair_cap));
            }
        }
        bool bin_redo = false;
        if (c.binned) {  // bins sized from this search's mean fill next time; an overflowing list: redo
            const u32 on = *reinterpret_cast<const u32*>(hs + o_bin);
            if (c.pair_cap) {
                const u32* np = reinterpret_cast<const u32*>(hs + o_pairs);
                u64 tot = 0;
                for (u64 b = 0; b < nbt; ++b) tot += std::min<u64>(np[b], c.pair_cap);
                ds->bin_hint = std::max<u64>(1, tot / (u64(c.nkt) * c.nbh));
            }
            if (on > c.ovf_cap) {
                ds->bin_ovf_hint = 2 * u64(on);
                bin_redo = true;
            }
        }
        const bool povf = *reinterpret_cast<const u32*>(hs + o_ovf) != 0;
        if (povf) c.no_hash = true;  // a hashed partition overflowed: redo on the sorted path
        const bool fovf = reinterpret_cast<const u32*>(hs + o_ovf)[1] != 0;
        if (fovf) {  // a fixed-capacity partition overflowed: count the partitions
            c.no_fixed_part = true;
            ds->part_fixed_fails += 1;
        }
        bool tk_redo = false;
        if (c.topk_all) {
            topk::State ts;
            std::memcpy(&ts, hs + o_tk, sizeof(ts));
            if (ts.fail & 2u) {  // the hit buffer overflowed during a batch
                H = std::max(H, ts.max_hits);
                tk_redo = true;
            }
            if (ts.fail & 4u) {  // binned: a window after the first ran with the threshold still at 0
                c.tk_all_windows = true;
                tk_redo = true;
            }
            if (ts.fail & 1u) {  // a batch's dropped band could hold top-K keys: emit more
                c.tk_level = std::min(c.tk_level + 1, 2);
                tk_redo = true;
            }
        }
        if (!povf && !fovf && !tk_redo && !bin_redo && H <= ds->hit_cap && need <= c.item_cap && pneed <= c.pair_cap) {
            std::memcpy(enumerated.data(), hs + o_enum, Rall * 8);
            std::memcpy(verified.data(), hs + o_ver, Rall * 8);
            if (c.pair_cap) {  // the pair list (16 B per canonical pair) is written by the join
                const u32* np = reinterpret_cast<const u32*>(hs + o_pairs);
                u64 tot = 0;
                for (u64 b = 0; b < nbt; ++b) tot += np[b];
                c.bytes[c.pairs_in_sort ? XYZB_STAGE_SORT : XYZB_STAGE_JOIN] += 16 * tot;
                // binned: level 1 reads 16 B and writes 8 B per pair, level 2 reads 8 B three times and writes 8 B
                // binned: the window pass reads the z column and the record and writes 8 B; the bucket and tile
                // splits each read 8 B twice and write 8 B
                if (c.binned) c.bytes[XYZB_STAGE_JOIN] += 72 * tot;
                if (c.topk_all) c.bytes[XYZB_STAGE_MERGE] += 8 * tot;  // pair ranks read by the histogram + emission
            }
            break;
        }
        // a buffer overflowed (the counters kept counting): grow and recompute
        if (H > ds->hit_cap) ds->hit_cap = static_cast<u32>(std::min<u64>(0xffffffffull, u64(H) * 2));
        if (need > c.item_cap) {
            if (c.item_cap == 0xffffffffull) throw internal_error("xyzb: work items exceed 2^32 in one batch");
            c.item_scale *= std::max<u64>(2, ceil_div(need, c.item_cap));
        }

        std::memset(c.launches, 0, sizeof(c.launches));
        std::memset(c.bytes, 0, sizeof(c.bytes));
        c.pairs_in_sort = false;
        c.verify_spans.clear();
        if (attempt == 7) throw internal_error("xyzb: hit buffer did not converge");
        if (c.topk_all && H > ds->hit_cap / 2)  // keep the top-K buffer's headroom
            ds->hit_cap = static_cast<u32>(std::min<u64>(0xffffffffull, u64(H) * 2));
    }
    u32 rmax = 0xffffffffu;
    std::vector<xyzb_hit> hits;
    std::vector<u64> order, topk;
    if (fused_merge && H <= fcap && fusedK != 0xffffffffu) {
        c.launches[XYZB_STAGE_MERGE] += 1;
        hits.resize(fusedK);
        order.resize(fusedK);
        topk.resize(fusedKK);
        if (fusedK) {
            const size_t hb = u64(fusedK) * sizeof(xyzb_hit), ob = u64(fusedK) * 8, tb = u64(fusedKK) * 8;
            ds->h_merge.ensure(hb + ob + tb + 8);
            char* hp = ds->h_merge.as<char>();
            small_copy(hp, ds->fin.p, hb, ds->stream);
            small_copy(hp + hb, ds->fin_order.p, ob, ds->stream);
            if (tb) small_copy(hp + hb + ob, ds->topidx.p, tb, ds->stream);
            XYZB_CUDA(cudaStreamSynchronize(ds->stream));
            std::memcpy(hits.data(), hp, hb);
            std::memcpy(order.data(), hp + hb, ob);
            if (tb) std::memcpy(topk.data(), hp + hb + ob, tb);
        }
    } else {
        if (q->stop_after_first_hit && H > 0) {
            ds->rmin.ensure(8);
            XYZB_CUDA(cudaMemsetAsync(ds->rmin.p, 0xff, 4, ds->stream));
            merge::min_rid<<<grid_for(H, 256), 256, 0, ds->stream>>>(ds->hits.as<kern::DevHit>(), H,
                                                                     ds->rmin.as<u32>());
            XYZB_LAUNCH_CHECK();
            XYZB_CUDA(cudaMemcpyAsync(&rmax, ds->rmin.p, 4, cudaMemcpyDeviceToHost, ds->stream));
        }
        // drop the fused merge's span (it only flagged the overflow)
        for (auto it = ds->clock.spans.begin(); it != ds->clock.spans.end();)
            it = it->first == XYZB_STAGE_MERGE ? ds->clock.spans.erase(it) : it + 1;
        cudaEvent_t ev_m0 = ds->clock.mark();
        XYZB_CUDA(cudaStreamSynchronize(ds->stream));
        merge_hits(c, H, rmax, hits, order, topk);
        cudaEvent_t ev_m1 = ds->clock.mark();
        ds->clock.span(XYZB_STAGE_MERGE, ev_m0, ev_m1);
        ev_dev_end = ev_m1;
    }
    if (turn.owns_lock()) turn.unlock();
    out->gamma_effective = c.gamma;
    if (c.topk_all) out->gamma_effective = topk_filter(hits, order, topk);
    out->devices_used = 1;
    out->attempts = c.attempts;
    // counters over executed runs (in pass/rep order)
    u64 reps = 0, enumc = 0, aborted = 0, ver = 0;
    for (u32 r : c.plan.rid) {
        if (r > rmax) continue;
        ++reps;
        enumc += enumerated[r];
        if (enumerated[r] > c.guard) ++aborted;
        ver += verified[r];
    }
    out->repetitions_run = reps;
    out->runs_executed = c.plan.rid.size();
    out->candidates_enumerated = enumc;
    out->aborted_repetitions = aborted;
    out->verified_pairs = ver;
    out->candidates_checked = ver;
    out->gamma0 = std::pow(double(c.p), -1.0 / double(c.M));
    out->m_used = c.M;
    out->l_used = q->l;
    if (q->estimate_complexity) {
        cudaEvent_t e0 = ds->clock.mark();
        out->estimated_c = estimate_complexity(c, [&](const u32* pr, u64 cnt, double* s) {
            device_pair_strengths(c, pr, cnt, s);
        });
        cudaEvent_t e1 = ds->clock.mark();
        ds->clock.span(XYZB_STAGE_ESTIMATE, e0, e1);
    }
    tr.mark("search:results");
    cudaEvent_t ev_end = ds->clock.mark();
    XYZB_CUDA(cudaEventSynchronize(ev_end));
    // device time: search start to the end of the merge (hits resident in HBM;
    // their copy to the host belongs to the end-to-end time), plus the
    // complexity estimate when it ran
    float ms = 0.f;
    XYZB_CUDA(cudaEventElapsedTime(&ms, ev_start, ev_dev_end ? ev_dev_end : ev_end));
    out->device_ms = ms;
    for (auto& sp : ds->clock.spans) {
        float m2 = 0.f;
        XYZB_CUDA(cudaEventElapsedTime(&m2, sp.second.first, sp.second.second));
        out->stage_ms[sp.first] += m2;
    }
    if (ev_dev_end) out->device_ms += out->stage_ms[XYZB_STAGE_ESTIMATE];
    for (auto& sp : c.verify_spans) {
        float m2 = 0.f;
        XYZB_CUDA(cudaEventElapsedTime(&m2, sp.first, sp.second));
        out->verify_kernel_ms += m2;
    }
    out->verify_launches = c.verify_spans.size();
    // algorithmic verify bytes: 2 columns per canonical pair + Y (the sign transform's bit-plane verify:
    // 2 sign-bit columns (+ 2 nonzero masks when X has zeros) per pair + the response's bit planes)
    const u64 wb = 8 * ceil_div(c.n, 64);
    if (c.sign_verify)
        c.bytes[XYZB_STAGE_VERIFY] = ver * 2 * wb * (ds->has_zero ? 2 : 1) + u64(c.qB + 1) * wb;
    else {
        const u64 colbytes = c.mode == XYZB_MODE_CONTINUOUS_XY ? 4 * c.n : wb;
        c.bytes[XYZB_STAGE_VERIFY] = ver * 2 * colbytes + colbytes;
    }
    u64 tl = 0;
    for (int s = 0; s < XYZB_NUM_STAGES; ++s) {
        out->stage_bytes[s] = c.bytes[s];
        out->stage_launches[s] = c.launches[s];
        tl += c.launches[s];
    }
    out->kernel_launches = tl;
    // report arrays (malloc-owned, xyzb_result_free)
    out->n_hits = hits.size();
    out->hits = static_cast<xyzb_hit*>(std::malloc(std::max<size_t>(1, hits.size()) * sizeof(xyzb_hit)));
    out->order_keys = static_cast<u64*>(std::malloc(std::max<size_t>(1, order.size()) * 8));
    if (!hits.empty()) {
        std::memcpy(out->hits, hits.data(), hits.size() * sizeof(xyzb_hit));
        std::memcpy(out->order_keys, order.data(), order.size() * 8);
    }
    out->n_top_k = topk.size();
    out->top_k = static_cast<u64*>(std::malloc(std::max<size_t>(1, topk.size()) * 8));
    if (!topk.empty()) std::memcpy(out->top_k, topk.data(), topk.size() * 8);
    out->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}


// ---- generic equal-key join (equal_pairs, pair_search.cpp:26-55) ----

struct EpBlock {
    u32 xs, xc, zs, zc;
};

__global__ void ep_blocks(const u64* __restrict__ sx, const u64* __restrict__ sz, u64 p, EpBlock* __restrict__ blk,
                          u64* __restrict__ work) {
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const u64 v = sx[i];
    u64 w = 0;
    EpBlock b{u32(i), 0, 0, 0};
    if (i == 0 || sx[i - 1] != v) {
        const u64 e = kern::run_end(sx, i, p, v);
        const u64 lo = kern::lower_bound(sz, 0, p, v);
        if (lo < p && sz[lo] == v) {
            const u64 hi = kern::run_end(sz, lo, p, v);
            b = {u32(i), u32(e - i), u32(lo), u32(hi - lo)};
            w = (e - i) * (hi - lo);
        }
    }
    blk[i] = b;
    work[i] = w;
}

__global__ void ep_emit(const EpBlock* __restrict__ blk, const u64* __restrict__ off, const u32* __restrict__ vx,
                        const u32* __restrict__ vz, u64 p, u32* __restrict__ out) {
    const u64 i = u64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= p) return;
    const EpBlock b = blk[i];
    if (b.xc == 0) return;
    u64 o = off[i];
    for (u32 a = 0; a < b.xc; ++a)
        for (u32 c = 0; c < b.zc; ++c, ++o) {
            out[2 * o] = vx[b.xs + a];
            out[2 * o + 1] = vz[b.zs + c];
        }
}

} // namespace

extern "C" int xyzb_equal_pairs(const uint64_t* x_keys, const uint64_t* z_keys, uint64_t p, int32_t device,
                                uint32_t** pairs_jk, uint64_t* n_pairs, uint64_t* total_pairs, char* err,
                                size_t errlen) {
    return guarded(err, errlen, [&] {
        *pairs_jk = nullptr;
        *n_pairs = 0;
        *total_pairs = 0;
        require_device();
        DeviceGuard dg(device);
        if (p == 0) {
            *pairs_jk = static_cast<uint32_t*>(std::malloc(8));
            return;
        }
        if (p > 0xffffffffull) throw data_error("equal_pairs: too many keys");
        cudaStream_t st;
        XYZB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        struct S { cudaStream_t s; ~S() { cudaStreamDestroy(s); } } sguard{st};
        StreamScope ss(st);
        DevBuf kb0, kb1, vb0, vb1, hist, blk, work, off, part, cnt, outp;
        kb0.ensure(2 * p * 8);
        kb1.ensure(2 * p * 8);
        vb0.ensure(2 * p * 4);
        vb1.ensure(2 * p * 4);
        u64 maxk = 0;
        for (u64 i = 0; i < p; ++i) maxk = std::max(maxk, std::max(x_keys[i], z_keys[i]));
        int bits = 1;
        while (bits < 64 && (maxk >> bits)) ++bits;
        XYZB_CUDA(cudaMemcpyAsync(kb0.p, x_keys, p * 8, cudaMemcpyHostToDevice, st));
        XYZB_CUDA(cudaMemcpyAsync(kb0.as<u64>() + p, z_keys, p * 8, cudaMemcpyHostToDevice, st));
        hist.ensure(rsort::hist_words(2, p) * 4);
        u64* kb[2] = {kb0.as<u64>(), kb1.as<u64>()};
        u32* vb[2] = {vb0.as<u32>(), vb1.as<u32>()};
        const int r = rsort::sort_segments<u64>(kb, vb, 2, p, bits, hist.as<u32>(), st);
        blk.ensure(p * sizeof(EpBlock));
        work.ensure(p * 8);
        off.ensure((p + 1) * 8);
        part.ensure(scan::kGrid * 8);
        cnt.ensure(8);
        const u32 pc = static_cast<u32>(p);
        XYZB_CUDA(cudaMemcpyAsync(cnt.p, &pc, 4, cudaMemcpyHostToDevice, st));
        ep_blocks<<<static_cast<u32>(ceil_div(p, 256)), 256, 0, st>>>(kb[r], kb[r] + p, p, blk.as<EpBlock>(),
                                                                      work.as<u64>());
        XYZB_LAUNCH_CHECK();
        scan::exclusive<u64>(work.as<u64>(), cnt.as<u32>(), off.as<u64>(), part.as<u64>(), st);
        u64 total = 0;
        XYZB_CUDA(cudaMemcpyAsync(&total, off.as<u64>() + p, 8, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        outp.ensure(std::max<u64>(1, total) * 8);
        ep_emit<<<static_cast<u32>(ceil_div(p, 256)), 256, 0, st>>>(blk.as<EpBlock>(), off.as<u64>(), vb[r],
                                                                    vb[r] + p, p, outp.as<u32>());
        XYZB_LAUNCH_CHECK();
        uint32_t* host = static_cast<uint32_t*>(std::malloc(std::max<u64>(1, total) * 8));
        XYZB_CUDA(cudaMemcpyAsync(host, outp.p, total * 8, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        *pairs_jk = host;
        *n_pairs = total;
        *total_pairs = total;
    });
}

extern "C" int xyzb_project_keys(xyzb_dataset* ds, const uint32_t* draws, uint64_t n_draws, uint64_t m,
                                 uint64_t* keys, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!ds || !ds->binary) throw data_error("project_keys: needs a binary dataset");
        if (m == 0 || m > 64) throw data_error("project_keys: draw size outside [1,64]");
        for (u64 t = 0; t < n_draws * m; ++t)
            if (draws[t] >= ds->n) throw data_error("project_keys: draw index out of range");
        if (n_draws == 0) return;
        DeviceGuard dg(ds->device);
        cudaStream_t st = ds->stream;
        StreamScope ss(st);
        DevBuf rows, kout, xc, sg, yk;
        rows.ensure(n_draws * m * 4);
        kout.ensure(n_draws * ds->p * 8);
        xc.ensure(n_draws * 8);
        sg.ensure(n_draws);
        yk.ensure(ds->Wp * 8);
        XYZB_CUDA(cudaMemsetAsync(yk.p, 0, ds->Wp * 8, st));
        XYZB_CUDA(cudaMemsetAsync(sg.p, 1, n_draws, st));
        XYZB_CUDA(cudaMemcpyAsync(rows.p, draws, n_draws * m * 4, cudaMemcpyHostToDevice, st));
        dim3 g(static_cast<u32>(ceil_div(ds->P32, 128)), static_cast<u32>(n_draws));
        kern::project_bits_t<u64><<<g, 128, 0, st>>>(ds->Xr.as<u32>(), ds->P32, ds->p, rows.as<u32>(), int(m),
                                                     kout.as<u64>());
        XYZB_LAUNCH_CHECK();
        XYZB_CUDA(cudaMemcpyAsync(keys, kout.p, n_draws * ds->p * 8, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
    });
}

extern "C" int xyzb_pair_agreements(xyzb_dataset* z, xyzb_dataset* x, const uint32_t* pairs_jk, uint64_t n_pairs,
                                    uint64_t* agree, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!z || !x || (n_pairs && (!pairs_jk || !agree))) throw data_error("xyzb_pair_agreements: null argument");
        if (!z->binary || !x->binary) throw data_error("xyzb_pair_agreements: needs binary datasets");
        if (z->n != x->n) throw data_error("interaction_strength: row count mismatch");
        if (z->device != x->device) throw data_error("xyzb_pair_agreements: datasets on different devices");
        for (u64 t = 0; t < n_pairs; ++t) {
            if (pairs_jk[2 * t] >= z->p) throw data_error("interaction_strength: index j out of range");
            if (pairs_jk[2 * t + 1] >= x->p) throw data_error("interaction_strength: index k out of range");
        }
        if (n_pairs == 0) return;
        DeviceGuard dg(x->device);
        StreamScope ss(x->stream);
        const cudaStream_t st = x->stream;
        XYZB_CUDA(cudaStreamSynchronize(z->stream));  // z's upload is complete
        DevBuf pd, od;
        pd.ensure(n_pairs * 8);
        od.ensure(n_pairs * 8);
        XYZB_CUDA(cudaMemcpyAsync(pd.p, pairs_jk, n_pairs * 8, cudaMemcpyHostToDevice, st));
        pair_agreements_kernel<<<grid_for(n_pairs, 128, kSMs * 32), 128, 0, st>>>(
            pd.as<u32>(), n_pairs, z->Xc.as<u64>(), static_cast<u32>(z->Wp), x->Xc.as<u64>(),
            static_cast<u32>(x->Wp), static_cast<u32>(x->W), x->n, od.as<u64>());
        XYZB_LAUNCH_CHECK();
        XYZB_CUDA(cudaMemcpyAsync(agree, od.p, n_pairs * 8, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
    });
}

extern "C" int xyzb_pair_strengths(xyzb_dataset* ds, const xyzb_response* resp, const xyzb_params* params,
                                   const uint32_t* pairs_jk, uint64_t n_pairs, double* strengths, char* err,
                                   size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!ds || !params) throw data_error("pair_strengths: null argument");
        DeviceGuard dg(ds->device);
        StreamScope ss(ds->stream);
        check_mode(ds, params, resp, false);  // strengths only: the transform's [-1, 1] domain is the search's
        SearchCtx c;
        c.ds = ds;
        c.q = params;
        c.mode = params->mode;
        c.n = ds->n;
        c.p = ds->p;
        c.M = params->m;
        c.gamma = params->gamma;
        upload_response(c, resp);
        device_pair_strengths(c, pairs_jk, n_pairs, strengths);
    });
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        XYZB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) throw cuda_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    return fn;
}

// 2-D K-major int8 operand [rows][Kp], boxes of 128 bytes x box_rows, 128-byte swizzle.
CUtensorMap operand_map(void* base, u64 rows, u64 Kp, u32 box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {Kp, rows};
    const cuuint64_t strides[1] = {Kp};
    const cuuint32_t box[2] = {128u, box_rows};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = encode_tiled()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw cuda_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return m;
}

namespace {
namespace brutew {

// The exhaustive oracle's continuous-response overload (oracle.cpp:93-100,
// scalar_weighted_strength): the weighted strength of every pair j < k,
// rows in order and fp64 adds (bit-identical to the host's loop), 16 x 16
// pair tiles of the upper triangle walked by persistent CTAs. PASS 0: the
// caller's histogram (shared per CTA when it fits) and, for top-K, a 2^20-bin
// histogram of the kept strengths (the host derives the top-K cutoff from
// it); PASS 1: the kept pairs at or above the cut, appended.
constexpr int kTile = 16;
constexpr int kFineBits = 20;
constexpr u32 kSmemBins = 8192;

struct Out {
    u32 j, k;
    double s;
};

__device__ __forceinline__ u32 fine_bin(double s) {
    const double x = s * double(1u << kFineBits);
    return x <= 0.0 ? 0u : (x >= double(1u << kFineBits) ? (1u << kFineBits) : u32(x));
}

template <int PASS>
__global__ void __launch_bounds__(kTile * kTile) weighted_pairs(
    const u64* __restrict__ Xc, u32 Wp, u32 W, u32 p, const u64* __restrict__ sb, const double* __restrict__ wabs,
    double norm, u32 bins, unsigned long long* __restrict__ uhist, int has_gamma, double gamma, int fine,
    unsigned int* __restrict__ fhist, unsigned long long* __restrict__ kept, double cut, Out* __restrict__ out,
    u32* __restrict__ nout, u32 cap) {
    extern __shared__ u32 sh[];
    const bool shist = PASS == 0 && bins > 0 && bins <= kSmemBins;
    if (shist) {
        for (u32 b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0;
        __syncthreads();
    }
    const u64 T = (u64(p) + kTile - 1) / kTile;
    const u64 ntiles = T * (T + 1) / 2;
    u64 mykept = 0;
    for (u64 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // tile -> (tj, tk), tj <= tk: row tj starts at tj*T - tj*(tj-1)/2
        u64 tj = u64((2.0 * double(T) + 1.0 - sqrt((2.0 * double(T) + 1.0) * (2.0 * double(T) + 1.0) - 8.0 * double(tile))) / 2.0);
        while (tj > 0 && tj * T - tj * (tj - 1) / 2 > tile) --tj;
        while ((tj + 1) * T - (tj + 1) * tj / 2 <= tile) ++tj;
        const u64 tk = tj + (tile - (tj * T - tj * (tj - 1) / 2));
        const u32 j = u32(tj * kTile + threadIdx.x / kTile), k = u32(tk * kTile + threadIdx.x % kTile);
        const bool valid = j < k && k < p;
        double s = -1.0;
        if (valid) {
            const u64 *a = Xc + u64(j) * Wp, *b = Xc + u64(k) * Wp;
            double acc = 0.0;
            for (u32 w = 0; w < W; ++w) {
                u64 m = a[w] ^ b[w] ^ sb[w];
                while (m) {
                    const int bit = __ffsll(static_cast<long long>(m)) - 1;
                    acc = __dadd_rn(acc, wabs[u64(w) * 64 + bit]);
                    m &= m - 1;
                }
            }
            s = acc / norm;
        }
        const bool keep = valid && (!has_gamma || s >= gamma);
        if (PASS == 0) {
            if (valid && bins) {
                u64 bin = u64(s * double(bins));
                if (bin >= bins) bin = bins - 1;
                if (shist) atomicAdd(sh + bin, 1u);
                else atomicAdd(uhist + bin, 1ull);
            }
            if (keep) {
                ++mykept;
                if (fine) atomicAdd(fhist + fine_bin(s), 1u);
            }
        } else if (keep && s >= cut) {
            const u32 slot = atomicAdd(nout, 1u);
            if (slot < cap) out[slot] = Out{j, k, s};
        }
    }
    if (PASS == 0) {
        if (mykept) atomicAdd(kept, static_cast<unsigned long long>(mykept));
        if (shist) {
            __syncthreads();
            for (u32 b = threadIdx.x; b < bins; b += blockDim.x)
                if (sh[b]) atomicAdd(uhist + b, static_cast<unsigned long long>(sh[b]));
        }
    }
}

} // namespace brutew
} // namespace

extern "C" int xyzb_brute_force_weighted(xyzb_dataset* ds, const double* y, int32_t has_gamma, double gamma,
                                         int32_t has_top_k, uint64_t top_k, uint64_t histogram_bins, int32_t force,
                                         xyzb_scored_pair** pairs, uint64_t* n_pairs, uint64_t* pairs_scanned,
                                         uint64_t** histogram, char* err, size_t errlen) {
    if (pairs) *pairs = nullptr;
    if (n_pairs) *n_pairs = 0;
    if (pairs_scanned) *pairs_scanned = 0;
    if (histogram) *histogram = nullptr;
    return guarded(err, errlen, [&] {
        if (!ds || !y || !pairs || !n_pairs || !pairs_scanned || !histogram)
            throw data_error("brute_force_search: null argument");
        if (!ds->binary) throw data_error("brute_force_search: the GPU brute force takes binary datasets");
        const u64 n = ds->n, p = ds->p, W = ds->W, Wp = ds->Wp;
        if (p > 20000 && !force)  // check_guard (oracle.cpp:16-22)
            throw guard_error("brute_force_search: p = " + std::to_string(p) +
                              " exceeds the 20000 guard; pass force to run anyway");
        if (p > 0xffffffffull) throw data_error("brute_force_search: matrix too large");
        double norm = 0.0;  // scalar_weighted_strength's norm, rows in order
        for (u64 i = 0; i < n; ++i) norm += std::abs(y[i]);
        if (p >= 2 && norm <= 0.0) throw data_error("scalar_weighted_strength: zero response vector");
        *pairs_scanned = p * (p - 1) / 2;
        u64* h = nullptr;
        if (histogram_bins > 0) {
            h = static_cast<u64*>(std::calloc(histogram_bins, 8));
            if (!h) throw internal_error("brute_force_search: out of host memory");
            *histogram = h;
        }
        if (p < 2) return;
        DeviceGuard dg(ds->device);
        const cudaStream_t st = ds->stream;
        StreamScope ss(st);
        std::vector<u64> hs(Wp + Wp * 64, 0ull);
        double* hw = reinterpret_cast<double*>(hs.data() + Wp);
        for (u64 i = 0; i < n; ++i) {
            if (y[i] > 0.0) hs[i >> 6] |= 1ull << (i & 63);
            hw[i] = std::abs(y[i]);
        }
        DevBuf yb, uh, fh, cnt, ob, no;
        yb.ensure(hs.size() * 8);
        XYZB_CUDA(cudaMemcpyAsync(yb.p, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice, st));
        const u64* sb = yb.as<u64>();
        const double* wabs = reinterpret_cast<const double*>(yb.as<u64>() + Wp);
        const bool fine = has_top_k != 0;
        const u64 nfine = (u64(1) << brutew::kFineBits) + 1;
        uh.ensure(std::max<u64>(1, histogram_bins) * 8);
        fh.ensure(fine ? nfine * 4 : 4);
        cnt.ensure(8);
        XYZB_CUDA(cudaMemsetAsync(uh.p, 0, std::max<u64>(1, histogram_bins) * 8, st));
        if (fine) XYZB_CUDA(cudaMemsetAsync(fh.p, 0, nfine * 4, st));
        XYZB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
        const u32 grid = kSMs * 8;
        const size_t shb = histogram_bins > 0 && histogram_bins <= brutew::kSmemBins ? histogram_bins * 4 : 0;
        brutew::weighted_pairs<0><<<grid, brutew::kTile * brutew::kTile, shb, st>>>(
            ds->Xc.as<u64>(), u32(Wp), u32(W), u32(p), sb, wabs, norm, u32(histogram_bins),
            uh.as<unsigned long long>(), has_gamma, gamma, fine ? 1 : 0, fh.as<unsigned int>(),
            cnt.as<unsigned long long>(), 0.0, nullptr, nullptr, 0u);
        XYZB_LAUNCH_CHECK();
        u64 kept = 0;
        std::vector<unsigned int> fhist(fine ? nfine : 0);
        if (histogram_bins) XYZB_CUDA(cudaMemcpyAsync(h, uh.p, histogram_bins * 8, cudaMemcpyDeviceToHost, st));
        if (fine) XYZB_CUDA(cudaMemcpyAsync(fhist.data(), fh.p, nfine * 4, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaMemcpyAsync(&kept, cnt.p, 8, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        if (!has_gamma && !has_top_k) return;
        // the emission cut: every kept pair (gamma), or the fine bin holding the K-th kept strength
        double cut = -1.0;
        u64 emit = kept;
        if (has_top_k) {
            const u64 want = std::min<u64>(top_k, kept);
            if (want == 0) return;
            u64 acc = 0, b = nfine;
            while (b-- > 0) {
                acc += fhist[b];
                if (acc >= want) break;
            }
            cut = double(b) / double(u64(1) << brutew::kFineBits);  // the bin's lower edge
            emit = acc;
        }
        if (emit > 0xffffffffull) throw internal_error("brute_force_search: more than 2^32 pairs above the cut");
        ob.ensure(std::max<u64>(1, emit) * sizeof(brutew::Out));
        no.ensure(4);
        XYZB_CUDA(cudaMemsetAsync(no.p, 0, 4, st));
        brutew::weighted_pairs<1><<<grid, brutew::kTile * brutew::kTile, 0, st>>>(
            ds->Xc.as<u64>(), u32(Wp), u32(W), u32(p), sb, wabs, norm, 0u, nullptr, has_gamma, gamma, 0, nullptr,
            nullptr, cut, ob.as<brutew::Out>(), no.as<u32>(), u32(emit));
        XYZB_LAUNCH_CHECK();
        std::vector<brutew::Out> got(emit);
        u32 nget = 0;
        if (emit) XYZB_CUDA(cudaMemcpyAsync(got.data(), ob.p, emit * sizeof(brutew::Out), cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaMemcpyAsync(&nget, no.p, 4, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        if (nget != emit) throw internal_error("brute_force_search: emitted pair count differs from the histogram");
        const auto by_jk = [](const brutew::Out& a, const brutew::Out& b) { return a.j != b.j ? a.j < b.j : a.k < b.k; };
        if (has_top_k) {  // scan_all_pairs (oracle.cpp:45-53): strength desc, (j, k) asc; the K best, then (j, k)
            std::sort(got.begin(), got.end(), [&](const brutew::Out& a, const brutew::Out& b) {
                if (a.s != b.s) return a.s > b.s;
                return by_jk(a, b);
            });
            got.resize(std::min<u64>(top_k, got.size()));
        }
        std::sort(got.begin(), got.end(), by_jk);
        auto* outp = static_cast<xyzb_scored_pair*>(std::malloc(std::max<size_t>(1, got.size()) * sizeof(xyzb_scored_pair)));
        if (!outp) throw internal_error("brute_force_search: out of host memory");
        for (size_t t = 0; t < got.size(); ++t) outp[t] = xyzb_scored_pair{got[t].j, got[t].k, got[t].s};
        *pairs = outp;
        *n_pairs = got.size();
    });
}

extern "C" int xyzb_brute_force(xyzb_dataset* ds, const int8_t* y_sign, int32_t has_gamma, double gamma,
                                int32_t has_top_k, uint64_t top_k, uint64_t histogram_bins, int32_t force,
                                xyzb_scored_pair** pairs, uint64_t* n_pairs, uint64_t* pairs_scanned,
                                uint64_t** histogram, char* err, size_t errlen) {
    if (pairs) *pairs = nullptr;
    if (n_pairs) *n_pairs = 0;
    if (pairs_scanned) *pairs_scanned = 0;
    if (histogram) *histogram = nullptr;
    return guarded(err, errlen, [&] {
        if (!ds || !y_sign || !pairs || !n_pairs || !pairs_scanned || !histogram)
            throw data_error("brute_force_search: null argument");
        if (!ds->binary) throw data_error("brute_force_search: the GPU brute force takes binary datasets");
        const u64 n = ds->n, p = ds->p, W = ds->W, Wp = ds->Wp;
        // check_guard (oracle.cpp:16-22)
        if (p > 20000 && !force)
            throw guard_error("brute_force_search: p = " + std::to_string(p) +
                              " exceeds the 20000 guard; pass force to run anyway");
        if (p > 0xffffffffull || n > 0xffffffffull) throw data_error("brute_force_search: matrix too large");
        DeviceGuard dg(ds->device);
        const cudaStream_t st = ds->stream;
        StreamScope ss(st);
        // Y bits (y > 0) and the rows that can agree (y != 0)
        std::vector<u64> hy(2 * Wp, 0ull);
        for (u64 i = 0; i < n; ++i) {
            if (y_sign[i] > 0) hy[i >> 6] |= 1ull << (i & 63);
            if (y_sign[i] == 1 || y_sign[i] == -1) hy[Wp + (i >> 6)] |= 1ull << (i & 63);
        }
        DevBuf yb, zc, hist;
        yb.ensure(2 * Wp * 8);
        XYZB_CUDA(cudaMemcpyAsync(yb.p, hy.data(), 2 * Wp * 8, cudaMemcpyHostToDevice, st));
        zc.ensure(p * Wp * 8);
        brute::make_z<<<grid_for(p * Wp, 256), 256, 0, st>>>(ds->Xc.as<u64>(), Wp, W, p, yb.as<u64>(), zc.as<u64>());
        XYZB_LAUNCH_CHECK();
        hist.ensure((n + 1) * 8);
        XYZB_CUDA(cudaMemsetAsync(hist.p, 0, (n + 1) * 8, st));
        const size_t hs = n <= brute::kSmemHistMax ? size_t(n + 1) * 4 : 0;
        func_smem(brute::all_pairs<false>, (brute::kSmemHistMax + 1) * 4);
        const u64* nzp = yb.as<u64>() + Wp;
        // tensor cores (tcgen05 kind::i8 Gram product); the brute_cuda test option runs the CUDA-core
        // popcount tiles instead (the independent cross-check of the tensor-core kernel)
        const bool tc = !topt().brute_cuda.load();
        u32 nz = 0;
        for (u64 i = 0; i < n; ++i) nz += (y_sign[i] == 1 || y_sign[i] == -1) ? 1u : 0u;
        const u64 Kp = round_up(n, 128);
        DevBuf opA, opB;
        CUtensorMap tmA{}, tmB{};
        if (tc) {
            opA.ensure(p * Kp);
            opB.ensure(p * Kp);
            brute::make_pm1<<<grid_for(p * Kp / 8, 256), 256, 0, st>>>(ds->Xc.as<u64>(), Wp, p, n, Kp, yb.as<u64>(),
                                                                     nzp, opA.as<int8_t>(), opB.as<int8_t>());
            XYZB_LAUNCH_CHECK();
            tmA = operand_map(opA.p, p, Kp, brute::kTcM);
            tmB = operand_map(opB.p, p, Kp, brute::kTcN);
            func_smem(brute::all_pairs_tc2<false>, brute::kTcSmem2);
            func_smem(brute::all_pairs_tc2<true>, brute::kTcSmem2);
        }
        const u64 ntc = u64((p + brute::kTcM - 1) / brute::kTcM) * ((p + brute::kTcN - 1) / brute::kTcN);
        const u32 tc_grid = static_cast<u32>(std::min<u64>(ntc, kSMs));
        if (tc) {
            brute::all_pairs_tc2<false><<<tc_grid, brute::kTcWarps * 32, brute::kTcSmem2, st>>>(
                tmA, tmB, u32(p), u32(n), nz, u32(Kp), hist.as<unsigned long long>(), 0u, nullptr, nullptr, 0u);
        } else {
            brute::all_pairs<false><<<brute::all_pairs_grid(), brute::kThreads, hs, st>>>(
                ds->Xc.as<u64>(), zc.as<u64>(), nzp, Wp, W, u32(p), u32(n), hist.as<unsigned long long>(), 0u,
                nullptr, nullptr, 0u);
        }
        XYZB_LAUNCH_CHECK();
        std::vector<u64> cnt(n + 1);
        XYZB_CUDA(cudaMemcpyAsync(cnt.data(), hist.p, (n + 1) * 8, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        *pairs_scanned = p * (p - 1) / 2;
        const auto strength = [&](u64 a) { return double(a) / double(n); };
        if (histogram_bins > 0) {
            // scan_all_pairs' binning (oracle.cpp:36-41) applied to each exact agree count
            u64* h = static_cast<u64*>(std::calloc(histogram_bins, 8));
            if (!h) throw internal_error("brute_force_search: out of host memory");
            for (u64 a = 0; a <= n; ++a) {
                if (!cnt[a]) continue;
                auto bin = static_cast<size_t>(strength(a) * static_cast<double>(histogram_bins));
                if (bin >= histogram_bins) bin = histogram_bins - 1;
                h[bin] += cnt[a];
            }
            *histogram = h;
        }
        if (!has_gamma && !has_top_k) return;
        // smallest agree count kept by gamma, then the top-K cutoff among those
        u64 a_lo = 0;
        if (has_gamma) {
            a_lo = n + 1;
            for (u64 a = 0; a <= n; ++a)
                if (strength(a) >= gamma) {
                    a_lo = a;
                    break;
                }
        }
        u64 kept = 0;
        for (u64 a = a_lo; a <= n; ++a) kept += cnt[a];
        u64 cutoff = a_lo;
        u64 want = kept;
        if (has_top_k) {
            want = std::min<u64>(top_k, kept);
            if (want == 0) return;
            u64 acc = 0;
            for (u64 a = n + 1; a-- > a_lo;) {
                acc += cnt[a];
                if (acc >= want) {
                    cutoff = a;
                    break;
                }
            }
        }
        if (want == 0 || cutoff > n) return;
        u64 emit = 0;
        for (u64 a = cutoff; a <= n; ++a) emit += cnt[a];
        if (emit > 0xffffffffull) throw internal_error("brute_force_search: more than 2^32 pairs above the cut");
        DevBuf outb, nout;
        outb.ensure(emit * sizeof(brute::PairOut));
        nout.ensure(4);
        XYZB_CUDA(cudaMemsetAsync(nout.p, 0, 4, st));
        if (tc) {
            brute::all_pairs_tc2<true><<<tc_grid, brute::kTcWarps * 32, brute::kTcSmem2, st>>>(
                tmA, tmB, u32(p), u32(n), nz, u32(Kp), nullptr, u32(cutoff), outb.as<brute::PairOut>(),
                nout.as<u32>(), u32(emit));
        } else {
            brute::all_pairs<true><<<brute::all_pairs_grid(), brute::kThreads, 0, st>>>(
                ds->Xc.as<u64>(), zc.as<u64>(), nzp, Wp, W, u32(p), u32(n), nullptr, u32(cutoff),
                outb.as<brute::PairOut>(), nout.as<u32>(), u32(emit));
        }
        XYZB_LAUNCH_CHECK();
        std::vector<brute::PairOut> got(emit);
        XYZB_CUDA(cudaMemcpyAsync(got.data(), outb.p, emit * sizeof(brute::PairOut), cudaMemcpyDeviceToHost, st));
        u32 nget = 0;
        XYZB_CUDA(cudaMemcpyAsync(&nget, nout.p, 4, cudaMemcpyDeviceToHost, st));
        XYZB_CUDA(cudaStreamSynchronize(st));
        if (nget != emit) throw internal_error("brute_force_search: emitted pair count differs from the histogram");
        const auto by_jk = [](const brute::PairOut& x, const brute::PairOut& y) {
            return x.j != y.j ? x.j < y.j : x.k < y.k;
        };
        if (has_top_k) {
            // oracle.cpp:45-56: strength desc, (j, k) asc; the K best, then (j, k) order
            std::sort(got.begin(), got.end(), [&](const brute::PairOut& x, const brute::PairOut& y) {
                if (x.agree != y.agree) return x.agree > y.agree;
                return by_jk(x, y);
            });
            got.resize(want);
        }
        std::sort(got.begin(), got.end(), by_jk);
        auto* outp = static_cast<xyzb_scored_pair*>(std::malloc(std::max<size_t>(1, got.size()) * sizeof(xyzb_scored_pair)));
        if (!outp) throw internal_error("brute_force_search: out of host memory");
        for (size_t t = 0; t < got.size(); ++t) outp[t] = xyzb_scored_pair{got[t].j, got[t].k, strength(got[t].agree)};
        *pairs = outp;
        *n_pairs = got.size();
    });
}

namespace {

// Merge per-shard results into one report identical to the unsharded search
// (xyzb_merge_results; the multi-device search's last step).
void merge_parts(xyzb_dataset* ds, const xyzb_result* parts, u64 n_parts, const xyzb_params* params,
                 xyzb_result* out) {
    {
        if (params->stop_after_first_hit) throw data_error("xyzb: stop_after_first_hit cannot be combined with a rep shard");
        DeviceGuard dg(ds->device);
        StreamScope ss(ds->stream);
        SearchCtx c;
        c.ds = ds;
        c.q = params;
        c.mode = params->mode;
        c.n = ds->n;
        c.p = ds->p;
        c.M = params->m;
        c.gamma = params->gamma;
        c.plan.L = params->l;
        c.plan.npass = params->search_negatives ? 2 : 1;
        c.plan.sign_by_rid.resize(c.plan.npass * c.plan.L);
        for (int ps = 0; ps < c.plan.npass; ++ps)
            for (u64 r = 0; r < c.plan.L; ++r) c.plan.sign_by_rid[ps * c.plan.L + r] = ps == 0 ? 1 : -1;
        const u64 Rall = c.plan.sign_by_rid.size();
        ds->sign_by_rid.ensure(Rall);
        XYZB_CUDA(cudaMemcpyAsync(ds->sign_by_rid.p, c.plan.sign_by_rid.data(), Rall, cudaMemcpyHostToDevice,
                                  ds->stream));
        std::vector<kern::DevHit> all;
        for (u64 t = 0; t < n_parts; ++t) {
            const xyzb_result& r = parts[t];
            for (u64 i = 0; i < r.n_hits; ++i) {
                kern::DevHit h;
                h.order = r.order_keys[i];  // x-side key v
                h.s = r.hits[i].strength;
                h.j = r.hits[i].j;
                h.k = r.hits[i].k;
                h.rid = static_cast<u32>((r.hits[i].sign > 0 ? 0 : c.plan.L) + r.hits[i].found_at_repetition - 1);
                h.sint = -1;
                all.push_back(h);
            }
            out->repetitions_run += r.repetitions_run;
            out->runs_executed += r.runs_executed;
            out->candidates_enumerated += r.candidates_enumerated;
            out->aborted_repetitions += r.aborted_repetitions;
            out->candidates_checked += r.candidates_checked;
            out->verified_pairs += r.verified_pairs;
            out->device_ms = std::max(out->device_ms, r.device_ms);
            out->wall_time_s = std::max(out->wall_time_s, r.wall_time_s);
            if (out->estimated_c == 0.0) out->estimated_c = r.estimated_c;
            for (int s = 0; s < XYZB_NUM_STAGES; ++s) {
                out->stage_ms[s] += r.stage_ms[s];
                out->stage_bytes[s] += r.stage_bytes[s];
                out->stage_launches[s] += r.stage_launches[s];
            }
            out->kernel_launches += r.kernel_launches;
            out->verify_kernel_ms += r.verify_kernel_ms;
            out->verify_launches += r.verify_launches;
            out->devices_used = std::max<u64>(out->devices_used, r.devices_used);
            out->attempts = std::max<u64>(out->attempts, r.attempts);
        }
        if (all.size() > 0xffffffffull) throw internal_error("xyzb_merge_results: too many hits");
        const u32 H = static_cast<u32>(all.size());
        if (H > ds->hit_cap) ds->hit_cap = H;
        ds->hits.ensure(std::max<u64>(1, all.size()) * sizeof(kern::DevHit));
        if (H) XYZB_CUDA(cudaMemcpyAsync(ds->hits.p, all.data(), all.size() * sizeof(kern::DevHit),
                                         cudaMemcpyHostToDevice, ds->stream));
        ds->partial.ensure(scan::kGrid * 8);
        std::vector<xyzb_hit> hits;
        std::vector<u64> order, topk;
        merge_hits(c, H, 0xffffffffu, hits, order, topk);
        out->gamma_effective = params->gamma;
        if (params->top_k_mode == XYZB_TOPK_CANDIDATES) out->gamma_effective = topk_filter(hits, order, topk);
        out->gamma0 = std::pow(double(c.p), -1.0 / double(c.M));
        out->m_used = c.M;
        out->l_used = params->l;
        out->n_hits = hits.size();
        out->hits = static_cast<xyzb_hit*>(std::malloc(std::max<size_t>(1, hits.size()) * sizeof(xyzb_hit)));
        out->order_keys = static_cast<u64*>(std::malloc(std::max<size_t>(1, order.size()) * 8));
        if (!hits.empty()) {
            std::memcpy(out->hits, hits.data(), hits.size() * sizeof(xyzb_hit));
            std::memcpy(out->order_keys, order.data(), order.size() * 8);
        }
        out->n_top_k = topk.size();
        out->top_k = static_cast<u64*>(std::malloc(std::max<size_t>(1, topk.size()) * 8));
        if (!topk.empty()) std::memcpy(out->top_k, topk.data(), topk.size() * 8);
    }
}

// Repetition shard g of G: [1 + L g / G, 1 + L (g + 1) / G) (parallel.shard_bounds)
std::pair<u64, u64> shard_bounds(u64 L, u64 g, u64 G) { return {1 + L * g / G, 1 + L * (g + 1) / G}; }

// A search over the dataset's replicas (xyzb_problem.devices): each device
// takes a contiguous repetition shard of each pass on its own host thread and
// stream, then the shard results merge on the primary device — the same
// report as one device (replaces the thread waves of run_pass,
// search.cpp:59-111).
void multi_search(xyzb_dataset* ds, const xyzb_response* resp, const xyzb_params* q, const uint32_t* draws,
                  xyzb_result* out) {
    Nvtx nv("xyzb_search:devices");
    const auto t0 = std::chrono::steady_clock::now();
    validate_params(q);
    std::vector<xyzb_dataset*> devs{ds};
    for (auto& r : ds->replicas) devs.push_back(r.get());
    const u64 G = std::min<u64>(devs.size(), q->l);  // no empty shards
    std::vector<xyzb_params> qs(G, *q);
    std::vector<xyzb_result> parts(G);
    std::vector<std::exception_ptr> errs(G);
    for (auto& r : parts) std::memset(&r, 0, sizeof(r));
    std::vector<std::thread> th;
    for (u64 g = 0; g < G; ++g) {
        const auto b = shard_bounds(q->l, g, G);
        qs[g].rep_begin = b.first;
        qs[g].rep_end = b.second;
        qs[g].estimate_complexity = g == 0 ? q->estimate_complexity : 0;  // a per-search quantity: once
        th.emplace_back([&, g] {
            try {
                do_search(devs[g], resp, &qs[g], draws, &parts[g]);
            } catch (...) {
                errs[g] = std::current_exception();
            }
        });
    }
    for (auto& t : th) t.join();
    struct Free {
        std::vector<xyzb_result>& v;
        ~Free() {
            for (auto& r : v) xyzb_result_free(&r);
        }
    } fr{parts};
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    merge_parts(ds, parts.data(), G, q, out);
    out->estimated_c = parts[0].estimated_c;
    out->devices_used = G;
    out->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

} // namespace

extern "C" int xyzb_merge_results(xyzb_dataset* ds, const xyzb_result* parts, uint64_t n_parts,
                                  const xyzb_params* params, xyzb_result* out, char* err, size_t errlen) {
    if (out) std::memset(out, 0, sizeof(*out));
    return guarded(err, errlen, [&] {
        if (!ds || !params || !out || (n_parts && !parts)) throw data_error("xyzb_merge_results: null argument");
        merge_parts(ds, parts, n_parts, params, out);
    });
}

namespace {

// ------------------------------------------------- xyz-regression design --
// Centered correlations of lasso_path's exact scans (lasso.cpp:74-92): one
// warp per column / pair, fp64 products rounded as the host's left-to-right
// r * (x_j - m_j) * (x_k - m_k), warp-tree sums.
namespace design {

__global__ void __launch_bounds__(256) main_corr(const double* __restrict__ X, const double* __restrict__ m, u64 n,
                                                 u64 p, const double* __restrict__ r, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const u64 nw = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 j = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < p; j += nw) {
        const double* col = X + j * n;
        const double mj = m[j];
        double acc = 0.0;
        for (u64 i = lane; i < n; i += 32) acc = __dadd_rn(acc, __dmul_rn(__ldg(r + i), __dsub_rn(__ldg(col + i), mj)));
        acc = warp_sum(acc);
        if (lane == 0) out[j] = acc;
    }
}

__global__ void __launch_bounds__(256) pair_corr(const double* __restrict__ X, const double* __restrict__ m, u64 n,
                                                 const u32* __restrict__ pairs, u64 cnt,
                                                 const double* __restrict__ r, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const u64 nw = (u64(gridDim.x) * blockDim.x) >> 5;
    for (u64 t = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; t < cnt; t += nw) {
        const u32 j = pairs[2 * t], k = pairs[2 * t + 1];
        const double *cj = X + u64(j) * n, *ck = X + u64(k) * n;
        const double mj = m[j], mk = m[k];
        double acc = 0.0;
        for (u64 i = lane; i < n; i += 32) {
            const double a = __dmul_rn(__ldg(r + i), __dsub_rn(__ldg(cj + i), mj));
            acc = __dadd_rn(acc, __dmul_rn(a, __dsub_rn(__ldg(ck + i), mk)));
        }
        acc = warp_sum(acc);
        if (lane == 0) out[t] = acc;
    }
}

} // namespace design

} // namespace

struct xyzb_design {
    int device = 0;
    u64 n = 0, p = 0;
    cudaStream_t stream = nullptr;
    DevBuf x, means, r, pairs, out;
    ~xyzb_design() {
        if (stream) {
            cudaStreamSynchronize(stream);
            cudaStreamDestroy(stream);
        }
    }
};

namespace {

void design_residual(xyzb_design* d, const double* residual) {
    if (!residual) throw data_error("xyzb_design: null residual");
    d->r.ensure(d->n * 8);
    XYZB_CUDA(cudaMemcpyAsync(d->r.p, residual, d->n * 8, cudaMemcpyHostToDevice, d->stream));
}

} // namespace

// ------------------------------------------------------------ C ABI --

extern "C" {

int xyzb_abi_version(void) { return XYZB_ABI_VERSION; }

void xyzb_params_init(xyzb_params* q) {
    std::memset(q, 0, sizeof(*q));
    q->m = 8;  // SearchConfig defaults (search.hpp:18-33)
    q->l = 1;
    q->gamma = 0.9;
    q->mode = XYZB_MODE_BINARY;
    q->transform = XYZB_TRANSFORM_NONE;
    q->search_negatives = 1;
    q->estimate_complexity = 1;
}

int xyzb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int xyzb_dataset_create(const xyzb_problem* pr, xyzb_dataset** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        *out = nullptr;
        if (!pr) throw data_error("xyzb_dataset_create: null problem");
        if (pr->n_rows == 0 || pr->n_cols == 0) throw data_error("PackedMatrix: n_rows and n_cols must be >= 1");
        if (int(pr->x_words != nullptr) + int(pr->x_real != nullptr) + int(pr->x_real32 != nullptr) != 1)
            throw data_error("xyzb_dataset_create: exactly one of x_words / x_real / x_real32 must be set");
        if (pr->n_rows > 0xffffffffull) throw data_error("xyzb: more than 2^32-1 rows");
        if (pr->n_devices && !pr->devices) throw data_error("xyzb_dataset_create: null device list");
        // padding bits must be clear (PackedMatrix invariant, packed_matrix.hpp:10-14): checked on
        // the host before any device work, except for page-locked X (DMA'd as is, checked on the device)
        const bool pinned_x = pr->x_words && is_pinned(pr->x_words);
        if (pr->x_words && !pinned_x) {
            const u64 W = ceil_div(pr->n_rows, 64);
            const u64 tail = pr->n_rows & 63;
            if (tail)
                for (u64 j = 0; j < pr->n_cols; ++j)
                    if (pr->x_words[j * W + W - 1] >> tail)
                        throw data_error("xyzb_dataset_create: padding bits of column " + std::to_string(j) +
                                         " are not zero");
        }
        require_device();
        const int ndev = xyzb_device_count();
        std::vector<int> devs;
        if (pr->n_devices) devs.assign(pr->devices, pr->devices + pr->n_devices);
        else devs.push_back(pr->device);
        for (int d : devs)
            if (d < 0 || d >= ndev)
                throw data_error("xyzb_dataset_create: device " + std::to_string(d) + " outside [0, " +
                                 std::to_string(ndev) + ")");
        Nvtx nv("xyzb_dataset_create");
        std::unique_ptr<xyzb_dataset> ds(new xyzb_dataset());
        ds->device = devs[0];
        if (const long long e = topt().hit_cap.load())  // tests force the hit-buffer regrow path
            ds->hit_cap = static_cast<u32>(std::max<u64>(1, u64(e)));
        {
            DeviceGuard dg(ds->device);
            XYZB_CUDA(cudaStreamCreateWithFlags(&ds->stream, cudaStreamNonBlocking));
            StreamScope ss(ds->stream);
            ds->n = pr->n_rows;
            ds->p = pr->n_cols;
            const cudaStream_t st = ds->stream;
            if (pr->x_words)
                create_binary(ds.get(), [&](void* d, size_t b) { upload(d, pr->x_words, b, st); }, pinned_x);
            else if (pr->x_real)
                create_real(ds.get(), [&](void* d, size_t b) { upload(d, pr->x_real, b, st); }, false);
            else
                create_real(ds.get(), [&](void* d, size_t b) { upload(d, pr->x_real32, b, st); }, true);
            XYZB_CUDA(cudaStreamSynchronize(ds->stream));
        }
        // further devices: peer copies of the primary's device-resident X
        for (size_t g = 1; g < devs.size(); ++g) ds->replicas.push_back(replicate(ds.get(), devs[g]));
        *out = ds.release();
    });
}

xyzb_dataset::~xyzb_dataset() {
    for (auto& r : replicas) xyzb_dataset_destroy(r.release());
}

void xyzb_dataset_destroy(xyzb_dataset* ds) {
    if (!ds) return;
    {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(ds->device);
        cudaStreamSynchronize(ds->stream);
        cudaStream_t st = ds->stream;
        cudaStream_t prev_drained = tl_drained;
        tl_drained = st;  // every buffer of the dataset is idle now
        delete ds;
        tl_drained = prev_drained;
        cudaStreamDestroy(st);
        cudaSetDevice(prev);
    }
}

int xyzb_dataset_open(const char* path, int32_t device, xyzb_dataset** out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        *out = nullptr;
        const std::string ps = path ? path : "";
        std::unique_ptr<std::FILE, int (*)(std::FILE*)> f(std::fopen(ps.c_str(), "rb"), std::fclose);
        if (!f) throw data_error("read_dataset: cannot open " + ps);
        unsigned char head[8];
        if (std::fread(head, 1, 8, f.get()) != 8 || std::memcmp(head, "XYZ1", 4) != 0)
            throw data_error("read_dataset: bad magic in " + ps);
        if (head[4] > 1) throw data_error("read_dataset: unknown dataset kind");
        u64 dims[2] = {0, 0};
        if (std::fread(dims, 8, 2, f.get()) != 2 || dims[0] == 0 || dims[1] == 0)
            throw data_error("read_dataset: bad header dimensions");
        const bool binary = head[4] == 0;
        if (dims[0] > 0xffffffffull) throw data_error("xyzb: more than 2^32-1 rows");
        require_device();
        std::unique_ptr<xyzb_dataset> ds(new xyzb_dataset());
        ds->device = device;
        DeviceGuard dg(device);
        XYZB_CUDA(cudaStreamCreateWithFlags(&ds->stream, cudaStreamNonBlocking));
        StreamScope ss(ds->stream);
        ds->n = dims[0];
        ds->p = dims[1];
        const cudaStream_t st = ds->stream;
        const u64 W = ceil_div(ds->n, 64);
        if (binary) {
            create_binary(ds.get(), [&](void* d, size_t b) { stream_file(d, f.get(), b, true, W, ds->n, ps, st); });
        } else {
            create_real(ds.get(), [&](void* d, size_t b) { stream_file(d, f.get(), b, false, W, ds->n, ps, st); },
                        false);
        }
        XYZB_CUDA(cudaStreamSynchronize(ds->stream));
        *out = ds.release();
    });
}

int xyzb_dataset_shape(const xyzb_dataset* ds, uint64_t* n_rows, uint64_t* n_cols, int32_t* binary) {
    if (!ds) return XYZB_E_DATA;
    if (n_rows) *n_rows = ds->n;
    if (n_cols) *n_cols = ds->p;
    if (binary) *binary = ds->binary ? 1 : 0;
    return XYZB_OK;
}

int xyzb_search(xyzb_dataset* ds, const xyzb_response* resp, const xyzb_params* params, const uint32_t* draws,
                xyzb_result* out, char* err, size_t errlen) {
    if (out) std::memset(out, 0, sizeof(*out));
    return guarded(err, errlen, [&] {
        if (!ds || !params || !out) throw data_error("xyzb_search: null argument");
        // replicas: shard the runs over the devices, unless the caller already shards (rep range) or the
        // search must stop at the first hit (sequential by definition)
        if (!ds->replicas.empty() && !params->stop_after_first_hit && !(params->rep_begin || params->rep_end))
            multi_search(ds, resp, params, draws, out);
        else
            do_search(ds, resp, params, draws, out);
    });
}

void xyzb_result_free(xyzb_result* r) {
    if (!r) return;
    std::free(r->hits);
    std::free(r->order_keys);
    std::free(r->top_k);
    r->hits = nullptr;
    r->order_keys = nullptr;
    r->top_k = nullptr;
}

int xyzb_design_create(const double* x, uint64_t n_rows, uint64_t n_cols, const double* means, int32_t device,
                       xyzb_design** out, char* err, size_t errlen) {
    if (out) *out = nullptr;
    return guarded(err, errlen, [&] {
        if (!x || !means || !out) throw data_error("xyzb_design_create: null argument");
        if (n_rows == 0 || n_cols == 0) throw data_error("xyzb_design_create: empty design");
        require_device();
        DeviceGuard g(device);
        auto d = std::make_unique<xyzb_design>();
        d->device = device;
        d->n = n_rows;
        d->p = n_cols;
        XYZB_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
        StreamScope sc(d->stream);
        d->x.ensure(n_rows * n_cols * 8);
        d->means.ensure(n_cols * 8);
        XYZB_CUDA(cudaMemcpyAsync(d->x.p, x, n_rows * n_cols * 8, cudaMemcpyHostToDevice, d->stream));
        XYZB_CUDA(cudaMemcpyAsync(d->means.p, means, n_cols * 8, cudaMemcpyHostToDevice, d->stream));
        XYZB_CUDA(cudaStreamSynchronize(d->stream));
        *out = d.release();
    });
}

void xyzb_design_destroy(xyzb_design* d) {
    if (!d) return;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(d->device);
    {
        StreamScope sc(d->stream);
        cudaStreamSynchronize(d->stream);
        tl_drained = d->stream;
        delete d;
        tl_drained = nullptr;
    }
    cudaSetDevice(cur);
}

int xyzb_design_main_correlations(xyzb_design* d, const double* residual, double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!d || !out) throw data_error("xyzb_design_main_correlations: null argument");
        DeviceGuard g(d->device);
        StreamScope sc(d->stream);
        design_residual(d, residual);
        d->out.ensure(d->p * 8);
        design::main_corr<<<static_cast<u32>(std::min<u64>(ceil_div(d->p * 32, 256), u64(kSMs) * 16)), 256, 0,
                            d->stream>>>(d->x.as<double>(), d->means.as<double>(), d->n, d->p, d->r.as<double>(),
                                         d->out.as<double>());
        XYZB_LAUNCH_CHECK();
        XYZB_CUDA(cudaMemcpyAsync(out, d->out.p, d->p * 8, cudaMemcpyDeviceToHost, d->stream));
        XYZB_CUDA(cudaStreamSynchronize(d->stream));
    });
}

int xyzb_design_pair_correlations(xyzb_design* d, const double* residual, const uint32_t* pairs_jk,
                                  uint64_t n_pairs, double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        if (!d || (n_pairs && (!pairs_jk || !out))) throw data_error("xyzb_design_pair_correlations: null argument");
        if (n_pairs == 0) return;
        for (u64 t = 0; t < 2 * n_pairs; ++t)
            if (pairs_jk[t] >= d->p) throw data_error("xyzb_design_pair_correlations: column index out of range");
        DeviceGuard g(d->device);
        StreamScope sc(d->stream);
        design_residual(d, residual);
        d->pairs.ensure(n_pairs * 8);
        d->out.ensure(n_pairs * 8);
        XYZB_CUDA(cudaMemcpyAsync(d->pairs.p, pairs_jk, n_pairs * 8, cudaMemcpyHostToDevice, d->stream));
        design::pair_corr<<<static_cast<u32>(std::min<u64>(ceil_div(n_pairs * 32, 256), u64(kSMs) * 16)), 256, 0,
                            d->stream>>>(d->x.as<double>(), d->means.as<double>(), d->n, d->pairs.as<u32>(), n_pairs,
                                         d->r.as<double>(), d->out.as<double>());
        XYZB_LAUNCH_CHECK();
        XYZB_CUDA(cudaMemcpyAsync(out, d->out.p, n_pairs * 8, cudaMemcpyDeviceToHost, d->stream));
        XYZB_CUDA(cudaStreamSynchronize(d->stream));
    });
}

void xyzb_free(void* p) { std::free(p); }

int xyzb_test_set_option(const char* name, long long value) {
    if (!name) return XYZB_E_DATA;
    TestOptions& o = topt();
    const std::string s = name;
    std::atomic<long long>* slot = s == "batch_entries"     ? &o.batch_entries
                                   : s == "hit_cap"         ? &o.hit_cap
                                   : s == "item_cap"        ? &o.item_cap
                                   : s == "pair_cap"        ? &o.pair_cap
                                   : s == "grouping"        ? &o.grouping
                                   : s == "merge_large"     ? &o.merge_large
                                   : s == "sign_verify_off" ? &o.sign_verify_off
                                   : s == "trace"           ? &o.trace
                                   : s == "brute_cuda"      ? &o.brute_cuda
                                   : s == "binned"          ? &o.binned
                                   : s == "binned_wshift"   ? &o.binned_wshift
                                   : s == "binned_cap"      ? &o.binned_cap
                                   : s == "one_pass_join"   ? &o.one_pass_join
                                   : s == "part_fixed"      ? &o.part_fixed
                                                            : nullptr;
    if (!slot) return XYZB_E_DATA;
    slot->store(value);
    return XYZB_OK;
}

} // extern "C"
