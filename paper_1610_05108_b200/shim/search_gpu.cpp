// Drop-in replacement for the reference's proj/core/src/search.cpp.
//
// Compiled against the reference's UNCHANGED public header xyz/search.hpp and
// linked in its place (shim/Makefile), it gives the reference's callers — the
// interaction Lasso's KKT screen (lasso.cpp:148-215), the CLI
// (xyz_main.cpp:184-191) and the experiments (experiments.cpp:71-72) — the
// B200 engine through the C ABI in include/xyzb.h:
//   * the three xyz_search overloads (search.hpp:100-111) validate exactly as
//     the reference does (search.cpp:119-134,325-334,367-374,415-434), then
//     run on the GPU; X is uploaded once and cached per matrix (the Lasso
//     screens the same rescaled X many times, lasso.cpp:118-141);
//   * the parameter selectors and the strength sampler (search.cpp:136-291)
//     are restated here on the host with the same formulas and evaluation
//     order, so auto-M / auto-L decisions are bit-identical to the reference.
// SearchConfig::threads is accepted and ignored: the searches shard their
// repetitions over the GPUs of gpu_devices() (devices.hpp, XYZ_GPU_DEVICES).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <mutex>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "xyz/errors.hpp"
#include "xyz/rng.hpp"
#include "xyz/search.hpp"
#include "xyz/transforms.hpp"
#include "xyzb.h"
#include "devices.hpp"

namespace xyz {

namespace {

double abs_sum(std::span<const double> v) {
    double s = 0.0;
    for (double t : v) s += std::abs(t);
    return s;
}

[[noreturn]] void rethrow(int code, const char* msg) {
    const std::string m = msg;
    if (code == XYZB_E_DATA) throw data_error(m);
    if (code == XYZB_E_GUARD) throw guard_error(m);
    if (code == XYZB_E_SOLVER) throw solver_error(m);
    throw std::runtime_error("xyz GPU engine: " + m);
}

// Full-content fingerprint (8 independent multiply-xor lanes per 64-byte
// block): the cache must never serve a stale matrix, so every byte is hashed.
// Large matrices are hashed in fixed 8 MiB segments on up to 16 host threads
// and the segment hashes folded in order (a 160 MB config 5 matrix: 22 ms on
// one thread, which the Lasso paid on each of its ~50 screens).
uint64_t fingerprint_segment(const unsigned char* b, size_t bytes) {
    uint64_t h[8];
    for (int l = 0; l < 8; ++l) h[l] = 0x9e3779b97f4a7c15ull * uint64_t(l + 1);
    size_t i = 0;
    for (; i + 64 <= bytes; i += 64) {
        uint64_t w[8];
        std::memcpy(w, b + i, 64);
        for (int l = 0; l < 8; ++l) h[l] = (h[l] ^ w[l]) * 0x100000001b3ull + (h[l] >> 29);
    }
    uint64_t r = 1469598103934665603ull;
    for (int l = 0; l < 8; ++l) r = (r ^ h[l]) * 1099511628211ull;
    for (; i < bytes; ++i) r = (r ^ b[i]) * 1099511628211ull;
    return r;
}

uint64_t fingerprint(const void* p, size_t bytes) {
    constexpr size_t kSeg = size_t(8) << 20;
    const unsigned char* b = static_cast<const unsigned char*>(p);
    const size_t nseg = (bytes + kSeg - 1) / kSeg;
    std::vector<uint64_t> seg(nseg, 0);
    const size_t nthr = std::min<size_t>({nseg, size_t(16), size_t(std::max(1u, std::thread::hardware_concurrency()))});
    auto work = [&](size_t t) {
        for (size_t s = t; s < nseg; s += nthr) seg[s] = fingerprint_segment(b + s * kSeg, std::min(kSeg, bytes - s * kSeg));
    };
    if (nthr <= 1) {
        work(0);
    } else {
        std::vector<std::thread> pool;
        for (size_t t = 1; t < nthr; ++t) pool.emplace_back(work, t);
        work(0);
        for (auto& th : pool) th.join();
    }
    uint64_t r = 1469598103934665603ull;
    for (const uint64_t v : seg) r = (r ^ v) * 1099511628211ull;
    return r ^ bytes;
}

// One resident dataset per distinct matrix (address, shape, content).
struct DatasetCache {
    std::mutex mu;
    xyzb_dataset* ds = nullptr;
    const void* ptr = nullptr;
    size_t n = 0, p = 0;
    bool binary = false;
    uint64_t fp = 0;
    ~DatasetCache() {
        if (ds) xyzb_dataset_destroy(ds);
    }
    xyzb_dataset* get(const uint64_t* words, const double* real, size_t n_, size_t p_, bool single = false) {
        const void* ptr_ = words ? static_cast<const void*>(words) : static_cast<const void*>(real);
        const size_t bytes = words ? p_ * ((n_ + 63) / 64) * 8 : n_ * p_ * 8;
        const uint64_t f = fingerprint(ptr_, bytes);
        if (ds && ptr == ptr_ && n == n_ && p == p_ && binary == (words != nullptr) && fp == f) return ds;
        if (ds) xyzb_dataset_destroy(ds);
        ds = nullptr;
        xyzb_problem prob{};
        prob.n_rows = n_;
        prob.n_cols = p_;
        prob.x_words = words;
        prob.x_real = real;
        std::vector<int32_t> devs = gpu_devices();  // X replicated on each; runs sharded over them
        if (single) devs.resize(1);
        prob.device = devs[0];
        prob.devices = devs.data();
        prob.n_devices = devs.size();
        char err[1024] = {0};
        const int code = xyzb_dataset_create(&prob, &ds, err, sizeof err);
        if (code != XYZB_OK) rethrow(code, err);
        ptr = ptr_;
        n = n_;
        p = p_;
        binary = words != nullptr;
        fp = f;
        return ds;
    }
};

DatasetCache& cache() {
    static DatasetCache c;
    return c;
}

// The Z matrix of sample_strengths' binary overload (the CLI's auto-M sample,
// xyz_main.cpp:142-149), resident beside X.
DatasetCache& zcache() {
    static DatasetCache c;
    return c;
}

xyzb_params to_params(const SearchConfig& c) {
    xyzb_params q;
    xyzb_params_init(&q);
    q.m = c.m;
    q.l = c.l;
    q.gamma = c.gamma;
    q.mode = static_cast<int32_t>(c.mode);
    q.transform = static_cast<int32_t>(c.transform);
    q.search_negatives = c.search_negatives ? 1 : 0;
    q.stop_after_first_hit = c.stop_after_first_hit ? 1 : 0;
    q.estimate_complexity = c.estimate_complexity ? 1 : 0;
    q.threads = static_cast<int32_t>(c.threads);
    q.seed = c.seed;
    q.max_candidates_per_rep = c.max_candidates_per_rep;
    q.strength_sample_size = c.strength_sample_size;
    return q;
}

// XYZB_SHIM_STATS=1: time spent in GPU searches, printed at exit (how much of
// a caller such as lasso_path is the screen).
struct ShimStats {
    double seconds = 0.0;
    size_t calls = 0, hits = 0;
    ~ShimStats() {
        if (std::getenv("XYZB_SHIM_STATS"))
            std::fprintf(stderr, "[xyz_search shim] %zu calls, %.3f s, %zu hits\n", calls, seconds, hits);
    }
};
ShimStats& shim_stats() {
    static ShimStats s;
    return s;
}

SearchReport run_gpu(const uint64_t* words, const double* real, size_t n, size_t p, const xyzb_response& resp,
                     const SearchConfig& cfg) {
    const auto t0 = std::chrono::steady_clock::now();
    std::lock_guard<std::mutex> lock(cache().mu);
    xyzb_dataset* ds = cache().get(words, real, n, p);
    const xyzb_params q = to_params(cfg);
    xyzb_result r;
    char err[1024] = {0};
    const int code = xyzb_search(ds, &resp, &q, nullptr, &r, err, sizeof err);
    if (code != XYZB_OK) {
        xyzb_result_free(&r);
        rethrow(code, err);
    }
    SearchReport rep;
    rep.hits.resize(r.n_hits);
    for (size_t i = 0; i < r.n_hits; ++i) {
        rep.hits[i].j = r.hits[i].j;
        rep.hits[i].k = r.hits[i].k;
        rep.hits[i].strength = r.hits[i].strength;
        rep.hits[i].found_at_repetition = r.hits[i].found_at_repetition;
        rep.hits[i].sign = r.hits[i].sign;
    }
    rep.repetitions_run = r.repetitions_run;
    rep.candidates_checked = r.candidates_checked;
    rep.candidates_enumerated = r.candidates_enumerated;
    rep.aborted_repetitions = r.aborted_repetitions;
    rep.wall_time_s = r.wall_time_s;
    rep.estimated_c = r.estimated_c;
    rep.gamma0 = r.gamma0;
    rep.m_used = r.m_used;
    rep.l_used = r.l_used;
    xyzb_result_free(&r);
    ShimStats& st = shim_stats();
    st.seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    ++st.calls;
    st.hits += rep.hits.size();
    return rep;
}

// Uniform (j, k), j != k, k redrawn on collision (search.cpp:229-238), in
// the reference's RNG order. `check(j, k)` runs after each draw: the
// reference evaluates each pair right after drawing it, so an argument error
// leaves the caller's generator exactly where the reference leaves it.
template <class Check>
std::vector<uint32_t> draw_pairs(size_t p, size_t count, std::mt19937_64& rng, Check&& check) {
    if (count < 1) throw data_error("sample_strengths: need n_samples >= 1");
    if (p > 0xffffffffull) throw data_error("sample_strengths: too many columns for the GPU engine");
    std::uniform_int_distribution<size_t> dist(0, p - 1);
    std::vector<uint32_t> jk(2 * count);
    for (size_t t = 0; t < count; ++t) {
        const size_t j = dist(rng);
        size_t k = dist(rng);
        while (p > 1 && k == j) k = dist(rng);
        check(j, k);
        jk[2 * t] = static_cast<uint32_t>(j);
        jk[2 * t + 1] = static_cast<uint32_t>(k);
    }
    return jk;
}

// The drawn pairs' strengths on the device, bit-identical to the host's
// (xyzb_pair_strengths evaluates each pair in the reference's order).
StrengthSample device_strengths(xyzb_dataset* ds, const xyzb_response& resp, int32_t mode, int32_t transform,
                                const std::vector<uint32_t>& jk) {
    xyzb_params q;
    xyzb_params_init(&q);
    q.mode = mode;
    q.transform = transform;
    StrengthSample s;
    s.strengths.resize(jk.size() / 2);
    char err[1024] = {0};
    const int code = xyzb_pair_strengths(ds, &resp, &q, jk.data(), s.strengths.size(), s.strengths.data(), err,
                                         sizeof err);
    if (code != XYZB_OK) rethrow(code, err);
    return s;
}

} // namespace

// ---- configuration and selectors (search.cpp:119-220), restated ----

void SearchConfig::validate() const {
    if (m < 1 || m > max_subsample_size)
        throw data_error("SearchConfig: M = " + std::to_string(m) + " outside [1,64]");
    if (l < 1) throw data_error("SearchConfig: L must be >= 1");
    if (!(gamma > 0.0 && gamma <= 1.0)) throw data_error("SearchConfig: gamma must lie in (0,1]");
    const bool xy = mode == SearchMode::continuous_xy;
    if (xy && transform == BinarizeTransform::none)
        throw data_error("SearchConfig: continuous-XY mode requires a binarize transform");
    if (!xy && transform != BinarizeTransform::none)
        throw data_error("SearchConfig: binarize transform is only valid in continuous-XY mode");
}

double StrengthSample::mean_pow(std::size_t m) const {
    if (strengths.empty()) throw data_error("StrengthSample: empty sample");
    double acc = 0.0;
    for (const double s : strengths) acc += std::pow(s, static_cast<double>(m));
    return acc / static_cast<double>(strengths.size());
}

double StrengthSample::se_pow(std::size_t m) const {
    if (strengths.empty()) throw data_error("StrengthSample: empty sample");
    const double mu = mean_pow(m);
    double ss = 0.0;
    for (const double s : strengths) {
        const double d = std::pow(s, static_cast<double>(m)) - mu;
        ss += d * d;
    }
    const double cnt = static_cast<double>(strengths.size());
    return std::sqrt(ss / cnt / cnt);
}

double discovery_probability(double gamma, std::size_t m, std::size_t l) {
    if (!(gamma > 0.0 && gamma <= 1.0)) throw data_error("discovery_probability: gamma outside (0,1]");
    if (m < 1 || l < 1) throw data_error("discovery_probability: M and L must be >= 1");
    return 1.0 - std::pow(1.0 - std::pow(gamma, static_cast<double>(m)), static_cast<double>(l));
}

std::size_t choose_l(std::size_t m, double gamma, double eta_target) {
    if (!(gamma > 0.0 && gamma <= 1.0)) throw data_error("choose_l: gamma outside (0,1]");
    if (!(eta_target >= 0.5 && eta_target < 1.0)) throw data_error("choose_l: eta target must lie in [0.5,1)");
    const double gm = std::pow(gamma, static_cast<double>(m));
    if (gm >= 1.0) return 1;
    if (gm <= 0.0) throw data_error("choose_l: gamma^M underflows to zero; choose a smaller M");
    const double lr = std::log1p(-eta_target) / std::log1p(-gm);  // minimal real L
    if (!(lr < 1e15)) throw data_error("choose_l: required L exceeds 1e15; choose a smaller M");
    return std::max<std::size_t>(1, static_cast<std::size_t>(std::ceil(lr)));
}

double expected_complexity(std::size_t m, std::size_t l, const StrengthSample& sample, std::size_t n,
                           std::size_t p) {
    if (l < 1) throw data_error("expected_complexity: L must be >= 1");
    const double pd = static_cast<double>(p);
    const double e1 = pd * pd * sample.mean_pow(m);
    return static_cast<double>(n) * pd +
           static_cast<double>(l) * (static_cast<double>(m) * pd + pd * std::log(pd) + static_cast<double>(n) * e1);
}

MSelection optimal_m(double gamma, const StrengthSample& sample, std::size_t n, std::size_t p, std::size_t m_lo,
                     std::size_t m_hi) {
    if (!(gamma > 0.0 && gamma < 1.0)) throw data_error("optimal_m: gamma must lie in (0,1)");
    if (sample.strengths.empty()) throw data_error("optimal_m: empty strength sample");
    if (m_lo < 1 || m_hi > max_subsample_size || m_lo > m_hi) throw data_error("optimal_m: invalid M range");
    const double pd = static_cast<double>(p), nd = static_cast<double>(n);
    MSelection best;
    double best_obj = std::numeric_limits<double>::infinity(), best_se = 0.0;
    for (std::size_t m = m_lo; m <= m_hi; ++m) {
        const double gm = std::pow(gamma, static_cast<double>(m));
        if (gm <= 0.0) break;
        const double denom = -std::log1p(-gm);
        const double obj = (static_cast<double>(m) * pd + pd * std::log(pd) + nd * pd * pd * sample.mean_pow(m)) /
                           denom;
        if (obj < best_obj) {  // strict: exact ties keep the smaller M
            best_obj = obj;
            best.m = m;
            best_se = nd * pd * pd * sample.se_pow(m) / denom;
        }
    }
    if (best.m == 0) throw data_error("optimal_m: objective not finite anywhere in range");
    best.objective = best_obj;
    best.objective_rel_err = best_obj > 0.0 ? best_se / best_obj : 0.0;
    best.gamma0 = std::pow(pd, -1.0 / static_cast<double>(best.m));
    best.hit_range_cap = best.m == m_hi;
    return best;
}

double runtime_exponent(double gamma, double gamma0) {
    if (!(gamma0 > 0.0 && gamma0 < gamma && gamma <= 1.0))
        throw data_error("runtime_exponent: need 0 < gamma0 < gamma <= 1");
    return 1.0 + std::log(gamma) / std::log(gamma0);
}

// sample_strengths (search.cpp:229-291): the pairs are drawn on the host in
// the reference's RNG order, their strengths computed on the GPU (one thread
// per pair, the reference's evaluation order: bit-identical samples, so
// optimal_m / expected_complexity decide exactly as the reference does).
StrengthSample sample_strengths(const PackedMatrix& x, const PackedMatrix& z, std::size_t n_samples,
                                std::mt19937_64& rng) {
    const auto jk = draw_pairs(x.n_cols(), n_samples, rng, [&](size_t j, size_t k) {
        // interaction_strength's argument checks (transforms.cpp:33-38), at the first failing pair
        if (j >= z.n_cols()) throw data_error("interaction_strength: index j out of range");
        if (k >= x.n_cols()) throw data_error("interaction_strength: index k out of range");
        if (x.n_rows() != z.n_rows()) throw data_error("interaction_strength: row count mismatch");
    });
    std::lock_guard<std::mutex> lock(cache().mu);
    std::lock_guard<std::mutex> zlock(zcache().mu);
    xyzb_dataset* xd = cache().get(x.column_words(0).data(), nullptr, x.n_rows(), x.n_cols());
    xyzb_dataset* zd = zcache().get(z.column_words(0).data(), nullptr, z.n_rows(), z.n_cols(), true);
    std::vector<uint64_t> agree(n_samples);
    char err[1024] = {0};
    const int code = xyzb_pair_agreements(zd, xd, jk.data(), n_samples, agree.data(), err, sizeof err);
    if (code != XYZB_OK) rethrow(code, err);
    StrengthSample s;
    s.strengths.resize(n_samples);
    for (size_t t = 0; t < n_samples; ++t)
        s.strengths[t] = static_cast<double>(agree[t]) / static_cast<double>(x.n_rows());
    return s;
}

StrengthSample sample_strengths(const PackedMatrix& x, std::span<const double> y, std::size_t n_samples,
                                std::mt19937_64& rng) {
    const auto jk = draw_pairs(x.n_cols(), n_samples, rng, [&](size_t, size_t) {
        // weighted_interaction_strength's checks (transforms.cpp:44-53), thrown at the first pair
        if (y.size() != x.n_rows()) throw data_error("weighted_interaction_strength: response length mismatch");
        if (abs_sum(y) <= 0.0) throw data_error("weighted_interaction_strength: zero response vector");
    });
    std::lock_guard<std::mutex> lock(cache().mu);
    xyzb_dataset* ds = cache().get(x.column_words(0).data(), nullptr, x.n_rows(), x.n_cols());
    xyzb_response resp{};
    resp.y_real = y.data();
    return device_strengths(ds, resp, XYZB_MODE_CONTINUOUS_Y, XYZB_TRANSFORM_NONE, jk);
}

StrengthSample sample_strengths(const RealMatrix& x, const RealVector& y, BinarizeTransform transform,
                                std::size_t n_samples, std::mt19937_64& rng) {
    if (n_samples < 1) throw data_error("sample_strengths: need n_samples >= 1");
    if (transform == BinarizeTransform::none)
        throw data_error("sample_strengths: continuous data needs a binarize transform");
    if (abs_sum(y) <= 0.0) throw data_error("sample_strengths: zero response vector");
    if (y.size() < x.n_rows()) throw data_error("sample_strengths: response shorter than the matrix");
    const auto jk = draw_pairs(x.n_cols(), n_samples, rng, [](size_t, size_t) {});
    std::lock_guard<std::mutex> lock(cache().mu);
    xyzb_dataset* ds = cache().get(nullptr, x.values().data(), x.n_rows(), x.n_cols());
    xyzb_response resp{};
    resp.y_real = y.data();
    return device_strengths(ds, resp, XYZB_MODE_CONTINUOUS_XY,
                            transform == BinarizeTransform::unbiased ? XYZB_TRANSFORM_UNBIASED : XYZB_TRANSFORM_SIGN,
                            jk);
}

// ---- the three entry points (search.cpp:325-506) on the GPU ----

SearchReport xyz_search(const PackedMatrix& x, std::span<const std::int8_t> y, const SearchConfig& config) {
    config.validate();
    if (config.mode != SearchMode::binary) throw data_error("xyz_search: packed X with sign Y requires binary mode");
    if (y.size() != x.n_rows()) throw data_error("xyz_search: response length mismatch");
    for (const std::int8_t v : y)
        if (v != 1 && v != -1) throw data_error("xyz_search: binary response must be +-1");
    xyzb_response resp{};
    resp.y_sign = y.data();
    return run_gpu(x.column_words(0).data(), nullptr, x.n_rows(), x.n_cols(), resp, config);
}

SearchReport xyz_search(const PackedMatrix& x, const RealVector& y, const SearchConfig& config) {
    config.validate();
    if (config.mode != SearchMode::continuous_y)
        throw data_error("xyz_search: packed X with real Y requires continuous-Y mode");
    if (y.size() != x.n_rows()) throw data_error("xyz_search: response length mismatch");
    if (abs_sum(y) <= 0.0) throw data_error("xyz_search: zero response vector");
    xyzb_response resp{};
    resp.y_real = y.data();
    return run_gpu(x.column_words(0).data(), nullptr, x.n_rows(), x.n_cols(), resp, config);
}

SearchReport xyz_search(const RealMatrix& x, const RealVector& y, const SearchConfig& config) {
    config.validate();
    if (config.mode != SearchMode::continuous_xy) throw data_error("xyz_search: real X requires continuous-XY mode");
    if (y.size() != x.n_rows()) throw data_error("xyz_search: response length mismatch");
    if (abs_sum(y) <= 0.0) throw data_error("xyz_search: zero response vector");
    // the [-1, 1] range the unbiased transform needs (search.cpp:417-434) is checked by the engine
    // against the resident matrix (set once per upload; same message) instead of a host scan of X
    // on every call (the Lasso screens one 160 MB matrix ~50 times)
    xyzb_response resp{};
    resp.y_real = y.data();
    return run_gpu(nullptr, x.values().data(), x.n_rows(), x.n_cols(), resp, config);
}

} // namespace xyz
