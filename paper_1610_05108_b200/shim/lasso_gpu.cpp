// GPU drop-in for the xyz-regression loop: xyz::lasso_path
// (lasso.cpp:447-597) and xyz::kkt_check_interactions (lasso.cpp:377-426).
//
// The reference's loop alternates a host coordinate-descent solve over the
// active set with three exact scans of the residual: every main column
// (p centered dot products per active-set iteration), every square term
// (continuous designs), and the re-verification of each candidate the xyz
// screen returns. Here the scans run on the GPU against a device-resident
// copy of X (xyzb_design_*: one upload per call, the column means taken from
// the caller's CenteredDesignView), the screen runs on the GPU through the
// xyz_search shim, and the solver, the lambda grid and the exhaustive
// certificate are the reference's own functions (active_set_solve,
// exhaustive_kkt_max_correlation, lasso.o unchanged; the automatic lambda
// grid's correlations also run on the device, lambda_grid). The
// reference's definitions of these two entry points are weak symbols in the
// drop-in build (objcopy --weaken-symbol, shim/Makefile), so this file
// replaces them at link time without touching the reference sources.
//
// Parity: the same active sets, screens (gamma_lambda, sample streams, M, L,
// guard) and solver calls as the reference; the scans' fp64 sums are taken in
// a different order, so correlations agree to a few ulps and the path's
// coefficients to the solver's tolerance (tests/test_dropin.py).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "xyz/errors.hpp"
#include "xyz/lasso.hpp"
#include "xyz/rng.hpp"
#include "xyz/search.hpp"
#include "xyz/transforms.hpp"
#include "xyzb.h"
#include "devices.hpp"

namespace xyz {
namespace {

[[noreturn]] void rethrow_design(int code, const char* msg) {
    if (code == XYZB_E_DATA) throw data_error(msg);
    if (code == XYZB_E_SOLVER) throw solver_error(msg);
    throw std::runtime_error(std::string("xyz GPU engine: ") + msg);
}

bool entries_are_pm1(const RealMatrix& x) {
    return std::all_of(x.values().begin(), x.values().end(), [](double v) { return v == 1.0 || v == -1.0; });
}

// X on the device with the view's column means; the exact scans of the loop.
class DeviceScans {
public:
    DeviceScans(const RealMatrix& x, const CenteredDesignView& view) : n_(x.n_rows()), p_(x.n_cols()) {
        std::vector<double> means(p_);
        for (std::size_t j = 0; j < p_; ++j) means[j] = view.column_mean(j);
        char err[1024] = {0};
        const int code =
            xyzb_design_create(x.values().data(), n_, p_, means.data(), gpu_devices()[0], &d_, err, sizeof err);
        if (code != XYZB_OK) rethrow_design(code, err);
    }
    ~DeviceScans() { xyzb_design_destroy(d_); }
    DeviceScans(const DeviceScans&) = delete;
    DeviceScans& operator=(const DeviceScans&) = delete;

    // |main_correlation(j, r)| / n for every column j
    std::vector<double> mains(const RealVector& r) const {
        std::vector<double> out(p_);
        char err[1024] = {0};
        const int code = xyzb_design_main_correlations(d_, r.data(), out.data(), err, sizeof err);
        if (code != XYZB_OK) rethrow_design(code, err);
        for (double& v : out) v = std::abs(v) / static_cast<double>(n_);
        return out;
    }
    // |pair_correlation(key, r)| / n for every key
    std::vector<double> pairs(const RealVector& r, const std::vector<PairKey>& keys) const {
        std::vector<double> out(keys.size());
        if (keys.empty()) return out;
        static_assert(sizeof(PairKey) == 8, "PairKey is two u32");
        char err[1024] = {0};
        const int code = xyzb_design_pair_correlations(d_, r.data(), reinterpret_cast<const uint32_t*>(keys.data()),
                                                       keys.size(), out.data(), err, sizeof err);
        if (code != XYZB_OK) rethrow_design(code, err);
        for (double& v : out) v = std::abs(v) / static_cast<double>(n_);
        return out;
    }

private:
    std::size_t n_, p_;
    xyzb_design* d_ = nullptr;
};

// The KKT screen of the raw product columns (InteractionScreener,
// lasso.cpp:114-215): binary designs search the packed matrix against the
// residual (continuous-Y); continuous designs are row-rescaled once so the
// unbiased transform applies (the response picks up nu_i^2).
class ProductScreen {
public:
    ProductScreen(const RealMatrix& x, const LassoPathConfig& config)
        : x_(x), config_(config), binary_(entries_are_pm1(x)) {
        const std::size_t n = x.n_rows(), p = x.n_cols();
        if (binary_) {
            packed_ = PackedMatrix(n, p);
            for (std::size_t j = 0; j < p; ++j) {
                const auto col = x.column(j);
                for (std::size_t i = 0; i < n; ++i) packed_.set(i, j, col[i] > 0.0 ? +1 : -1);
            }
            return;
        }
        rescaled_ = rescale_rows(x, RealVector(n, 0.0)).first;
        std::vector<double> row_max(n, 0.0);
        for (std::size_t j = 0; j < p; ++j) {
            const auto col = x.column(j);
            for (std::size_t i = 0; i < n; ++i) row_max[i] = std::max(row_max[i], std::abs(col[i]));
        }
        nu_sq_.resize(n);
        for (std::size_t i = 0; i < n; ++i) nu_sq_[i] = row_max[i] * row_max[i];
    }

    // Pairs whose raw product correlation may exceed `threshold`; sets
    // `degenerate` when the strength threshold collapses to 1/2.
    std::vector<PairKey> candidates(const RealVector& residual, double threshold, std::uint64_t stream,
                                    bool& degenerate) const {
        degenerate = false;
        const std::size_t n = x_.n_rows(), p = x_.n_cols();
        RealVector response(residual);
        if (!binary_)
            for (std::size_t i = 0; i < n; ++i) response[i] = residual[i] * nu_sq_[i];
        double l1 = 0.0;
        for (const double v : response) l1 += std::abs(v);
        if (l1 <= 0.0) return {};
        const double gamma = 0.5 + static_cast<double>(n) * threshold / (2.0 * l1);
        if (gamma >= 1.0) return {};
        if (gamma <= 0.5) {
            degenerate = true;
            return {};
        }
        std::mt19937_64 sample_rng = make_stream(config_.seed ^ 0x6b, stream);
        SearchConfig s;
        s.gamma = gamma;
        s.search_negatives = true;
        std::uint64_t st = config_.seed ^ (stream * 0x9e3779b97f4a7c15ULL);
        s.seed = splitmix64(st);
        s.estimate_complexity = false;
        s.threads = config_.threads;
        s.max_candidates_per_rep = config_.kkt_max_candidates ? config_.kkt_max_candidates
                                                              : std::numeric_limits<std::uint64_t>::max();
        const StrengthSample sample =
            binary_ ? sample_strengths(packed_, std::span<const double>(response), config_.kkt_strength_sample,
                                       sample_rng)
                    : sample_strengths(rescaled_, response, BinarizeTransform::unbiased, config_.kkt_strength_sample,
                                       sample_rng);
        s.m = optimal_m(gamma, sample, n, p).m;
        if (config_.kkt_l)
            s.l = *config_.kkt_l;
        else if (config_.kkt_eta > 0.0)
            s.l = choose_l(s.m, gamma, config_.kkt_eta);
        else
            s.l = static_cast<std::size_t>(std::ceil(std::sqrt(static_cast<double>(p))));
        SearchReport rep;
        if (binary_) {
            s.mode = SearchMode::continuous_y;
            rep = xyz_search(packed_, response, s);
        } else {
            s.mode = SearchMode::continuous_xy;
            s.transform = BinarizeTransform::unbiased;
            rep = xyz_search(rescaled_, response, s);
        }
        // distinct unordered pairs in ascending order (an unguarded screen returns millions)
        std::vector<PairKey> keys;
        keys.reserve(rep.hits.size());
        for (const InteractionHit& h : rep.hits) keys.push_back(make_pair_key(h.j, h.k));
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        return keys;
    }

private:
    const RealMatrix& x_;
    LassoPathConfig config_;
    bool binary_;
    PackedMatrix packed_;
    RealMatrix rescaled_;
    RealVector nu_sq_;
};

// XYZB_LASSO_STATS=1: where lasso_path's time goes (printed per call).
struct LassoStats {
    using clock = std::chrono::steady_clock;
    double solve = 0, scans = 0, screen = 0, setup = 0;
    clock::time_point t = clock::now();
    double lap() {
        const auto now = clock::now();
        const double d = std::chrono::duration<double>(now - t).count();
        t = now;
        return d;
    }
};

std::vector<PairKey> all_off_diagonal(std::size_t p) {
    std::vector<PairKey> out;
    out.reserve(p * (p - 1) / 2);
    for (std::uint32_t j = 0; j + 1 < p; ++j)
        for (std::uint32_t k = j + 1; k < p; ++k) out.push_back({j, k});
    return out;
}

// auto_lambda_grid (lasso.cpp:232-268) with its correlations on the device:
// lambda_1 = the largest |centered correlation| / n of a main column or of an
// interaction column with centered y (every pair for p <= 512, else the
// reference's sample of min(1e5, 10p) pairs drawn from make_stream(seed,
// 0xa117)), then t log-spaced values down to ratio * lambda_1.
std::vector<double> lambda_grid(const RealMatrix& x, const RealVector& y, std::size_t t, double ratio,
                                std::uint64_t seed, bool binary, const DeviceScans& gpu) {
    if (t < 2) throw data_error("auto_lambda_grid: grid size must be >= 2");
    if (!(ratio > 0.0 && ratio < 1.0)) throw data_error("auto_lambda_grid: ratio must lie in (0,1)");
    if (y.size() != x.n_rows()) throw data_error("auto_lambda_grid: response length mismatch");
    const std::size_t p = x.n_cols();
    RealVector yc(y);
    double ysum = 0.0;
    for (const double v : yc) ysum += v;
    const double ybar = ysum / static_cast<double>(yc.size());
    double yvar = 0.0;
    for (double& v : yc) {
        v -= ybar;
        yvar += v * v;
    }
    if (yvar <= 0.0) throw data_error("auto_lambda_grid: response has zero variance");
    std::vector<PairKey> keys;
    if (p <= 512) {
        for (std::uint32_t j = 0; j < p; ++j)
            for (std::uint32_t k = j; k < p; ++k)
                if (!(binary && j == k)) keys.push_back({j, k});
    } else {
        std::mt19937_64 rng = make_stream(seed, 0xa117);
        std::uniform_int_distribution<std::uint32_t> dist(0, static_cast<std::uint32_t>(p - 1));
        const std::size_t samples = std::min<std::size_t>(100000, 10 * p);
        keys.reserve(samples);
        for (std::size_t s = 0; s < samples; ++s) {
            const std::uint32_t j = dist(rng), k = dist(rng);
            if (binary && j == k) continue;
            keys.push_back(make_pair_key(j, k));
        }
    }
    double lmax = 0.0;  // max(|corr| / n) == max(|corr|) / n: division is monotonic
    for (const double v : gpu.mains(yc)) lmax = std::max(lmax, v);
    for (const double v : gpu.pairs(yc, keys)) lmax = std::max(lmax, v);
    std::vector<double> grid(t);
    for (std::size_t i = 0; i < t; ++i)
        grid[i] = lmax * std::pow(ratio, static_cast<double>(i) / static_cast<double>(t - 1));
    return grid;
}

} // namespace

std::vector<PairKey> kkt_check_interactions(const RealVector& residual, const RealMatrix& x, double lambda,
                                            const LassoPathConfig& config, std::uint64_t seed_stream) {
    if (residual.size() != x.n_rows()) throw data_error("kkt_check_interactions: residual length mismatch");
    double l1 = 0.0;
    for (const double v : residual) l1 += std::abs(v);
    if (l1 <= 0.0) return {};
    const CenteredDesignView view(x);
    const DeviceScans gpu(x, view);
    const double threshold = lambda * config.interaction_penalty;
    // the screen runs on raw products: lower its level by the centering
    // correction 2 mu_max max_j |r^T Xc_j| / n
    const std::vector<double> mains = gpu.mains(residual);
    const double max_main = mains.empty() ? 0.0 : *std::max_element(mains.begin(), mains.end());
    const double screen_threshold = threshold - 2.0 * view.max_abs_column_mean() * max_main;
    const ProductScreen screen(x, config);
    bool degenerate = screen_threshold <= 0.0;
    std::vector<PairKey> cand;
    if (!degenerate) cand = screen.candidates(residual, screen_threshold, seed_stream, degenerate);
    if (degenerate) {
        if (x.n_cols() > 2000)
            throw solver_error(
                "kkt_check_interactions: threshold too small for probabilistic screening "
                "and p too large for the exact fallback");
        cand = all_off_diagonal(x.n_cols());
    }
    const std::vector<double> corr = gpu.pairs(residual, cand);
    std::vector<PairKey> violations;
    for (std::size_t t = 0; t < cand.size(); ++t)
        if (corr[t] > threshold) violations.push_back(cand[t]);
    std::sort(violations.begin(), violations.end());
    return violations;
}

std::vector<SparseFit> lasso_path(const RealMatrix& x, const RealVector& y, const LassoPathConfig& config_in) {
    if (y.size() != x.n_rows()) throw data_error("lasso_path: response length mismatch");
    const std::size_t n = x.n_rows(), p = x.n_cols();
    LassoPathConfig config = config_in;
    const bool binary = entries_are_pm1(x);
    if (binary) config.exclude_diagonal = true;  // no square terms for +-1 data

    RealVector yc(y);
    double ysum = 0.0;
    for (const double v : yc) ysum += v;
    const double ybar = ysum / static_cast<double>(yc.size());
    for (double& v : yc) v -= ybar;

    LassoStats st;
    const CenteredDesignView view(x);
    const DeviceScans gpu(x, view);
    std::vector<double> lambdas = config.lambdas;
    if (lambdas.empty()) {
        lambdas = lambda_grid(x, y, config.grid_size, config.grid_ratio, config.seed, binary, gpu);
    } else {
        for (std::size_t i = 0; i < lambdas.size(); ++i)
            if (!(lambdas[i] > 0.0) || !(i == 0 || lambdas[i - 1] > lambdas[i]))
                throw data_error("lasso_path: lambda grid must be strictly decreasing and positive");
    }

    const ProductScreen screen(x, config);
    st.setup += st.lap();
    std::vector<PairKey> squares;
    if (!config.exclude_diagonal) {
        squares.resize(p);
        for (std::uint32_t j = 0; j < p; ++j) squares[j] = {j, j};
    }

    std::vector<SparseFit> path;
    std::vector<std::uint32_t> active_main;
    std::vector<PairKey> active_pairs;
    std::vector<char> in_main(p, 0);
    std::set<PairKey> in_pairs;
    SparseFit warm;
    bool have_warm = false;

    for (std::size_t li = 0; li < lambdas.size(); ++li) {
        const double lambda = lambdas[li];
        const double pair_threshold = lambda * config.interaction_penalty;
        if (have_warm) {  // warm start: the previous solution's support
            active_main.clear();
            active_pairs.clear();
            for (const auto& kv : warm.beta) active_main.push_back(kv.first);
            for (const auto& kv : warm.theta) active_pairs.push_back(kv.first);
        }
        std::fill(in_main.begin(), in_main.end(), 0);
        for (const std::uint32_t j : active_main) in_main[j] = 1;
        in_pairs.clear();
        in_pairs.insert(active_pairs.begin(), active_pairs.end());

        ActiveSetResult solved;
        bool degenerate_seen = false;
        std::size_t iterations = 0;
        double kkt_max = -std::numeric_limits<double>::infinity();
        for (bool closed = false; !closed;) {
            if (iterations >= config.max_active_set_iterations)
                throw solver_error("lasso_path: active set did not close at lambda index " + std::to_string(li));
            ++iterations;
            st.lap();
            solved = active_set_solve(view, active_main, active_pairs, yc, lambda, config,
                                      have_warm || iterations > 1 ? &warm : nullptr);
            warm = solved.fit;
            have_warm = true;
            st.solve += st.lap();

            // exact main-effect sweep (device)
            kkt_max = -std::numeric_limits<double>::infinity();
            const std::vector<double> mc = gpu.mains(solved.residual);
            std::vector<std::uint32_t> add_main;
            double max_main = 0.0;
            for (std::uint32_t j = 0; j < p; ++j) {
                max_main = std::max(max_main, mc[j]);
                kkt_max = std::max(kkt_max, mc[j] - lambda);
                if (mc[j] > lambda && !in_main[j]) add_main.push_back(j);
            }
            // square terms, exact (device); none for binary designs
            std::vector<PairKey> add_pairs;
            if (!squares.empty()) {
                const std::vector<double> sc = gpu.pairs(solved.residual, squares);
                for (std::size_t j = 0; j < p; ++j) {
                    kkt_max = std::max(kkt_max, sc[j] - pair_threshold);
                    if (sc[j] > pair_threshold && !in_pairs.count(squares[j])) add_pairs.push_back(squares[j]);
                }
            }
            // off-diagonal pairs: xyz screen (device) + exact re-verification (device)
            const double screen_threshold = pair_threshold - 2.0 * view.max_abs_column_mean() * max_main;
            bool degenerate = screen_threshold <= 0.0;
            std::vector<PairKey> cand;
            st.scans += st.lap();
            if (!degenerate)
                cand = screen.candidates(solved.residual, screen_threshold,
                                         li * config.max_active_set_iterations + iterations, degenerate);
            st.screen += st.lap();
            if (degenerate) {
                degenerate_seen = true;
                if (p > 2000)
                    throw solver_error("lasso_path: degenerate screening threshold at lambda index " +
                                       std::to_string(li) + " with p too large for exact fallback");
                cand = all_off_diagonal(p);
            }
            const std::vector<double> pc = gpu.pairs(solved.residual, cand);
            for (std::size_t t = 0; t < cand.size(); ++t) {
                kkt_max = std::max(kkt_max, pc[t] - pair_threshold);
                if (pc[t] > pair_threshold && !in_pairs.count(cand[t])) add_pairs.push_back(cand[t]);
            }

            if (add_main.empty() && add_pairs.empty()) {
                closed = true;
            } else {
                for (const std::uint32_t j : add_main) {
                    active_main.push_back(j);
                    in_main[j] = 1;
                }
                std::sort(add_pairs.begin(), add_pairs.end());
                add_pairs.erase(std::unique(add_pairs.begin(), add_pairs.end()), add_pairs.end());
                for (const PairKey& k : add_pairs) {
                    active_pairs.push_back(k);
                    in_pairs.insert(k);
                }
            }
        }

        SparseFit fit = solved.fit;
        fit.active_set_iterations = iterations;
        fit.kkt_residual_max = kkt_max;
        fit.screening_degenerate = degenerate_seen;
        if (config.certify_exhaustive && p <= config.certify_max_p) {
            const double worst = exhaustive_kkt_max_correlation(view, solved.residual, config.interaction_penalty,
                                                                config.exclude_diagonal);
            fit.certified_exhaustive = worst <= lambda * (1.0 + 1e-6);
        }
        path.push_back(fit);
        warm = path.back();
        st.scans += st.lap();
    }
    if (std::getenv("XYZB_LASSO_STATS"))
        std::fprintf(stderr, "[lasso_path gpu] setup %.3f s, solve %.3f s, scans %.3f s, screens %.3f s\n", st.setup,
                     st.solve, st.scans, st.screen);
    return path;
}

} // namespace xyz
