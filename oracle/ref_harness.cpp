// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// extern "C" harness around the UNMODIFIED reference core, compiled from the
// sources where they lie under /root/reference/proj/core (see oracle/Makefile)
// into oracle/_ref/libxyzref.so. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it: as the checker and
// as the reference CPU arm, never as part of the product path.
//
// The signatures reuse the plain structs of include/xyzb.h so that the
// product (libxyzb.so), the restatement (oracle/liboracle.so) and the
// reference are driven by the same arguments.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "xyz/dataset_io.hpp"
#include "xyz/errors.hpp"
#include "xyz/lasso.hpp"
#include "xyz/oracle.hpp"
#include "xyz/pair_search.hpp"
#include "xyz/projection.hpp"
#include "xyz/rng.hpp"
#include "xyz/search.hpp"
#include "xyz/synthetic.hpp"
#include "xyz/transforms.hpp"
#include "xyzb.h"

namespace {

void set_err(char* err, size_t errlen, const std::string& msg) {
    if (err == nullptr || errlen == 0) return;
    std::snprintf(err, errlen, "%s", msg.c_str());
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        return XYZB_OK;
    } catch (const xyz::data_error& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_DATA;
    } catch (const xyz::guard_error& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_GUARD;
    } catch (const xyz::solver_error& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_SOLVER;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_INTERNAL;
    }
}

xyz::PackedMatrix packed_from_words(const uint64_t* words, size_t n, size_t p) {
    xyz::PackedMatrix x(n, p);
    const size_t wpc = x.words_per_col();
    for (size_t j = 0; j < p; ++j) {
        auto col = x.column_words(j);
        std::memcpy(col.data(), words + j * wpc, wpc * sizeof(uint64_t));
    }
    return x;
}

xyz::RealMatrix real_from_colmajor(const double* v, size_t n, size_t p) {
    xyz::RealMatrix x(n, p);
    for (size_t j = 0; j < p; ++j) {
        auto col = x.column(j);
        std::memcpy(col.data(), v + j * n, n * sizeof(double));
    }
    return x;
}

xyz::SearchConfig config_from(const xyzb_params* q) {
    xyz::SearchConfig c;
    c.m = q->m;
    c.l = q->l;
    c.gamma = q->gamma;
    c.mode = static_cast<xyz::SearchMode>(q->mode);
    c.transform = static_cast<xyz::BinarizeTransform>(q->transform);
    c.search_negatives = q->search_negatives != 0;
    c.seed = q->seed;
    c.max_candidates_per_rep = q->max_candidates_per_rep;
    c.stop_after_first_hit = q->stop_after_first_hit != 0;
    c.estimate_complexity = q->estimate_complexity != 0;
    c.threads = static_cast<unsigned>(q->threads);
    c.strength_sample_size = q->strength_sample_size;
    return c;
}

// Top-K by the oracle comparator (oracle.cpp:47-51) extended with the sign
// (SURVEY Appendix A.10): strength desc, min asc, max asc, sign desc.
void fill_topk(const std::vector<xyz::InteractionHit>& hits, uint64_t k, xyzb_result* out) {
    out->top_k = nullptr;
    out->n_top_k = 0;
    if (k == 0) return;
    std::vector<uint64_t> idx(hits.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
        const auto& x = hits[a];
        const auto& y = hits[b];
        if (x.strength != y.strength) return x.strength > y.strength;
        const uint32_t xl = std::min(x.j, x.k), xh = std::max(x.j, x.k);
        const uint32_t yl = std::min(y.j, y.k), yh = std::max(y.j, y.k);
        if (xl != yl) return xl < yl;
        if (xh != yh) return xh < yh;
        return x.sign > y.sign;
    });
    const size_t kk = std::min<size_t>(k, idx.size());
    out->n_top_k = kk;
    out->top_k = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, kk) * sizeof(uint64_t)));
    for (size_t i = 0; i < kk; ++i) out->top_k[i] = idx[i];
}

void fill_result(const xyz::SearchReport& r, uint64_t top_k, xyzb_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->n_hits = r.hits.size();
    out->hits = static_cast<xyzb_hit*>(std::malloc(std::max<size_t>(1, r.hits.size()) * sizeof(xyzb_hit)));
    for (size_t i = 0; i < r.hits.size(); ++i) {
        out->hits[i].j = r.hits[i].j;
        out->hits[i].k = r.hits[i].k;
        out->hits[i].strength = r.hits[i].strength;
        out->hits[i].found_at_repetition = r.hits[i].found_at_repetition;
        out->hits[i].sign = r.hits[i].sign;
    }
    out->repetitions_run = r.repetitions_run;
    out->candidates_checked = r.candidates_checked;
    out->candidates_enumerated = r.candidates_enumerated;
    out->aborted_repetitions = r.aborted_repetitions;
    out->wall_time_s = r.wall_time_s;
    out->estimated_c = r.estimated_c;
    out->gamma0 = r.gamma0;
    out->m_used = r.m_used;
    out->l_used = r.l_used;
    out->runs_executed = r.repetitions_run;
    fill_topk(r.hits, top_k, out);
}

} // namespace

extern "C" {

int ref_abi_version(void) { return XYZB_ABI_VERSION; }

// xyz::xyz_search, all three overloads (search.cpp:325,367,415).
int ref_search(const xyzb_problem* prob, const xyzb_response* resp, const xyzb_params* params,
               xyzb_result* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const xyz::SearchConfig cfg = config_from(params);
        const size_t n = prob->n_rows, p = prob->n_cols;
        xyz::SearchReport report;
        if (params->mode == XYZB_MODE_CONTINUOUS_XY) {
            if (prob->x_real == nullptr || resp->y_real == nullptr)
                throw xyz::data_error("ref_search: continuous-XY needs x_real and y_real");
            const xyz::RealMatrix x = real_from_colmajor(prob->x_real, n, p);
            const xyz::RealVector y(resp->y_real, resp->y_real + n);
            report = xyz::xyz_search(x, y, cfg);
        } else if (params->mode == XYZB_MODE_CONTINUOUS_Y) {
            if (prob->x_words == nullptr || resp->y_real == nullptr)
                throw xyz::data_error("ref_search: continuous-Y needs x_words and y_real");
            const xyz::PackedMatrix x = packed_from_words(prob->x_words, n, p);
            const xyz::RealVector y(resp->y_real, resp->y_real + n);
            report = xyz::xyz_search(x, y, cfg);
        } else {
            if (prob->x_words == nullptr || resp->y_sign == nullptr)
                throw xyz::data_error("ref_search: binary mode needs x_words and y_sign");
            const xyz::PackedMatrix x = packed_from_words(prob->x_words, n, p);
            report = xyz::xyz_search(x, std::span<const std::int8_t>(resp->y_sign, n), cfg);
        }
        fill_result(report, params->top_k, out);
    });
}

void ref_result_free(xyzb_result* r) {
    if (r == nullptr) return;
    std::free(r->hits);
    std::free(r->top_k);
    std::free(r->order_keys);
    r->hits = nullptr;
    r->top_k = nullptr;
    r->order_keys = nullptr;
}

void ref_free(void* p) { std::free(p); }

// draw_subsample (projection.cpp:12-30) on stream make_stream(seed, stream);
// weighted when y != NULL (WeightedSampler::from_magnitudes, real_matrix.cpp:36-54).
int ref_draw_subsample(uint64_t n, uint64_t m, uint64_t seed, uint64_t stream, const double* y,
                       uint64_t* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::mt19937_64 rng = xyz::make_stream(seed, stream);
        xyz::SubsampleDraw d;
        if (y != nullptr) {
            const auto w = xyz::WeightedSampler::from_magnitudes(std::span<const double>(y, n));
            d = xyz::draw_subsample(n, m, &w, rng);
        } else {
            d = xyz::draw_subsample(n, m, nullptr, rng);
        }
        for (size_t s = 0; s < m; ++s) out[s] = d.indices[s];
    });
}

// project_keys (projection.cpp:32-57) for explicit draws.
int ref_project_keys(const uint64_t* x_words, uint64_t n, uint64_t p, const uint64_t* draw,
                     uint64_t m, uint64_t* keys, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const xyz::PackedMatrix x = packed_from_words(x_words, n, p);
        xyz::SubsampleDraw d;
        d.indices.assign(draw, draw + m);
        const auto k = xyz::project_keys(x, d);
        for (size_t j = 0; j < p; ++j) keys[j] = k[j].key;
    });
}

// build_z (transforms.cpp:13-31)
int ref_build_z(const uint64_t* x_words, uint64_t n, uint64_t p, const int8_t* y,
                uint64_t* z_words, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const xyz::PackedMatrix x = packed_from_words(x_words, n, p);
        const xyz::PackedMatrix z = xyz::build_z(x, std::span<const std::int8_t>(y, n));
        const size_t wpc = z.words_per_col();
        for (size_t j = 0; j < p; ++j) {
            const auto c = z.column_words(j);
            std::memcpy(z_words + j * wpc, c.data(), wpc * sizeof(uint64_t));
        }
    });
}

// equal_pairs (pair_search.cpp:26-55), enumerated in filter order
// (pair_search.hpp:95-97): blocks by key, j asc, k asc.
int ref_equal_pairs(const uint64_t* x_keys, const uint64_t* z_keys, uint64_t p,
                    uint32_t** pairs_jk, uint64_t* n_pairs, uint64_t* total_pairs,
                    char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<xyz::ProjectionKey> xk(p), zk(p);
        for (uint32_t i = 0; i < p; ++i) {
            xk[i] = {i, x_keys[i]};
            zk[i] = {i, z_keys[i]};
        }
        const xyz::CandidatePairSet s = xyz::equal_pairs(xk, zk);
        std::vector<uint32_t> flat;
        for (const auto& b : s.groups)
            for (uint32_t j : b.x_indices)
                for (uint32_t k : b.z_indices) {
                    flat.push_back(j);
                    flat.push_back(k);
                }
        *n_pairs = flat.size() / 2;
        *total_pairs = s.total_pairs;
        *pairs_jk = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, flat.size()) * sizeof(uint32_t)));
        std::copy(flat.begin(), flat.end(), *pairs_jk);
    });
}

// interaction_strength (transforms.cpp:33-40) of pair (j,k) as the pass-+1
// strength function calls it (search.cpp:347-349): agreements(Z_k, X_j)/n.
int ref_pair_strengths(const xyzb_problem* prob, const xyzb_response* resp, int32_t mode,
                       int32_t transform, const uint32_t* pairs_jk, uint64_t n_pairs,
                       double* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const size_t n = prob->n_rows, p = prob->n_cols;
        if (mode == XYZB_MODE_BINARY) {
            const xyz::PackedMatrix x = packed_from_words(prob->x_words, n, p);
            const xyz::PackedMatrix z = xyz::build_z(x, std::span<const std::int8_t>(resp->y_sign, n));
            for (size_t t = 0; t < n_pairs; ++t)
                out[t] = xyz::interaction_strength(x, z, pairs_jk[2 * t + 1], pairs_jk[2 * t]);
        } else if (mode == XYZB_MODE_CONTINUOUS_Y) {
            const xyz::PackedMatrix x = packed_from_words(prob->x_words, n, p);
            const std::span<const double> y(resp->y_real, n);
            for (size_t t = 0; t < n_pairs; ++t)
                out[t] = xyz::weighted_interaction_strength(x, y, pairs_jk[2 * t], pairs_jk[2 * t + 1]);
        } else {
            // continuous-XY strength (search.cpp:477-493), sign +1
            const double* xv = prob->x_real;
            const double* y = resp->y_real;
            double norm = 0.0;
            for (size_t i = 0; i < n; ++i) norm += std::abs(y[i]);
            for (size_t t = 0; t < n_pairs; ++t) {
                const double* cj = xv + size_t(pairs_jk[2 * t]) * n;
                const double* ck = xv + size_t(pairs_jk[2 * t + 1]) * n;
                double acc = 0.0;
                if (transform == XYZB_TRANSFORM_UNBIASED) {
                    for (size_t i = 0; i < n; ++i) acc += y[i] * cj[i] * ck[i];
                } else {
                    for (size_t i = 0; i < n; ++i) {
                        const double tj = cj[i] > 0.0 ? 1.0 : (cj[i] < 0.0 ? -1.0 : 0.0);
                        const double tk = ck[i] > 0.0 ? 1.0 : (ck[i] < 0.0 ? -1.0 : 0.0);
                        acc += y[i] * tj * tk;
                    }
                }
                out[t] = 0.5 + acc / (2.0 * norm);
            }
        }
    });
}

// xyz::sample_strengths, the overload of `mode` (search.cpp:229-291), on
// make_stream(seed, stream) — binary: Z = build_z(X, y_sign) as the CLI's
// auto-M sample builds it (xyz_main.cpp:142-149) — and optimal_m(gamma, ...)
// over the sample (search.cpp:189-220). In the drop-in build these resolve to
// the GPU shim's sample_strengths.
int ref_sample_strengths(const xyzb_problem* prob, const xyzb_response* resp, int32_t mode, int32_t transform,
                         uint64_t n_samples, uint64_t seed, uint64_t stream, double gamma, double* out,
                         uint64_t* m_out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const size_t n = prob->n_rows, p = prob->n_cols;
        std::mt19937_64 rng = xyz::make_stream(seed, stream);
        xyz::StrengthSample s;
        if (mode == XYZB_MODE_BINARY) {
            const xyz::PackedMatrix x = packed_from_words(prob->x_words, n, p);
            const xyz::PackedMatrix z = xyz::build_z(x, std::span<const std::int8_t>(resp->y_sign, n));
            s = xyz::sample_strengths(x, z, n_samples, rng);
        } else if (mode == XYZB_MODE_CONTINUOUS_Y) {
            const xyz::PackedMatrix x = packed_from_words(prob->x_words, n, p);
            s = xyz::sample_strengths(x, std::span<const double>(resp->y_real, n), n_samples, rng);
        } else {
            const xyz::RealMatrix x = real_from_colmajor(prob->x_real, n, p);
            const xyz::RealVector y(resp->y_real, resp->y_real + n);
            s = xyz::sample_strengths(x, y,
                                      transform == XYZB_TRANSFORM_UNBIASED ? xyz::BinarizeTransform::unbiased
                                                                           : xyz::BinarizeTransform::sign,
                                      n_samples, rng);
        }
        std::copy(s.strengths.begin(), s.strengths.end(), out);
        *m_out = xyz::optimal_m(gamma, s, n, p).m;
    });
}

// ---- synthetic generators (synthetic.cpp:12-69), fixture generation only ----

int ref_rademacher_matrix(uint64_t n, uint64_t p, uint64_t seed, uint64_t stream,
                          uint64_t* x_words, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::mt19937_64 rng = xyz::make_stream(seed, stream);
        const xyz::PackedMatrix x = xyz::rademacher_matrix(n, p, rng);
        const size_t wpc = x.words_per_col();
        for (size_t j = 0; j < p; ++j)
            std::memcpy(x_words + j * wpc, x.column_words(j).data(), wpc * sizeof(uint64_t));
    });
}

// rademacher_matrix followed by plant_interaction on the same stream
// (the recipe of planted_binary_instance, synthetic.cpp:40-50, with (j,k) free).
int ref_planted_instance(uint64_t n, uint64_t p, uint64_t j, uint64_t k, double gamma,
                         uint64_t seed, uint64_t stream, uint64_t* x_words, int8_t* y,
                         char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::mt19937_64 rng = xyz::make_stream(seed, stream);
        const xyz::PackedMatrix x = xyz::rademacher_matrix(n, p, rng);
        const auto yy = xyz::plant_interaction(x, j, k, gamma, rng);
        const size_t wpc = x.words_per_col();
        for (size_t c = 0; c < p; ++c)
            std::memcpy(x_words + c * wpc, x.column_words(c).data(), wpc * sizeof(uint64_t));
        std::copy(yy.begin(), yy.end(), y);
    });
}

int ref_gaussian_matrix(uint64_t n, uint64_t p, uint64_t seed, uint64_t stream, double* out,
                        char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::mt19937_64 rng = xyz::make_stream(seed, stream);
        const xyz::RealMatrix x = xyz::gaussian_matrix(n, p, rng);
        std::copy(x.values().begin(), x.values().end(), out);
    });
}

int ref_uniform_matrix(uint64_t n, uint64_t p, uint64_t seed, uint64_t stream, double* out,
                       char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::mt19937_64 rng = xyz::make_stream(seed, stream);
        const xyz::RealMatrix x = xyz::uniform_matrix(n, p, rng);
        std::copy(x.values().begin(), x.values().end(), out);
    });
}

// brute_force_search top-k (oracle.cpp:24-59,84-91): pairs (j<k) re-sorted by (j,k).
int ref_brute_force_topk(const uint64_t* x_words, uint64_t n, uint64_t p, const int8_t* y,
                         uint64_t k, uint32_t* out_jk, double* out_s, uint64_t* n_out,
                         char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const xyz::PackedMatrix x = packed_from_words(x_words, n, p);
        xyz::oracle::BruteForceOptions o;
        o.top_k = k;
        o.force = true;
        const auto r = xyz::oracle::brute_force_search(x, std::span<const std::int8_t>(y, n), o);
        *n_out = r.pairs.size();
        for (size_t t = 0; t < r.pairs.size(); ++t) {
            out_jk[2 * t] = r.pairs[t].j;
            out_jk[2 * t + 1] = r.pairs[t].k;
            out_s[t] = r.pairs[t].strength;
        }
    });
}

// oracle::brute_force_search, binary overload (oracle.cpp:84-91), every
// option. Outputs malloc'ed (ref_free): out_jk [2 * n_out], out_s [n_out],
// out_hist [bins].
int ref_brute_force(const uint64_t* x_words, uint64_t n, uint64_t p, const int8_t* y, int32_t has_gamma,
                    double gamma, int32_t has_top_k, uint64_t top_k, uint64_t bins, int32_t force, uint32_t** out_jk,
                    double** out_s, uint64_t* n_out, uint64_t* scanned, uint64_t** out_hist, char* err,
                    size_t errlen) {
    *out_jk = nullptr;
    *out_s = nullptr;
    *out_hist = nullptr;
    return guarded(err, errlen, [&] {
        const xyz::PackedMatrix x = packed_from_words(x_words, n, p);
        xyz::oracle::BruteForceOptions o;
        if (has_gamma) o.gamma = gamma;
        if (has_top_k) o.top_k = top_k;
        o.histogram_bins = bins;
        o.force = force != 0;
        const auto r = xyz::oracle::brute_force_search(x, std::span<const std::int8_t>(y, n), o);
        *n_out = r.pairs.size();
        *scanned = r.pairs_scanned;
        *out_jk = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, 2 * r.pairs.size()) * 4));
        *out_s = static_cast<double*>(std::malloc(std::max<size_t>(1, r.pairs.size()) * 8));
        for (size_t t = 0; t < r.pairs.size(); ++t) {
            (*out_jk)[2 * t] = r.pairs[t].j;
            (*out_jk)[2 * t + 1] = r.pairs[t].k;
            (*out_s)[t] = r.pairs[t].strength;
        }
        *out_hist = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, r.histogram.size()) * 8));
        for (size_t t = 0; t < r.histogram.size(); ++t) (*out_hist)[t] = r.histogram[t];
    });
}

// oracle::brute_force_search, continuous-response overload (oracle.cpp:93-100).
int ref_brute_force_weighted(const uint64_t* x_words, uint64_t n, uint64_t p, const double* y, int32_t has_gamma,
                             double gamma, int32_t has_top_k, uint64_t top_k, uint64_t bins, int32_t force,
                             uint32_t** out_jk, double** out_s, uint64_t* n_out, uint64_t* scanned,
                             uint64_t** out_hist, char* err, size_t errlen) {
    *out_jk = nullptr;
    *out_s = nullptr;
    *out_hist = nullptr;
    return guarded(err, errlen, [&] {
        const xyz::PackedMatrix x = packed_from_words(x_words, n, p);
        xyz::oracle::BruteForceOptions o;
        if (has_gamma) o.gamma = gamma;
        if (has_top_k) o.top_k = top_k;
        o.histogram_bins = bins;
        o.force = force != 0;
        const auto r = xyz::oracle::brute_force_search(x, std::span<const double>(y, n), o);
        *n_out = r.pairs.size();
        *scanned = r.pairs_scanned;
        *out_jk = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, 2 * r.pairs.size()) * 4));
        *out_s = static_cast<double*>(std::malloc(std::max<size_t>(1, r.pairs.size()) * 8));
        for (size_t t = 0; t < r.pairs.size(); ++t) {
            (*out_jk)[2 * t] = r.pairs[t].j;
            (*out_jk)[2 * t + 1] = r.pairs[t].k;
            (*out_s)[t] = r.pairs[t].strength;
        }
        *out_hist = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, r.histogram.size()) * 8));
        for (size_t t = 0; t < r.histogram.size(); ++t) (*out_hist)[t] = r.histogram[t];
    });
}

// lasso_path (lasso.cpp:447-597) with the config fields the benchmarks pin.
// Output: per fit t, lambda[t], mains in [main_off[t], main_off[t+1]) of
// (main_idx, main_val), pairs in [pair_off[t], pair_off[t+1]) of (pair_j,
// pair_k, pair_val), and diagnostics. Arrays malloc'ed; free with ref_free.
struct ref_lasso_out {
    uint64_t n_fits;
    double* lambda;
    uint64_t* main_off;
    uint32_t* main_idx;
    double* main_val;
    uint64_t* pair_off;
    uint32_t* pair_j;
    uint32_t* pair_k;
    double* pair_val;
    double* kkt_residual_max;
    uint8_t* certified;
    uint8_t* degenerate;
    uint64_t* active_set_iterations;
    uint64_t* cd_cycles;
    double wall_s;
};

int ref_lasso_path(const double* x, uint64_t n, uint64_t p, const double* y, uint64_t grid_size, double grid_ratio,
                   uint64_t kkt_l, uint64_t kkt_max_candidates, uint64_t seed, uint32_t threads,
                   int32_t certify_exhaustive, ref_lasso_out* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const xyz::RealMatrix xm = real_from_colmajor(x, n, p);
        const xyz::RealVector yv(y, y + n);
        xyz::LassoPathConfig cfg;
        cfg.grid_size = grid_size;
        cfg.grid_ratio = grid_ratio;
        if (kkt_l) cfg.kkt_l = kkt_l;
        cfg.kkt_max_candidates = kkt_max_candidates;
        cfg.seed = seed;
        cfg.threads = threads;
        cfg.certify_exhaustive = certify_exhaustive != 0;
        const auto t0 = std::chrono::steady_clock::now();
        const auto fits = xyz::lasso_path(xm, yv, cfg);
        out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const size_t T = fits.size();
        size_t nm = 0, np = 0;
        for (const auto& f : fits) {
            nm += f.beta.size();
            np += f.theta.size();
        }
        auto al = [](size_t cnt, size_t sz) { return std::malloc(std::max<size_t>(1, cnt) * sz); };
        out->n_fits = T;
        out->lambda = static_cast<double*>(al(T, 8));
        out->main_off = static_cast<uint64_t*>(al(T + 1, 8));
        out->pair_off = static_cast<uint64_t*>(al(T + 1, 8));
        out->main_idx = static_cast<uint32_t*>(al(nm, 4));
        out->main_val = static_cast<double*>(al(nm, 8));
        out->pair_j = static_cast<uint32_t*>(al(np, 4));
        out->pair_k = static_cast<uint32_t*>(al(np, 4));
        out->pair_val = static_cast<double*>(al(np, 8));
        out->kkt_residual_max = static_cast<double*>(al(T, 8));
        out->certified = static_cast<uint8_t*>(al(T, 1));
        out->degenerate = static_cast<uint8_t*>(al(T, 1));
        out->active_set_iterations = static_cast<uint64_t*>(al(T, 8));
        out->cd_cycles = static_cast<uint64_t*>(al(T, 8));
        size_t mi = 0, pi = 0;
        for (size_t t = 0; t < T; ++t) {
            const auto& f = fits[t];
            out->lambda[t] = f.lambda;
            out->main_off[t] = mi;
            out->pair_off[t] = pi;
            for (const auto& [j, v] : f.beta) {
                out->main_idx[mi] = j;
                out->main_val[mi++] = v;
            }
            for (const auto& [key, v] : f.theta) {
                out->pair_j[pi] = key.j;
                out->pair_k[pi] = key.k;
                out->pair_val[pi++] = v;
            }
            out->kkt_residual_max[t] = f.kkt_residual_max;
            out->certified[t] = f.certified_exhaustive;
            out->degenerate[t] = f.screening_degenerate;
            out->active_set_iterations[t] = f.active_set_iterations;
            out->cd_cycles[t] = f.cd_cycles;
        }
        out->main_off[T] = mi;
        out->pair_off[T] = pi;
    });
}

void ref_lasso_free(ref_lasso_out* o) {
    if (!o) return;
    for (void* q : {static_cast<void*>(o->lambda), static_cast<void*>(o->main_off), static_cast<void*>(o->main_idx),
                    static_cast<void*>(o->main_val), static_cast<void*>(o->pair_off), static_cast<void*>(o->pair_j),
                    static_cast<void*>(o->pair_k), static_cast<void*>(o->pair_val),
                    static_cast<void*>(o->kkt_residual_max), static_cast<void*>(o->certified),
                    static_cast<void*>(o->degenerate), static_cast<void*>(o->active_set_iterations),
                    static_cast<void*>(o->cd_cycles)})
        std::free(q);
    std::memset(o, 0, sizeof(*o));
}

// kkt_check_interactions (lasso.cpp:377-426): sorted violating pairs as
// 2 * count column indices, malloc'ed (free with ref_free).
int ref_kkt_check_interactions(const double* x, uint64_t n, uint64_t p, const double* residual, double lambda,
                               uint64_t kkt_l, uint64_t kkt_max_candidates, uint64_t seed, uint64_t stream,
                               uint32_t threads, uint32_t** pairs_jk, uint64_t* count, char* err, size_t errlen) {
    *pairs_jk = nullptr;
    *count = 0;
    return guarded(err, errlen, [&] {
        const xyz::RealMatrix xm = real_from_colmajor(x, n, p);
        const xyz::RealVector r(residual, residual + n);
        xyz::LassoPathConfig cfg;
        if (kkt_l) cfg.kkt_l = kkt_l;
        cfg.kkt_max_candidates = kkt_max_candidates;
        cfg.seed = seed;
        cfg.threads = threads;
        const auto v = xyz::kkt_check_interactions(r, xm, lambda, cfg, stream);
        *pairs_jk = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, v.size()) * 8));
        for (size_t t = 0; t < v.size(); ++t) {
            (*pairs_jk)[2 * t] = v[t].j;
            (*pairs_jk)[2 * t + 1] = v[t].k;
        }
        *count = v.size();
    });
}

// write_dataset / read_dataset (dataset_io.cpp:65-129)
int ref_write_dataset(const char* path, int32_t kind, const uint64_t* x_words, const double* x_real, uint64_t n,
                      uint64_t p, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        xyz::Dataset d;
        d.kind = kind == 0 ? xyz::DatasetKind::binary : xyz::DatasetKind::real;
        if (kind == 0) d.packed = packed_from_words(x_words, n, p); else d.real = real_from_colmajor(x_real, n, p);
        xyz::write_dataset(path, d);
    });
}

int ref_read_dataset(const char* path, int32_t* kind, uint64_t* n, uint64_t* p, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const xyz::Dataset d = xyz::read_dataset(path);
        *kind = d.kind == xyz::DatasetKind::binary ? 0 : 1;
        *n = d.n_rows();
        *p = d.n_cols();
    });
}

// rescale_rows (transforms.cpp:116-135): X/nu and y*nu^2, column-major in place copies.
int ref_rescale_rows(const double* x, uint64_t n, uint64_t p, const double* y, double* x_out,
                     double* y_out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const xyz::RealMatrix xm = real_from_colmajor(x, n, p);
        const xyz::RealVector yv(y, y + n);
        const auto [xr, yr] = xyz::rescale_rows(xm, yv);
        std::copy(xr.values().begin(), xr.values().end(), x_out);
        std::copy(yr.begin(), yr.end(), y_out);
    });
}

} // extern "C"
