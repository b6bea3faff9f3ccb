// TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.
//
// CPU restatement of the reference's xyz search hot path (the parity contract
// of SURVEY.md Appendix A), written independently of the reference's code and
// of the CUDA engine:
//   * keys come from the XNOR/XOR algebra z+ = ~(x ^ y) & mask, z- = (x ^ y)
//     (transforms.cpp:26-28, search.cpp:32-33) instead of materialising Z;
//   * buckets are a std::map from key to column list instead of a sorted
//     KeyEntry array (pair_search.cpp:26-55);
//   * dedup is the first-occurrence rule of Appendix A.8 instead of the
//     seen-set / emitted-set pair (search.cpp:65-111);
//   * strengths are scalar loops over the bits (no word popcount).
// It is pinned against the compiled reference (oracle/_ref/libxyzref.so) by
// the golden fixtures in tests/golden/ (tests/test_oracle_golden.py).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
// this library (oracle/liboracle.so), and only as the checker.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "xyzb.h"

namespace {

struct data_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---- RNG contract (rng.hpp:8-31) ----
uint64_t splitmix64(uint64_t& state) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

std::mt19937_64 make_stream(uint64_t seed, uint64_t stream) {
    uint64_t s = seed;
    const uint64_t a = splitmix64(s);
    s ^= stream * 0xd1342543de82ef95ULL + 0x2545f4914f6cdd1dULL;
    const uint64_t b = splitmix64(s);
    std::seed_seq seq{uint32_t(a), uint32_t(a >> 32), uint32_t(b), uint32_t(b >> 32)};
    return std::mt19937_64(seq);
}

double uniform_unit(std::mt19937_64& rng) { return double(rng() >> 11) * 0x1.0p-53; }

// WeightedSampler::from_magnitudes + sample (real_matrix.cpp:20-54)
struct Sampler {
    std::vector<double> cum;
    explicit Sampler(const double* y, size_t n) {
        double norm = 0.0;
        for (size_t i = 0; i < n; ++i) norm += std::abs(y[i]);
        if (norm <= 0.0) throw data_error("WeightedSampler: zero response vector");
        std::vector<double> w(n);
        for (size_t i = 0; i < n; ++i) w[i] = std::abs(y[i]) / norm;
        double acc = 0.0;
        for (double v : w) acc += v;
        for (double& v : w) v /= acc;
        cum.resize(n);
        double c = 0.0;
        for (size_t i = 0; i < n; ++i) {
            c += w[i];
            cum[i] = c;
        }
        if (std::abs(c - 1.0) > 1e-12) throw data_error("WeightedSampler: weights do not sum to 1");
        cum.back() = 1.0;
    }
    size_t sample(std::mt19937_64& rng) const {
        const double u = uniform_unit(rng);
        const size_t pos = size_t(std::upper_bound(cum.begin(), cum.end(), u) - cum.begin());
        return std::min(pos, cum.size() - 1);
    }
};

// draw_subsample (projection.cpp:12-30)
std::vector<size_t> draw_rows(size_t n, size_t m, const Sampler* w, std::mt19937_64& rng) {
    std::vector<size_t> idx(m);
    if (w != nullptr) {
        for (size_t s = 0; s < m; ++s) idx[s] = w->sample(rng);
    } else {
        std::uniform_int_distribution<size_t> dist(0, n - 1);
        for (size_t s = 0; s < m; ++s) idx[s] = dist(rng);
    }
    return idx;
}

inline int xbit(const uint64_t* xw, size_t W, size_t i, size_t j) {
    return int((xw[j * W + (i >> 6)] >> (i & 63)) & 1u);
}

struct Hit {
    uint32_t j, k;
    double s;
    uint32_t rep;
    int sign;
};

struct RunOutcome {
    uint64_t enumerated = 0;
    uint64_t evaluated = 0;
    uint64_t canonical = 0;  // engine counter: canonical off-diagonal candidates of a non-aborted run
    bool aborted = false;
    std::vector<Hit> hits;  // every evaluated candidate with s >= gamma, A.5 order
};

// One run given its keys (Appendix A.4-A.7). x_keys[j]; z-key of column k is
// zkey(k). Candidate (j,k): x_keys[j] == zkey(k). Pairs in (key, j, k) order.
template <class ZKey, class Strength>
RunOutcome run_once(const std::vector<uint64_t>& xk, ZKey zkey, Strength strength, double gamma,
                    uint64_t guard, uint32_t rep, int sign, std::unordered_set<uint64_t>& seen) {
    RunOutcome out;
    const size_t p = xk.size();
    std::map<uint64_t, std::vector<uint32_t>> xs, zs;
    for (uint32_t j = 0; j < p; ++j) xs[xk[j]].push_back(j);
    for (uint32_t k = 0; k < p; ++k) zs[zkey(k)].push_back(k);
    for (const auto& [key, cols] : xs) {
        auto it = zs.find(key);
        if (it != zs.end()) out.enumerated += uint64_t(cols.size()) * it->second.size();
    }
    if (out.enumerated > guard) {
        out.aborted = true;
        return out;
    }
    for (const auto& [key, cols] : xs) {
        auto it = zs.find(key);
        if (it == zs.end()) continue;
        for (uint32_t j : cols) {
            for (uint32_t k : it->second) {
                if (j == k) continue;
                if (j < k) ++out.canonical;
                const uint64_t canon = (uint64_t(std::min(j, k)) << 32) | std::max(j, k);
                if (!seen.insert(canon).second) continue;  // reference's threads=1 evaluation count
                ++out.evaluated;
                const double s = strength(j, k);
                if (s >= gamma) out.hits.push_back({j, k, s, rep, sign});
            }
        }
    }
    return out;
}

struct Report {
    std::vector<Hit> hits;
    uint64_t reps = 0, checked = 0, enumerated = 0, aborted = 0, verified = 0;
    double estimated_c = 0.0, gamma0 = 0.0;
};

// A.8: passes in order, runs in order; first occurrence of (min,max,sign) wins.
// stop_after_first_hit: stop after the first run that emitted a hit (threads=1).
struct Merger {
    Report& rep;
    std::unordered_set<uint64_t> emitted;
    bool stop_after_first;
    bool stopped = false;
    void add(const RunOutcome& o) {
        ++rep.reps;
        rep.enumerated += o.enumerated;
        rep.checked += o.evaluated;
        rep.verified += o.canonical;
        if (o.aborted) ++rep.aborted;
        for (const Hit& h : o.hits) {
            const uint64_t canon = (uint64_t(std::min(h.j, h.k)) << 32) | std::max(h.j, h.k);
            const uint64_t tag = canon ^ (h.sign < 0 ? (uint64_t(1) << 63) : 0);
            if (emitted.insert(tag).second) rep.hits.push_back(h);
        }
        if (stop_after_first && !rep.hits.empty()) stopped = true;
    }
};

void validate(const xyzb_params* q) {
    if (q->m < 1 || q->m > 64) throw data_error("SearchConfig: M = " + std::to_string(q->m) + " outside [1,64]");
    if (q->l < 1) throw data_error("SearchConfig: L must be >= 1");
    if (!(q->gamma > 0.0 && q->gamma <= 1.0)) throw data_error("SearchConfig: gamma must lie in (0,1]");
    const bool wants = q->mode == XYZB_MODE_CONTINUOUS_XY;
    if (wants && q->transform == XYZB_TRANSFORM_NONE)
        throw data_error("SearchConfig: continuous-XY mode requires a binarize transform");
    if (!wants && q->transform != XYZB_TRANSFORM_NONE)
        throw data_error("SearchConfig: binarize transform is only valid in continuous-XY mode");
}

double mean_pow(const std::vector<double>& s, size_t m) {
    double acc = 0.0;
    for (double v : s) acc += std::pow(v, double(m));
    return acc / double(s.size());
}

// expected_complexity (search.cpp:179-188)
double complexity(size_t m, size_t l, const std::vector<double>& s, size_t n, size_t p) {
    const double np = double(n) * double(p), pd = double(p);
    const double e1 = pd * pd * mean_pow(s, m);
    return np + double(l) * (double(m) * pd + pd * std::log(pd) + double(n) * e1);
}

// strength sample pair draws (search.cpp:229-242): j,k uniform, k redrawn while equal.
template <class F>
std::vector<double> sample_pairs(size_t p, size_t count, std::mt19937_64& rng, F strength) {
    std::uniform_int_distribution<size_t> dist(0, p - 1);
    std::vector<double> out;
    out.reserve(count);
    for (size_t t = 0; t < count; ++t) {
        size_t j = dist(rng), k = dist(rng);
        while (p > 1 && k == j) k = dist(rng);
        out.push_back(strength(j, k));
    }
    return out;
}

// ---- binary mode (search.cpp:325-365) ----
Report search_binary(const uint64_t* xw, size_t n, size_t p, const int8_t* y, const xyzb_params* q) {
    const size_t W = (n + 63) / 64;
    for (size_t i = 0; i < n; ++i)
        if (y[i] != 1 && y[i] != -1) throw data_error("xyz_search: binary response must be +-1");
    std::vector<int> yb(n);
    for (size_t i = 0; i < n; ++i) yb[i] = y[i] > 0;
    const size_t m = q->m;
    const uint64_t mask = m == 64 ? ~uint64_t(0) : ((uint64_t(1) << m) - 1);
    const uint64_t guard = q->max_candidates_per_rep ? q->max_candidates_per_rep : 16 * uint64_t(p);
    // scalar agreement count: rows where Y_i == X_ij * X_ik  <=> xj ^ xk ^ y == 1
    auto agree = [&](uint32_t j, uint32_t k) {
        size_t a = 0;
        for (size_t i = 0; i < n; ++i) a += (xbit(xw, W, i, j) ^ xbit(xw, W, i, k) ^ yb[i]) & 1;
        return a;
    };
    Report rep;
    Merger mg{rep, {}, q->stop_after_first_hit != 0};
    const int npass = q->search_negatives ? 2 : 1;
    for (int pass = 0; pass < npass && !mg.stopped; ++pass) {
        const int sign = pass == 0 ? +1 : -1;
        const uint64_t offset = pass == 0 ? 0 : q->l;
        std::unordered_set<uint64_t> seen;
        for (uint32_t r = 1; r <= q->l && !mg.stopped; ++r) {
            std::mt19937_64 rng = make_stream(q->seed, offset + r);
            const auto rows = draw_rows(n, m, nullptr, rng);
            std::vector<uint64_t> xk(p, 0);
            uint64_t yk = 0;
            for (size_t s = 0; s < m; ++s) {
                yk |= uint64_t(yb[rows[s]]) << s;
                for (size_t j = 0; j < p; ++j) xk[j] |= uint64_t(xbit(xw, W, rows[s], j)) << s;
            }
            const uint64_t c = sign > 0 ? (~yk & mask) : yk;
            auto zkey = [&](uint32_t k) { return xk[k] ^ c; };
            auto strength = [&](uint32_t j, uint32_t k) {
                const size_t a = agree(j, k);
                return sign > 0 ? double(a) / double(n) : double(n - a) / double(n);
            };
            mg.add(run_once(xk, zkey, strength, q->gamma, guard, r, sign, seen));
        }
    }
    if (q->estimate_complexity) {
        std::mt19937_64 rng = make_stream(q->seed, 0);
        const size_t cnt = q->strength_sample_size ? q->strength_sample_size : std::min<size_t>(100000, 10 * p);
        // sample_strengths(x, z_plus): interaction_strength(x, z, j, k) = agreements(Z_j, X_k)/n
        const auto s = sample_pairs(p, cnt, rng, [&](size_t j, size_t k) {
            return double(agree(uint32_t(j), uint32_t(k))) / double(n);
        });
        rep.estimated_c = complexity(m, q->l, s, n, p);
    }
    return rep;
}

// weighted strength (transforms.cpp:42-76): sum |y_i| over rows with
// sgn(resp_i) == X_ij X_ik (resp_i > 0 read as +), over ||resp||_1.
double weighted_strength(const uint64_t* xw, size_t W, size_t n, const double* resp, double norm,
                         uint32_t j, uint32_t k) {
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const int s = resp[i] > 0.0;
        if ((xbit(xw, W, i, j) ^ xbit(xw, W, i, k) ^ s) & 1) acc += std::abs(resp[i]);
    }
    return acc / norm;
}

// ---- continuous-Y mode (search.cpp:367-413) ----
Report search_cy(const uint64_t* xw, size_t n, size_t p, const double* y, const xyzb_params* q) {
    const size_t W = (n + 63) / 64;
    double norm = 0.0;
    for (size_t i = 0; i < n; ++i) norm += std::abs(y[i]);
    if (norm <= 0.0) throw data_error("xyz_search: zero response vector");
    const Sampler sampler(y, n);
    std::vector<double> yneg(n);
    for (size_t i = 0; i < n; ++i) yneg[i] = -y[i];
    const size_t m = q->m;
    const uint64_t mask = m == 64 ? ~uint64_t(0) : ((uint64_t(1) << m) - 1);
    const uint64_t guard = q->max_candidates_per_rep ? q->max_candidates_per_rep : 16 * uint64_t(p);
    Report rep;
    Merger mg{rep, {}, q->stop_after_first_hit != 0};
    const int npass = q->search_negatives ? 2 : 1;
    for (int pass = 0; pass < npass && !mg.stopped; ++pass) {
        const int sign = pass == 0 ? +1 : -1;
        const uint64_t offset = pass == 0 ? 0 : q->l;
        const double* resp = pass == 0 ? y : yneg.data();
        std::unordered_set<uint64_t> seen;
        for (uint32_t r = 1; r <= q->l && !mg.stopped; ++r) {
            std::mt19937_64 rng = make_stream(q->seed, offset + r);
            const auto rows = draw_rows(n, m, &sampler, rng);
            std::vector<uint64_t> xk(p, 0);
            uint64_t yk = 0;
            for (size_t s = 0; s < m; ++s) {
                yk |= uint64_t(y[rows[s]] >= 0.0) << s;  // y_sign (search.cpp:377-378)
                for (size_t j = 0; j < p; ++j) xk[j] |= uint64_t(xbit(xw, W, rows[s], j)) << s;
            }
            const uint64_t c = sign > 0 ? (~yk & mask) : yk;
            auto zkey = [&](uint32_t k) { return xk[k] ^ c; };
            double rnorm = 0.0;
            for (size_t i = 0; i < n; ++i) rnorm += std::abs(resp[i]);
            auto strength = [&](uint32_t j, uint32_t k) {
                return weighted_strength(xw, W, n, resp, rnorm, j, k);
            };
            mg.add(run_once(xk, zkey, strength, q->gamma, guard, r, sign, seen));
        }
    }
    if (q->estimate_complexity) {
        std::mt19937_64 rng = make_stream(q->seed, 0);
        const size_t cnt = q->strength_sample_size ? q->strength_sample_size : std::min<size_t>(100000, 10 * p);
        const auto s = sample_pairs(p, cnt, rng, [&](size_t j, size_t k) {
            return weighted_strength(xw, W, n, y, norm, uint32_t(j), uint32_t(k));
        });
        rep.estimated_c = complexity(m, q->l, s, n, p);
    }
    return rep;
}

double sgn(double v) { return v > 0.0 ? 1.0 : (v < 0.0 ? -1.0 : 0.0); }

// ---- continuous-XY mode (search.cpp:415-506) ----
Report search_cxy(const double* x, size_t n, size_t p, const double* y, const xyzb_params* q) {
    double norm = 0.0;
    for (size_t i = 0; i < n; ++i) norm += std::abs(y[i]);
    if (norm <= 0.0) throw data_error("xyz_search: zero response vector");
    const bool unbiased = q->transform == XYZB_TRANSFORM_UNBIASED;
    if (unbiased) {
        for (size_t t = 0; t < n * p; ++t)
            if (!(x[t] >= -1.0 && x[t] <= 1.0))
                throw data_error("xyz_search: unbiased transform needs entries in [-1,1]; apply rescale_rows or cap_entries first");
    }
    const Sampler sampler(y, n);
    const size_t m = q->m;
    const uint64_t guard = q->max_candidates_per_rep ? q->max_candidates_per_rep : 16 * uint64_t(p);
    auto dot = [&](size_t j, size_t k) {
        const double* cj = x + j * n;
        const double* ck = x + k * n;
        double acc = 0.0;
        if (unbiased) {
            for (size_t i = 0; i < n; ++i) acc += y[i] * cj[i] * ck[i];
        } else {
            for (size_t i = 0; i < n; ++i) acc += y[i] * sgn(cj[i]) * sgn(ck[i]);
        }
        return acc;
    };
    Report rep;
    Merger mg{rep, {}, q->stop_after_first_hit != 0};
    const int npass = q->search_negatives ? 2 : 1;
    for (int pass = 0; pass < npass && !mg.stopped; ++pass) {
        const int sign = pass == 0 ? +1 : -1;
        const uint64_t offset = pass == 0 ? 0 : q->l;
        std::unordered_set<uint64_t> seen;
        for (uint32_t r = 1; r <= q->l && !mg.stopped; ++r) {
            std::mt19937_64 rng = make_stream(q->seed, offset + r);
            const auto rows = draw_rows(n, m, &sampler, rng);
            std::vector<int> resp_pos(m);
            for (size_t s = 0; s < m; ++s) resp_pos[s] = (sign > 0 ? y[rows[s]] : -y[rows[s]]) > 0.0;
            std::vector<uint64_t> xk(p, 0), zk(p, 0);
            // RNG order: j-major, s-minor (search.cpp:449-466)
            for (size_t j = 0; j < p; ++j) {
                for (size_t s = 0; s < m; ++s) {
                    const double v = x[j * n + rows[s]];
                    int plus;
                    if (unbiased) plus = uniform_unit(rng) < (v + 1.0) / 2.0;
                    else if (v > 0.0) plus = 1;
                    else if (v < 0.0) plus = 0;
                    else plus = int(rng() & 1u);
                    xk[j] |= uint64_t(plus) << s;
                    zk[j] |= uint64_t(plus == resp_pos[s]) << s;
                }
            }
            auto zkey = [&](uint32_t k) { return zk[k]; };
            auto strength = [&](uint32_t j, uint32_t k) { return 0.5 + sign * dot(j, k) / (2.0 * norm); };
            mg.add(run_once(xk, zkey, strength, q->gamma, guard, r, sign, seen));
        }
    }
    if (q->estimate_complexity) {
        std::mt19937_64 rng = make_stream(q->seed, 0);
        const size_t cnt = q->strength_sample_size ? q->strength_sample_size : std::min<size_t>(100000, 10 * p);
        const auto s = sample_pairs(p, cnt, rng, [&](size_t j, size_t k) { return 0.5 + dot(j, k) / (2.0 * norm); });
        rep.estimated_c = complexity(m, q->l, s, n, p);
    }
    return rep;
}

void set_err(char* err, size_t errlen, const std::string& msg) {
    if (err != nullptr && errlen > 0) std::snprintf(err, errlen, "%s", msg.c_str());
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        return XYZB_OK;
    } catch (const data_error& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_DATA;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return XYZB_E_INTERNAL;
    }
}

void fill(const Report& r, const xyzb_params* q, size_t p, xyzb_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->n_hits = r.hits.size();
    out->hits = static_cast<xyzb_hit*>(std::malloc(std::max<size_t>(1, r.hits.size()) * sizeof(xyzb_hit)));
    for (size_t i = 0; i < r.hits.size(); ++i)
        out->hits[i] = {r.hits[i].j, r.hits[i].k, r.hits[i].s, r.hits[i].rep, r.hits[i].sign};
    out->repetitions_run = r.reps;
    out->runs_executed = r.reps;
    out->candidates_checked = r.checked;
    out->candidates_enumerated = r.enumerated;
    out->aborted_repetitions = r.aborted;
    out->verified_pairs = r.verified;
    out->estimated_c = r.estimated_c;
    out->gamma0 = std::pow(double(p), -1.0 / double(q->m));
    out->m_used = q->m;
    out->l_used = q->l;
    // A.10 top-K: strength desc, min asc, max asc, sign desc (oracle.cpp:47-51 + sign)
    if (q->top_k > 0) {
        std::vector<uint64_t> idx(r.hits.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
        std::stable_sort(idx.begin(), idx.end(), [&](uint64_t a, uint64_t b) {
            const Hit& x = r.hits[a];
            const Hit& y = r.hits[b];
            if (x.s != y.s) return x.s > y.s;
            const auto xl = std::min(x.j, x.k), yl = std::min(y.j, y.k);
            if (xl != yl) return xl < yl;
            const auto xh = std::max(x.j, x.k), yh = std::max(y.j, y.k);
            if (xh != yh) return xh < yh;
            return x.sign > y.sign;
        });
        const size_t kk = std::min<size_t>(q->top_k, idx.size());
        out->n_top_k = kk;
        out->top_k = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, kk) * sizeof(uint64_t)));
        for (size_t i = 0; i < kk; ++i) out->top_k[i] = idx[i];
    }
}

} // namespace

extern "C" {

int oracle_abi_version(void) { return XYZB_ABI_VERSION; }

int oracle_search(const xyzb_problem* prob, const xyzb_response* resp, const xyzb_params* q,
                  xyzb_result* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        validate(q);
        const size_t n = prob->n_rows, p = prob->n_cols;
        if (n == 0 || p == 0) throw data_error("xyz_search: empty matrix");
        Report r;
        if (q->mode == XYZB_MODE_BINARY) {
            if (!prob->x_words || !resp->y_sign) throw data_error("binary mode needs x_words and y_sign");
            r = search_binary(prob->x_words, n, p, resp->y_sign, q);
        } else if (q->mode == XYZB_MODE_CONTINUOUS_Y) {
            if (!prob->x_words || !resp->y_real) throw data_error("continuous-Y needs x_words and y_real");
            r = search_cy(prob->x_words, n, p, resp->y_real, q);
        } else {
            if (!prob->x_real || !resp->y_real) throw data_error("continuous-XY needs x_real and y_real");
            r = search_cxy(prob->x_real, n, p, resp->y_real, q);
        }
        fill(r, q, p, out);
    });
}

void oracle_result_free(xyzb_result* r) {
    if (!r) return;
    std::free(r->hits);
    std::free(r->top_k);
    std::free(r->order_keys);
    r->hits = nullptr;
    r->top_k = nullptr;
    r->order_keys = nullptr;
}

void oracle_free(void* p) { std::free(p); }

// Row draws of every run of a search, uint32 [passes][L][M] in pass order
// (stream offset + rep, rep = 1..L; A.1-A.2). y != NULL selects weighted draws.
int oracle_draws(uint64_t n, uint64_t m, uint64_t l, int32_t negatives, uint64_t seed,
                 const double* y, uint32_t* out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const Sampler* w = nullptr;
        std::vector<Sampler> holder;
        if (y != nullptr) {
            holder.emplace_back(y, n);
            w = &holder[0];
        }
        const int npass = negatives ? 2 : 1;
        for (int pass = 0; pass < npass; ++pass)
            for (uint64_t r = 1; r <= l; ++r) {
                std::mt19937_64 rng = make_stream(seed, (pass == 0 ? 0 : l) + r);
                const auto rows = draw_rows(n, m, w, rng);
                for (size_t s = 0; s < m; ++s) out[((pass * l) + (r - 1)) * m + s] = uint32_t(rows[s]);
            }
    });
}

// Keys of every column for explicit draws (A.3, binary).
int oracle_project_keys(const uint64_t* xw, uint64_t n, uint64_t p, const uint32_t* draws,
                        uint64_t n_draws, uint64_t m, uint64_t* keys, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const size_t W = (n + 63) / 64;
        for (size_t d = 0; d < n_draws; ++d)
            for (size_t j = 0; j < p; ++j) {
                uint64_t k = 0;
                for (size_t s = 0; s < m; ++s) k |= uint64_t(xbit(xw, W, draws[d * m + s], j)) << s;
                keys[d * p + j] = k;
            }
    });
}

// Generic equal-key join in filter order (key asc, j asc, k asc).
int oracle_equal_pairs(const uint64_t* xk, const uint64_t* zk, uint64_t p, uint32_t** pairs,
                       uint64_t* n_pairs, uint64_t* total, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::map<uint64_t, std::vector<uint32_t>> xs, zs;
        for (uint32_t j = 0; j < p; ++j) xs[xk[j]].push_back(j);
        for (uint32_t k = 0; k < p; ++k) zs[zk[k]].push_back(k);
        std::vector<uint32_t> flat;
        uint64_t t = 0;
        for (const auto& [key, cols] : xs) {
            auto it = zs.find(key);
            if (it == zs.end()) continue;
            t += uint64_t(cols.size()) * it->second.size();
            for (uint32_t j : cols)
                for (uint32_t k : it->second) {
                    flat.push_back(j);
                    flat.push_back(k);
                }
        }
        *total = t;
        *n_pairs = flat.size() / 2;
        *pairs = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, flat.size()) * sizeof(uint32_t)));
        std::copy(flat.begin(), flat.end(), *pairs);
    });
}

// Pass-+1 strengths of explicit pairs (A.6).
int oracle_pair_strengths(const xyzb_problem* prob, const xyzb_response* resp, int32_t mode,
                          int32_t transform, const uint32_t* pairs, uint64_t n_pairs, double* out,
                          char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const size_t n = prob->n_rows;
        const size_t W = (n + 63) / 64;
        if (mode == XYZB_MODE_BINARY) {
            for (size_t t = 0; t < n_pairs; ++t) {
                size_t a = 0;
                for (size_t i = 0; i < n; ++i)
                    a += (xbit(prob->x_words, W, i, pairs[2 * t]) ^ xbit(prob->x_words, W, i, pairs[2 * t + 1]) ^
                          int(resp->y_sign[i] > 0)) & 1;
                out[t] = double(a) / double(n);
            }
        } else if (mode == XYZB_MODE_CONTINUOUS_Y) {
            double norm = 0.0;
            for (size_t i = 0; i < n; ++i) norm += std::abs(resp->y_real[i]);
            if (norm <= 0.0) throw data_error("zero response vector");
            for (size_t t = 0; t < n_pairs; ++t)
                out[t] = weighted_strength(prob->x_words, W, n, resp->y_real, norm, pairs[2 * t], pairs[2 * t + 1]);
        } else {
            double norm = 0.0;
            for (size_t i = 0; i < n; ++i) norm += std::abs(resp->y_real[i]);
            for (size_t t = 0; t < n_pairs; ++t) {
                const double* cj = prob->x_real + size_t(pairs[2 * t]) * n;
                const double* ck = prob->x_real + size_t(pairs[2 * t + 1]) * n;
                double acc = 0.0;
                for (size_t i = 0; i < n; ++i)
                    acc += transform == XYZB_TRANSFORM_UNBIASED ? resp->y_real[i] * cj[i] * ck[i]
                                                                : resp->y_real[i] * sgn(cj[i]) * sgn(ck[i]);
                out[t] = 0.5 + acc / (2.0 * norm);
            }
        }
    });
}

} // extern "C"
