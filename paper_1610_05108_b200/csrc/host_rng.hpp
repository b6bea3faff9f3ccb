// Host side of the draw contract. Row draws stay on
// the host because they are pinned to libstdc++'s std::mt19937_64 /
// std::seed_seq / std::uniform_int_distribution — the same standard-library
// code the reference calls (rng.hpp:8-31, projection.cpp:12-30,
// real_matrix.cpp:36-54) — and cost microseconds per run.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace xyzb {
namespace host {

// splitmix64 step (rng.hpp:8-13)
inline uint64_t splitmix64(uint64_t& state) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// Generator for (seed, stream) (rng.hpp:18-26): two splitmix64 outputs seed a
// std::seed_seq of their four 32-bit halves.
inline std::mt19937_64 make_stream(uint64_t seed, uint64_t stream) {
    uint64_t s = seed;
    const uint64_t a = splitmix64(s);
    s ^= stream * 0xd1342543de82ef95ULL + 0x2545f4914f6cdd1dULL;
    const uint64_t b = splitmix64(s);
    std::seed_seq seq{static_cast<uint32_t>(a), static_cast<uint32_t>(a >> 32), static_cast<uint32_t>(b),
                      static_cast<uint32_t>(b >> 32)};
    return std::mt19937_64(seq);
}

// 53-bit uniform in [0,1) (rng.hpp:29-31)
inline double uniform_unit(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// Inverse-CDF sampler over |y| (real_matrix.cpp:20-54): normalise by the L1
// norm, renormalise by the sum, cumulate, pin the last entry to 1.
class WeightedSampler {
public:
    WeightedSampler(const double* y, size_t n) {
        double norm = 0.0;
        for (size_t i = 0; i < n; ++i) norm += std::abs(y[i]);
        if (norm <= 0.0) throw std::invalid_argument("WeightedSampler: zero response vector");
        std::vector<double> w(n);
        for (size_t i = 0; i < n; ++i) w[i] = std::abs(y[i]) / norm;
        double acc = 0.0;
        for (double v : w) acc += v;
        for (double& v : w) v /= acc;
        cum_.resize(n);
        double c = 0.0;
        for (size_t i = 0; i < n; ++i) {
            if (!(w[i] >= 0.0)) throw std::invalid_argument("WeightedSampler: negative or NaN weight");
            c += w[i];
            cum_[i] = c;
        }
        if (std::abs(c - 1.0) > 1e-12)
            throw std::invalid_argument("WeightedSampler: weights sum to " + std::to_string(c) + ", expected 1");
        cum_.back() = 1.0;
    }
    size_t sample(std::mt19937_64& rng) const {
        const double u = uniform_unit(rng);
        const size_t pos = static_cast<size_t>(std::upper_bound(cum_.begin(), cum_.end(), u) - cum_.begin());
        return std::min(pos, cum_.size() - 1);
    }
    void copy_cumulative(double* out) const { std::copy(cum_.begin(), cum_.end(), out); }

private:
    std::vector<double> cum_;
};

// M row indices for one run (draw_subsample, projection.cpp:12-30).
inline void draw_rows(size_t n, size_t m, const WeightedSampler* w, std::mt19937_64& rng, uint32_t* out) {
    if (w != nullptr) {
        for (size_t s = 0; s < m; ++s) out[s] = static_cast<uint32_t>(w->sample(rng));
    } else {
        std::uniform_int_distribution<size_t> dist(0, n - 1);
        for (size_t s = 0; s < m; ++s) out[s] = static_cast<uint32_t>(dist(rng));
    }
}

// The engine's full state (312 words + position) through the standard
// stream insertion operator, so the device generator resumes exactly where
// the host draws stopped (continuous-XY transform draws, search.cpp:449-463).
inline void export_state(const std::mt19937_64& rng, uint64_t* state313) {
    std::ostringstream os;
    os << rng;
    std::istringstream is(os.str());
    for (int i = 0; i < 313; ++i) {
        unsigned long long v = 0;
        is >> v;
        state313[i] = v;
    }
    if (!is) throw std::runtime_error("export_state: unexpected mt19937_64 serialisation");
}

} // namespace host
} // namespace xyzb
