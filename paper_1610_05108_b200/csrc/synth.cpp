// Seeded synthetic inputs (see include/xyzb_synth.h for the recipes).
#include "xyzb_synth.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "host_rng.hpp"

namespace {

inline uint64_t mix(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t s = a ^ (b * 0x9e3779b97f4a7c15ULL) ^ (c * 0xc2b2ae3d27d4eb4fULL);
    return xyzb::host::splitmix64(s);
}

struct Counter {  // splitmix64 sequence keyed by (seed, stream)
    uint64_t state;
    Counter(uint64_t seed, uint64_t stream) : state(mix(seed, stream, 0x51f7)) {}
    uint64_t next() { return xyzb::host::splitmix64(state); }
    double unit() { return double(next() >> 11) * 0x1.0p-53; }
    double normal() {  // Box-Muller, one value per call
        double u1 = unit();
        while (u1 <= 0.0) u1 = unit();
        const double u2 = unit();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
    float fast_normal() {  // Irwin-Hall(4) standardised: 2 draws, no transcendentals
        const uint64_t a = next(), b = next();
        const float s = float(uint32_t(a)) + float(uint32_t(a >> 32)) + float(uint32_t(b)) + float(uint32_t(b >> 32));
        return (s * 2.3283064365386963e-10f - 2.0f) * 1.7320508075688772f;
    }
};

void planted_pairs(uint64_t p, uint64_t n_pairs, uint64_t seed, uint32_t* pairs) {
    // disjoint pairs of distinct columns, j < k
    Counter c(seed, 0xfeed);
    std::vector<uint32_t> used;
    for (uint64_t q = 0; q < n_pairs; ++q) {
        uint32_t a, b;
        do {
            a = uint32_t(c.next() % p);
            b = uint32_t(c.next() % p);
        } while (a == b || std::find(used.begin(), used.end(), a) != used.end() ||
                 std::find(used.begin(), used.end(), b) != used.end());
        used.push_back(a);
        used.push_back(b);
        pairs[2 * q] = std::min(a, b);
        pairs[2 * q + 1] = std::max(a, b);
    }
}

// static-partition parallel for over [0, n) with std::thread (no OpenMP here)
template <class F>
void parallel_for(int64_t n, F&& f) {
    const int64_t T = std::max<int64_t>(1, std::min<int64_t>(n, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int64_t t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) f(i);
        });
    for (auto& th : pool) th.join();
}

inline int xbit(const uint64_t* xw, uint64_t W, uint64_t i, uint64_t j) {
    return int((xw[j * W + (i >> 6)] >> (i & 63)) & 1u);
}

} // namespace

extern "C" {

int xyzb_synth_toy(uint64_t n, uint64_t p, uint64_t j, uint64_t k, double gamma, uint64_t seed, uint64_t* x_words,
                   int8_t* y) {
    if (n == 0 || p == 0 || j >= p || k >= p) return 3;
    std::mt19937_64 rng = xyzb::host::make_stream(seed, 0x5e17);
    const uint64_t W = (n + 63) / 64;
    const uint64_t tail = n & 63;
    const uint64_t mask = tail == 0 ? ~0ull : ((1ull << tail) - 1);
    for (uint64_t c = 0; c < p; ++c) {
        for (uint64_t w = 0; w < W; ++w) x_words[c * W + w] = rng();
        x_words[c * W + W - 1] &= mask;
    }
    const uint64_t agree = uint64_t(std::llround(gamma * double(n)));
    std::vector<uint64_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::shuffle(order.begin(), order.end(), rng);
    for (uint64_t t = 0; t < n; ++t) {
        const uint64_t i = order[t];
        const int prod = (xbit(x_words, W, i, j) == xbit(x_words, W, i, k)) ? 1 : -1;
        y[i] = int8_t(t < agree ? prod : -prod);
    }
    return 0;
}

int xyzb_synth_gwas(uint64_t n, uint64_t p, uint64_t n_pairs, double coef, uint64_t seed, uint64_t* x_words, int8_t* y,
                    uint32_t* pairs) {
    if (n == 0 || p < 2 * n_pairs) return 3;
    const uint64_t W = (n + 63) / 64;
    parallel_for(int64_t(p), [&](int64_t c) {
        Counter r(seed, uint64_t(c) + 1);
        const double maf = 0.05 + 0.45 * r.unit();
        const double pplus = 1.0 - (1.0 - maf) * (1.0 - maf);
        for (uint64_t w = 0; w < W; ++w) {
            uint64_t word = 0;
            const uint64_t rows = std::min<uint64_t>(64, n - w * 64);
            for (uint64_t b = 0; b < rows; ++b)
                if (r.unit() < pplus) word |= 1ull << b;
            x_words[uint64_t(c) * W + w] = word;
        }
    });
    planted_pairs(p, n_pairs, seed, pairs);
    Counter ry(seed, 0);
    for (uint64_t i = 0; i < n; ++i) {
        double eta = 0.0;
        for (uint64_t q = 0; q < n_pairs; ++q) {
            const int a = xbit(x_words, W, i, pairs[2 * q]) ? 1 : -1;
            const int b = xbit(x_words, W, i, pairs[2 * q + 1]) ? 1 : -1;
            eta += coef * a * b;
        }
        const double pr = 1.0 / (1.0 + std::exp(-eta));
        y[i] = ry.unit() < pr ? 1 : -1;
    }
    return 0;
}

int xyzb_synth_gauss(uint64_t n, uint64_t p, uint64_t n_pairs, double theta, double noise_sd, uint64_t n_mains,
                     double beta, uint64_t seed, double* x, double* y, uint32_t* pairs, uint32_t* mains) {
    if (n < 2 || p < 2 * n_pairs + n_mains) return 3;
    parallel_for(int64_t(p), [&](int64_t c) {
        Counter r(seed, uint64_t(c) + 1);
        double* col = x + uint64_t(c) * n;
        double mean = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            col[i] = r.normal();
            mean += col[i];
        }
        mean /= double(n);
        double ss = 0.0;
        for (uint64_t i = 0; i < n; ++i) ss += (col[i] - mean) * (col[i] - mean);
        const double sd = std::sqrt(ss / double(n));
        for (uint64_t i = 0; i < n; ++i) col[i] = double(float((col[i] - mean) / sd));  // fp32-exact values
    });
    planted_pairs(p, n_pairs, seed, pairs);
    // main effects: distinct columns outside the planted pairs
    {
        Counter c(seed, 0xa1a1);
        std::vector<uint32_t> used(pairs, pairs + 2 * n_pairs);
        for (uint64_t q = 0; q < n_mains; ++q) {
            uint32_t a;
            do a = uint32_t(c.next() % p);
            while (std::find(used.begin(), used.end(), a) != used.end());
            used.push_back(a);
            mains[q] = a;
        }
    }
    Counter ry(seed, 0);
    for (uint64_t i = 0; i < n; ++i) {
        double v = 0.0;
        for (uint64_t q = 0; q < n_mains; ++q) v += beta * x[uint64_t(mains[q]) * n + i];
        for (uint64_t q = 0; q < n_pairs; ++q) v += theta * x[uint64_t(pairs[2 * q]) * n + i] * x[uint64_t(pairs[2 * q + 1]) * n + i];
        y[i] = v + noise_sd * ry.normal();
    }
    return 0;
}

int xyzb_synth_ar1(uint64_t n, uint64_t p, uint64_t block, double rho, uint64_t n_pairs, double flip, uint64_t seed,
                   uint64_t* x_words, int8_t* y, uint32_t* pairs) {
    if (n == 0 || block == 0 || p < 2 * n_pairs) return 3;
    const uint64_t W = (n + 63) / 64;
    const uint64_t nblk = (p + block - 1) / block;
    const double sr = std::sqrt(1.0 - rho * rho);
    // one task per (column block, 64-row word)
    const float rf = float(rho), srf = float(sr);
    parallel_for(int64_t(nblk * W), [&](int64_t t) {
        const uint64_t cb = uint64_t(t) / W, w = uint64_t(t) % W;
        Counter r(seed, (cb << 24) ^ w ^ 0x77);
        const uint64_t rows = std::min<uint64_t>(64, n - w * 64);
        float z[64];
        for (uint64_t b = 0; b < rows; ++b) z[b] = r.fast_normal();
        for (uint64_t c = cb * block; c < std::min(p, (cb + 1) * block); ++c) {
            if (c != cb * block)
                for (uint64_t b = 0; b < rows; ++b) z[b] = rf * z[b] + srf * r.fast_normal();
            uint64_t word = 0;
            for (uint64_t b = 0; b < rows; ++b)
                if (z[b] > 0.0f) word |= 1ull << b;
            x_words[c * W + w] = word;
        }
    });
    planted_pairs(p, n_pairs, seed, pairs);
    Counter ry(seed, 0);
    for (uint64_t i = 0; i < n; ++i) {
        int s = 0;
        for (uint64_t q = 0; q < n_pairs; ++q) {
            const int a = xbit(x_words, W, i, pairs[2 * q]) ? 1 : -1;
            const int b = xbit(x_words, W, i, pairs[2 * q + 1]) ? 1 : -1;
            s += a * b;
        }
        int v = s >= 0 ? 1 : -1;
        if (ry.unit() < flip) v = -v;
        y[i] = int8_t(v);
    }
    return 0;
}

} // extern "C"
