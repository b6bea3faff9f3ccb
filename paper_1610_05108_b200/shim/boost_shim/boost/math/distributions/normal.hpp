// Test infrastructure only (oracle build). Boost.Math is absent from this
// image; the reference includes <boost/math/distributions/normal.hpp> solely
// for normal_cdf / normal_quantile (proj/core/src/projection.cpp:6,83-91),
// which serve the Gaussian-baseline helpers and are off the xyz hot path.
// This header supplies the two calls with erfc and a bisection quantile.
#pragma once

#include <cmath>

namespace boost {
namespace math {

template <class T = double>
class normal_distribution {
public:
    explicit normal_distribution(T mean = 0, T sd = 1) : mean_(mean), sd_(sd) {}
    T mean() const { return mean_; }
    T standard_deviation() const { return sd_; }

private:
    T mean_, sd_;
};

template <class T>
T cdf(const normal_distribution<T>& d, T x) {
    const T z = (x - d.mean()) / d.standard_deviation();
    return T(0.5) * std::erfc(-z / std::sqrt(T(2)));
}

template <class T>
T quantile(const normal_distribution<T>& d, T q) {
    if (q <= T(0)) return -INFINITY;
    if (q >= T(1)) return INFINITY;
    T lo = -40, hi = 40;
    const normal_distribution<T> unit;
    for (int it = 0; it < 200; ++it) {
        const T mid = (lo + hi) / 2;
        if (cdf(unit, mid) < q) lo = mid; else hi = mid;
    }
    return d.mean() + d.standard_deviation() * (lo + hi) / 2;
}

} // namespace math
} // namespace boost
