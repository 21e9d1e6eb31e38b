// colour_rng.cpp -- host API surface of color.hpp and rng.hpp (reference
// include/quant/color.hpp:47-72, include/quant/rng.hpp:17-64, src/rng.cpp).
// The device kernels draw from the same mt19937_64 stream (csrc/init.cu).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "context.hpp"

namespace quant {

double dist2(const ColorPoint &a, const ColorPoint &b) {
    const double d[3] = {a.r - b.r, a.g - b.g, a.b - b.b};
    return (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]; // built with -ffp-contract=off
}
double dist2(const ColorPoint &a, const Rgb8 &b) { return dist2(a, ColorPoint(b)); }

std::uint8_t channel_to_u8(double v) {
    const double r = std::clamp(std::floor(v + 0.5), 0.0, 255.0);
    return static_cast<std::uint8_t>(r);
}
Rgb8 to_rgb8(const ColorPoint &c) { return {channel_to_u8(c.r), channel_to_u8(c.g), channel_to_u8(c.b)}; }

std::uint64_t Rng::next_below(std::uint64_t n) {
    if (n == 0) throw std::invalid_argument("next_below: empty range");
    // accept only draws below the largest multiple of n (no modulo bias)
    const std::uint64_t accept = UINT64_MAX - UINT64_MAX % n;
    for (;;) {
        const std::uint64_t x = gen_();
        if (x < accept) return x % n;
    }
}

std::size_t weighted_draw(std::span<const double> mass, Rng &rng) {
    double total = 0.0;
    for (double m : mass) total += m;
    if (!(total > 0.0)) throw std::invalid_argument("weighted_draw: total mass must be positive");
    const double target = rng.next_unit() * total;
    double prefix = 0.0;
    const std::size_t last = mass.size() - 1;
    for (std::size_t i = 0; i < last; ++i) {
        prefix += mass[i];
        if (target < prefix) return i;
    }
    return last;
}

std::vector<std::size_t> sample_indices_uniform(std::size_t n, std::size_t k, Rng &rng) {
    if (k > n) throw std::invalid_argument("sample_indices_uniform: k exceeds population");
    std::vector<std::size_t> perm(n);
    std::iota(perm.begin(), perm.end(), std::size_t{0});
    for (std::size_t i = 0; i < k; ++i) // partial Fisher-Yates: slot i takes a draw from [i, n)
        std::swap(perm[i], perm[i + static_cast<std::size_t>(rng.next_below(n - i))]);
    perm.resize(k);
    return perm;
}

std::vector<std::size_t> sample_indices_weighted(std::span<const double> weights, std::size_t k, Rng &rng) {
    const std::size_t n = weights.size();
    if (k > n) throw std::invalid_argument("sample_indices_weighted: k exceeds population");
    // Efraimidis-Spirakis: key_i = log(u_i) / w_i, keep the k largest (ties: lower index)
    std::vector<std::pair<double, std::size_t>> keys(n);
    for (std::size_t i = 0; i < n; ++i) {
        if (!(weights[i] > 0.0)) throw std::invalid_argument("sample_indices_weighted: weights must be positive");
        const double u = rng.next_unit();
        keys[i] = {std::log(u > 0.0 ? u : 0x1.0p-53) / weights[i], i};
    }
    std::partial_sort(keys.begin(), keys.begin() + static_cast<std::ptrdiff_t>(k), keys.end(),
                      [](const auto &a, const auto &b) { return a.first != b.first ? a.first > b.first : a.second < b.second; });
    std::vector<std::size_t> out(k);
    for (std::size_t i = 0; i < k; ++i) out[i] = keys[i].second;
    return out;
}

} // namespace quant
