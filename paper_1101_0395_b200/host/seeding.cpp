// seeding.cpp -- init.hpp on the device (reference src/init.cpp:37-52,
// 127-138, 295-335): maximin and k-means++ (bit-exact draws), the k-means++
// mass law and maximin padding.
#include "context.hpp"

namespace quant {

using detail::check;
using detail::ctx;
using detail::flatten;
using detail::unflatten;

namespace {
std::vector<ColorPoint> seed_on_device(int kind, const WeightedHistogram &hist, const SeedConfig &cfg) {
    const std::vector<std::uint32_t> packed = detail::pack_all(hist.colors);
    std::vector<double> out(3 * static_cast<std::size_t>(std::max(cfg.k, 1)));
    if (kind == CQG_INIT_MAXIMIN)
        check(cqg_init_maximin(ctx(), packed.data(), hist.counts.data(), hist.size(), hist.source_pixel_count, cfg.k,
                               cfg.seed, cfg.maximin_weighted_first ? 1 : 0, out.data()));
    else
        check(cqg_init_kmeanspp(ctx(), packed.data(), hist.counts.data(), hist.size(), hist.source_pixel_count, cfg.k,
                                cfg.seed, out.data()));
    return unflatten(out.data(), static_cast<std::size_t>(cfg.k));
}
} // namespace

std::vector<ColorPoint> init_maximin(const WeightedHistogram &hist, const SeedConfig &cfg) {
    return seed_on_device(CQG_INIT_MAXIMIN, hist, cfg);
}

std::vector<ColorPoint> init_kmeanspp(const WeightedHistogram &hist, const SeedConfig &cfg) {
    return seed_on_device(CQG_INIT_KMEANSPP, hist, cfg);
}

std::vector<double> kmeanspp_next_masses(const WeightedHistogram &hist, std::span<const ColorPoint> centers) {
    if (centers.empty() || hist.size() == 0) return {hist.weights.begin(), hist.weights.end()};
    const std::vector<double> cols = flatten(hist.colors), c = flatten(centers);
    std::vector<double> mass(hist.size());
    check(cqg_kmeanspp_next_masses(ctx(), cols.data(), hist.weights.data(), hist.size(), c.data(),
                                   static_cast<int>(centers.size()), mass.data()));
    return mass;
}

std::vector<ColorPoint> maximin_pad(const WeightedHistogram &hist, std::vector<ColorPoint> centers, int k) {
    const std::vector<double> cols = flatten(hist.colors), c = flatten(centers);
    const std::size_t k0 = centers.size(), kk = std::max<std::size_t>(k0, k > 0 ? static_cast<std::size_t>(k) : 0);
    std::vector<double> out(3 * std::max<std::size_t>(kk, 1));
    check(cqg_maximin_pad(ctx(), cols.empty() ? nullptr : cols.data(), hist.size(), c.empty() ? nullptr : c.data(),
                          static_cast<int>(k0), k, out.data()));
    return unflatten(out.data(), kk);
}

} // namespace quant
