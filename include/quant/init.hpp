// quant/init.hpp -- drop-in for the hot-path initialisers of
// /root/reference/proj/include/quant/init.hpp:17-72: maximin and k-means++
// (device kernels, bit-exact draws), the k-means++ mass law and maximin
// padding (device). The other seeding schemes (forgy, lbg, density, variance,
// split-forgy) are outside the device path and are not declared here.
#ifndef QUANT_INIT_HPP
#define QUANT_INIT_HPP

#include <cstdint>
#include <span>
#include <vector>

#include "quant/color.hpp"
#include "quant/histogram.hpp"
#include "quant/kmeans.hpp"

namespace quant {

struct SeedConfig {
    int k = 8;
    std::uint64_t seed = 1;
    ColorPoint lbg_perturbation{0.255, 0.255, 0.255};
    Termination lbg_refine{};
    int density_grid = 8;
    bool maximin_weighted_first = true;
};

// The device reads the histogram's counts (weights == counts * (1/P), as
// build_histogram produces them).
std::vector<ColorPoint> init_maximin(const WeightedHistogram &hist, const SeedConfig &cfg);
std::vector<ColorPoint> init_kmeanspp(const WeightedHistogram &hist, const SeedConfig &cfg);

std::vector<double> kmeanspp_next_masses(const WeightedHistogram &hist, std::span<const ColorPoint> centers);
std::vector<ColorPoint> maximin_pad(const WeightedHistogram &hist, std::vector<ColorPoint> centers, int k);

} // namespace quant

#endif
