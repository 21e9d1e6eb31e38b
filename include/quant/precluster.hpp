// quant/precluster.hpp -- the part of /root/reference/proj/include/quant/precluster.hpp:16-34
// on the device path: the 32x32x32 coarse histogram every box-splitting
// preclusterer reads (cqg_coarse_histogram / _weighted: exact integer sums).
// The preclusterers themselves (median cut, Wan, Wu, octree, Otto, binary
// split) are outside the device path and are not declared here; their
// palettes can seed the device engine through run_quantize's init_centers
// overload (pipeline.hpp).
#ifndef QUANT_PRECLUSTER_HPP
#define QUANT_PRECLUSTER_HPP

#include <cstdint>
#include <span>
#include <vector>

#include "quant/color.hpp"
#include "quant/histogram.hpp"

namespace quant {

struct CoarseHistogram {
    static constexpr int grid = 32;
    static constexpr std::size_t bins = 32768;
    std::vector<std::uint64_t> count;
    std::vector<std::int64_t> sum_r, sum_g, sum_b, sum_sq; // original 8-bit values; sum_sq = r^2+g^2+b^2
    CoarseHistogram() : count(bins, 0), sum_r(bins, 0), sum_g(bins, 0), sum_b(bins, 0), sum_sq(bins, 0) {}
    static std::size_t bin_index(int br, int bg, int bb) {
        return (static_cast<std::size_t>(br) * grid + bg) * grid + bb;
    }
    static std::size_t bin_of(Rgb8 c) { return bin_index(c.r >> 3, c.g >> 3, c.b >> 3); }
};

CoarseHistogram build_coarse_histogram(std::span<const Rgb8> pixels);
CoarseHistogram build_coarse_histogram(const WeightedHistogram &hist);

} // namespace quant

#endif
