// histogram_api.cpp -- histogram.hpp and the coarse grid of precluster.hpp
// (reference src/histogram.cpp:19-104, src/precluster.cpp:13-47). The
// histogram and the coarse grid are built on the device; the hash parameters
// are drawn on the host only to fill WeightedHistogram::hash as the reference does.
#include <functional>

#include "context.hpp"

namespace quant {

using detail::check;
using detail::ctx;
using detail::pack;
using detail::unpack;

namespace detail {
DeviceHist device_hist(std::span<const Rgb8> pixels) {
    DeviceHist h;
    h.P = pixels.size();
    if (h.P == 0) throw std::invalid_argument("build_histogram: no pixels"); // histogram.cpp:70
    const std::size_t cap = std::min<std::size_t>(h.P, 1u << 24);
    h.packed.resize(cap);
    h.counts.resize(cap);
    std::uint64_t n = 0;
    check(cqg_histogram(ctx(), reinterpret_cast<const std::uint8_t *>(pixels.data()), h.P, h.packed.data(),
                        h.counts.data(), nullptr, &n));
    h.packed.resize(n);
    h.counts.resize(n);
    return h;
}
} // namespace detail

using detail::DeviceHist;
using detail::device_hist;

const char *sampling_mode_token(SamplingMode mode) {
    switch (mode) {
        case SamplingMode::None: return "none";
        case SamplingMode::TwoToOne: return "2to1";
        case SamplingMode::Unique: return "unique";
        case SamplingMode::TwoToOneUnique: return "both";
    }
    return "?";
}

SamplingMode parse_sampling_mode(const std::string &t) {
    if (t == "none") return SamplingMode::None;
    if (t == "2to1") return SamplingMode::TwoToOne;
    if (t == "unique") return SamplingMode::Unique;
    if (t == "both") return SamplingMode::TwoToOneUnique;
    throw std::invalid_argument("unknown sampling mode '" + t + "' (expected none|2to1|unique|both)");
}

std::uint64_t hash_color(Rgb8 c, const HashParams &p) {
    return (p.a[0] * c.r + p.a[1] * c.g + p.a[2] * c.b) % p.m;
}

std::uint64_t next_prime_at_least(std::uint64_t n) {
    if (n <= 2) return 2;
    for (std::uint64_t c = n | 1;; c += 2) {
        bool prime = true;
        for (std::uint64_t d = 3; d * d <= c; d += 2)
            if (c % d == 0) {
                prime = false;
                break;
            }
        if (prime) return c;
    }
}

HashParams make_hash_params(std::size_t pixel_count, Rng &rng) {
    if (pixel_count == 0) throw std::invalid_argument("make_hash_params: no pixels");
    HashParams p;
    p.m = next_prime_at_least(2 * static_cast<std::uint64_t>(pixel_count));
    do {
        for (auto &a : p.a) a = rng.next_below(p.m);
    } while (p.a[0] == 0 && p.a[1] == 0 && p.a[2] == 0);
    return p;
}

std::vector<Rgb8> subsample_2to1(const RawImage &image) {
    std::vector<Rgb8> out;
    for (int y = 0; y < image.height; y += 2)
        for (int x = 0; x < image.width; x += 2) out.push_back(image.at(x, y));
    return out;
}

WeightedHistogram build_histogram(std::span<const Rgb8> pixels, std::uint64_t seed) {
    const DeviceHist d = device_hist(pixels);
    WeightedHistogram h;
    h.source_pixel_count = d.P;
    Rng rng(seed); // the reference's hash coefficients (histogram.cpp:73-74), kept for API parity
    h.hash = make_hash_params(d.P, rng);
    const double inv = 1.0 / static_cast<double>(d.P);
    h.colors.reserve(d.packed.size());
    h.weights.reserve(d.packed.size());
    for (std::size_t i = 0; i < d.packed.size(); ++i) {
        h.colors.push_back(unpack(d.packed[i]));
        h.weights.push_back(static_cast<double>(d.counts[i]) * inv);
    }
    h.counts = d.counts;
    return h;
}

// ---- coarse histogram (precluster.cpp:13-47) on the device ----------------
namespace {
CoarseHistogram coarse_from_device(const std::function<int(std::int64_t *const *)> &call) {
    CoarseHistogram ch;
    std::int64_t *outs[5] = {reinterpret_cast<std::int64_t *>(ch.count.data()), ch.sum_r.data(), ch.sum_g.data(),
                             ch.sum_b.data(), ch.sum_sq.data()};
    check(call(outs));
    return ch;
}
} // namespace

CoarseHistogram build_coarse_histogram(std::span<const Rgb8> pixels) {
    if (pixels.empty()) throw std::invalid_argument("build_coarse_histogram: no pixels");
    return coarse_from_device([&](std::int64_t *const *o) {
        return cqg_coarse_histogram(ctx(), reinterpret_cast<const std::uint8_t *>(pixels.data()), pixels.size(),
                                    reinterpret_cast<std::uint64_t *>(o[0]), o[1], o[2], o[3], o[4]);
    });
}

CoarseHistogram build_coarse_histogram(const WeightedHistogram &hist) {
    if (hist.size() == 0) throw std::invalid_argument("build_coarse_histogram: empty histogram");
    std::vector<std::uint32_t> packed(hist.size());
    for (std::size_t i = 0; i < hist.size(); ++i) packed[i] = pack(hist.colors[i]);
    return coarse_from_device([&](std::int64_t *const *o) {
        return cqg_coarse_histogram_weighted(ctx(), packed.data(), hist.counts.data(), hist.size(),
                                             reinterpret_cast<std::uint64_t *>(o[0]), o[1], o[2], o[3], o[4]);
    });
}

} // namespace quant
