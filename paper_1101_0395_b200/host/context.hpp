// context.hpp -- internal plumbing of libquant_b200.so: the calling thread's
// device context, C-ABI error -> exception translation and array packing.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "cqg.h"
#include "quant/quant.hpp"

namespace quant::detail {

// one cqg context per (host thread, device), created on first use
cqg_ctx *ctx();
int current_device(); // the calling thread's set_device value

// CQG_E_INVALID -> std::invalid_argument, everything else -> std::runtime_error,
// with the library's (the reference's) message text
inline void check(int rc) {
    if (rc == CQG_OK) return;
    const std::string msg = cqg_last_error();
    if (rc == CQG_E_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline std::uint32_t pack(const ColorPoint &c) {
    return (static_cast<std::uint32_t>(c.r) << 16) | (static_cast<std::uint32_t>(c.g) << 8) |
           static_cast<std::uint32_t>(c.b);
}
inline ColorPoint unpack(std::uint32_t c) {
    return {static_cast<double>((c >> 16) & 255u), static_cast<double>((c >> 8) & 255u),
            static_cast<double>(c & 255u)};
}
// true when every point is an 8-bit grid colour (the packed-colour engine's domain)
bool on_grid(std::span<const ColorPoint> pts);
std::vector<std::uint32_t> pack_all(std::span<const ColorPoint> pts);

inline std::vector<double> flatten(std::span<const ColorPoint> c) {
    std::vector<double> v(3 * c.size());
    for (std::size_t i = 0; i < c.size(); ++i) {
        v[3 * i] = c[i].r;
        v[3 * i + 1] = c[i].g;
        v[3 * i + 2] = c[i].b;
    }
    return v;
}
inline std::vector<ColorPoint> unflatten(const double *v, std::size_t k) {
    std::vector<ColorPoint> c(k);
    for (std::size_t i = 0; i < k; ++i) c[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    return c;
}

// Termination + record_history -> cqg_term (kmeans.cpp:187-188 message)
cqg_term to_term(const ClusterOptions &o);

// ClusterState from the device engines' flat outputs (history optional)
ClusterState make_state(const std::vector<double> &cen, std::size_t k, const std::vector<std::uint32_t> &labels,
                        std::size_t n, const std::vector<double> &sse, const cqg_lloyd_stats &st,
                        const std::vector<std::uint32_t> &hl, const std::vector<double> &hc);

// distinct colours of a pixel span on the device (cqg_histogram)
struct DeviceHist {
    std::vector<std::uint32_t> packed, counts;
    std::uint64_t P = 0;
};
DeviceHist device_hist(std::span<const Rgb8> pixels);

// the count-weighted hot-path engine (cqg_lloyd) on packed colours
ClusterState lloyd_counts(const std::vector<std::uint32_t> &packed, const std::vector<std::uint32_t> &counts,
                          std::uint64_t P, std::span<const ColorPoint> init, const ClusterOptions &options);

} // namespace quant::detail
