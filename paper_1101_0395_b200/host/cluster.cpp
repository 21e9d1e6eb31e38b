// cluster.cpp -- kmeans.hpp (reference include/quant/kmeans.hpp:17-130,
// src/kmeans.cpp). Clustering and the table / SSE / repair helpers run on the
// device; only the single-point searches below are host code (one point
// against at most K centres, the API's per-point contract).
#include <algorithm>
#include <cmath>

#include "context.hpp"

namespace quant {

using detail::check;
using detail::ctx;
using detail::flatten;
using detail::unflatten;

bool check_convergence(double sse_prev, double sse_cur, double epsilon) {
    return sse_cur == 0.0 || (sse_prev - sse_cur) / sse_cur <= epsilon;
}

CenterDistanceTable build_center_distance_table(std::span<const ColorPoint> centers) {
    CenterDistanceTable t;
    t.k = centers.size();
    t.dist2.resize(t.k * t.k);
    t.order.resize(t.k * t.k);
    if (t.k == 0) return t;
    const std::vector<double> c = flatten(centers);
    check(cqg_center_table(ctx(), c.data(), static_cast<int>(t.k), t.dist2.data(), t.order.data()));
    return t;
}

namespace {
// One pass over a walk row: the seed (previous label / hint) first, then the
// row's centres by increasing distance from it until the table distance
// reaches the cutoff 4 * d2(x, seed). `lowest_index` selects the mapping
// variant (break only on '>', equal distances go to the lower index,
// kmeans.cpp:81-105) over the assignment one (break on '>=', the incumbent
// keeps ties, kmeans.cpp:56-79).
std::uint32_t walk_row(const ColorPoint &x, std::uint32_t seed, const CenterDistanceTable &t,
                       std::span<const ColorPoint> c, std::uint64_t &ndc, bool lowest_index) {
    double best_d = dist2(x, c[seed]);
    std::uint32_t best = seed;
    ++ndc;
    const double cutoff = 4.0 * best_d;
    for (std::size_t pos = 1; pos < t.k; ++pos) {
        const std::uint32_t cand = t.order_at(seed, pos);
        const double dd = t.d2(seed, cand);
        if (lowest_index ? dd > cutoff : dd >= cutoff) break;
        const double d = dist2(x, c[cand]);
        ++ndc;
        if (d < best_d || (lowest_index && d == best_d && cand < best)) {
            best_d = d;
            best = cand;
        }
    }
    return best;
}
} // namespace

std::uint32_t nearest_full(const ColorPoint &x, std::span<const ColorPoint> centers, std::uint64_t &ndc) {
    std::uint32_t best = 0;
    double best_d = 0.0;
    for (std::size_t j = 0; j < centers.size(); ++j) {
        const double d = dist2(x, centers[j]);
        if (j == 0 || d < best_d) { // strict: the lowest index keeps ties
            best_d = d;
            best = static_cast<std::uint32_t>(j);
        }
    }
    ndc += centers.size();
    return best;
}

std::uint32_t assign_point_sortmeans(const ColorPoint &x, std::uint32_t prev, const CenterDistanceTable &table,
                                     std::span<const ColorPoint> centers, std::uint64_t &ndc) {
    return walk_row(x, prev, table, centers, ndc, false);
}

std::uint32_t nearest_pruned_lowest_index(const ColorPoint &x, std::uint32_t hint, const CenterDistanceTable &table,
                                          std::span<const ColorPoint> centers, std::uint64_t &ndc) {
    return walk_row(x, hint, table, centers, ndc, true);
}

namespace {
double sse_on_device(std::span<const ColorPoint> points, const double *weights, std::span<const ColorPoint> centers,
                     std::span<const std::uint32_t> memberships) {
    if (memberships.size() != points.size()) throw std::invalid_argument("compute_sse: memberships/points size mismatch");
    if (points.empty()) return 0.0;
    const std::vector<double> p = flatten(points), c = flatten(centers);
    double out = 0.0;
    check(cqg_compute_sse(ctx(), p.data(), weights, points.size(), c.data(), static_cast<int>(centers.size()),
                          memberships.data(), &out));
    return out;
}
} // namespace

double compute_sse(std::span<const ColorPoint> points, std::span<const double> weights,
                   std::span<const ColorPoint> centers, std::span<const std::uint32_t> memberships) {
    if (weights.size() != points.size()) throw std::invalid_argument("compute_sse: weights/points size mismatch");
    return sse_on_device(points, weights.data(), centers, memberships);
}

double compute_sse(std::span<const ColorPoint> points, std::span<const ColorPoint> centers,
                   std::span<const std::uint32_t> memberships) {
    return sse_on_device(points, nullptr, centers, memberships);
}

int repair_empty_clusters(std::span<const ColorPoint> points, std::span<const double> weights,
                          std::vector<ColorPoint> &centers, std::vector<std::uint32_t> &memberships) {
    if (centers.empty()) return 0;
    if (points.empty()) throw std::runtime_error("repair_empty_clusters: more clusters than points");
    if (weights.size() != points.size() || memberships.size() != points.size())
        throw std::invalid_argument("repair_empty_clusters: size mismatch");
    const std::vector<double> p = flatten(points);
    std::vector<double> c = flatten(centers);
    int repairs = 0;
    check(cqg_repair_empty_clusters(ctx(), p.data(), weights.data(), points.size(), c.data(),
                                    static_cast<int>(centers.size()), memberships.data(), &repairs));
    centers = unflatten(c.data(), centers.size());
    return repairs;
}

namespace {
// the general engine (cqg_lloyd_exact): wsm with weights, kmeans_full without
ClusterState lloyd_general(std::span<const ColorPoint> points, const double *weights, std::vector<ColorPoint> init,
                           const ClusterOptions &options) {
    const cqg_term term = detail::to_term(options);
    const std::size_t n = points.size(), k = init.size();
    const int limit = term.fixed_iterations > 0 ? term.fixed_iterations : std::max(term.max_iterations, 1);
    const std::vector<double> p = flatten(points), in = flatten(init);
    std::vector<double> cen(3 * std::max<std::size_t>(k, 1)), sse(limit), hc;
    std::vector<std::uint32_t> labels(std::max<std::size_t>(n, 1)), hl;
    if (options.record_history) {
        hl.resize(static_cast<std::size_t>(limit) * n);
        hc.resize(static_cast<std::size_t>(limit) * 3 * k);
    }
    cqg_lloyd_stats st{};
    check(cqg_lloyd_exact(ctx(), p.empty() ? nullptr : p.data(), weights, n, in.empty() ? nullptr : in.data(),
                          static_cast<int>(k), &term, cen.data(), labels.data(), sse.data(), &st,
                          hl.empty() ? nullptr : hl.data(), hc.empty() ? nullptr : hc.data()));
    return detail::make_state(cen, k, labels, n, sse, st, hl, hc);
}

// counts c_i with weights[i] == c_i * (1.0 / P) exactly and sum c_i == P
// (what build_histogram and the 'none' / '2to1' substrates produce), or P = 0
std::uint64_t decode_counts(std::span<const double> weights, std::vector<std::uint32_t> &counts) {
    const double wmin = *std::min_element(weights.begin(), weights.end());
    counts.assign(weights.size(), 0);
    for (int cmin = 1; cmin <= 256; ++cmin) {
        const double guess = std::nearbyint(cmin / wmin);
        if (!(guess >= 1.0 && guess < 18446744073709551615.0)) continue;
        const std::uint64_t P = static_cast<std::uint64_t>(guess);
        const double inv = 1.0 / static_cast<double>(P);
        std::uint64_t total = 0;
        bool ok = true;
        for (std::size_t i = 0; i < weights.size() && ok; ++i) {
            const double c = std::nearbyint(weights[i] * static_cast<double>(P));
            ok = c >= 1.0 && c <= 4294967295.0 && c * inv == weights[i];
            counts[i] = ok ? static_cast<std::uint32_t>(c) : 0u;
            total += counts[i];
        }
        if (ok && total == P) return P;
    }
    return 0;
}
} // namespace

ClusterState kmeans_full(std::span<const ColorPoint> points, std::vector<ColorPoint> init,
                         const ClusterOptions &options) {
    return lloyd_general(points, nullptr, std::move(init), options);
}

ClusterState wsm(std::span<const ColorPoint> points, std::span<const double> weights, std::vector<ColorPoint> init,
                 const ClusterOptions &options) {
    const std::size_t n = points.size(), k = init.size();
    if (k == 0) throw std::invalid_argument("clustering: no initial centers");
    if (n == 0) throw std::invalid_argument("clustering: no points");
    if (k > n)
        throw std::invalid_argument("clustering: k (" + std::to_string(k) + ") exceeds number of points (" +
                                    std::to_string(n) + ")");
    if (weights.size() != n) throw std::invalid_argument("clustering: weights/points size mismatch");
    for (double w : weights)
        if (!(w > 0.0)) throw std::invalid_argument("wsm: weights must be positive");
    std::vector<std::uint32_t> counts;
    const std::uint64_t P = detail::on_grid(points) ? decode_counts(weights, counts) : 0;
    if (P == 0) return lloyd_general(points, weights.data(), std::move(init), options);
    return detail::lloyd_counts(detail::pack_all(points), counts, P, init, options);
}

} // namespace quant
