// quant/kmeans.hpp -- drop-in for /root/reference/proj/include/quant/kmeans.hpp:17-130.
//
// wsm over count-weighted points on the 8-bit grid (what run_quantize and
// build_histogram produce: weights[i] == count_i * (1/P)) runs on the hot-path
// engine (cqg_lloyd: FP32 sweep + exact FP64 replay, exact integer moments).
// Any other points or positive weights, and kmeans_full, run on the general
// device engine (cqg_lloyd_exact), which reproduces the reference's sequential
// FP64 sums in order. build_center_distance_table, compute_sse and
// repair_empty_clusters are device calls too; the three single-point search
// helpers are host functions (one point, at most K distances).
#ifndef QUANT_KMEANS_HPP
#define QUANT_KMEANS_HPP

#include <cstdint>
#include <optional>
#include <span>
#include <vector>

#include "quant/color.hpp"

namespace quant {

struct Termination {
    double epsilon = 1e-3;                // stop when (sse_prev - sse) / sse <= epsilon
    int max_iterations = 100;
    std::optional<int> fixed_iterations;  // overrides both when set
};

bool check_convergence(double sse_prev, double sse_cur, double epsilon);

struct ClusterOptions {
    Termination term;
    bool record_history = false; // per-iteration centres + pre-repair memberships
};

struct IterationSnapshot {
    std::vector<ColorPoint> centers;
    std::vector<std::uint32_t> memberships;
};

struct ClusterState {
    std::vector<ColorPoint> centers;
    std::vector<std::uint32_t> memberships;
    std::vector<double> sse_trace;
    int iterations = 0;
    std::uint64_t ndc_total = 0;
    int repair_count = 0;
    std::vector<IterationSnapshot> history;

    double ndc_per_point_iter(std::size_t point_count) const {
        if (point_count == 0 || iterations == 0) return 0.0;
        return static_cast<double>(ndc_total) / (static_cast<double>(point_count) * static_cast<double>(iterations));
    }
};

struct CenterDistanceTable {
    std::size_t k = 0;
    std::vector<double> dist2;        // k x k, row-major
    std::vector<std::uint32_t> order; // k x k, row i by increasing distance, order[i*k] == i
    double d2(std::size_t i, std::size_t j) const { return dist2[i * k + j]; }
    std::uint32_t order_at(std::size_t i, std::size_t n) const { return order[i * k + n]; }
};

CenterDistanceTable build_center_distance_table(std::span<const ColorPoint> centers);

std::uint32_t nearest_full(const ColorPoint &x, std::span<const ColorPoint> centers, std::uint64_t &ndc);
std::uint32_t assign_point_sortmeans(const ColorPoint &x, std::uint32_t prev, const CenterDistanceTable &table,
                                     std::span<const ColorPoint> centers, std::uint64_t &ndc);
std::uint32_t nearest_pruned_lowest_index(const ColorPoint &x, std::uint32_t hint, const CenterDistanceTable &table,
                                          std::span<const ColorPoint> centers, std::uint64_t &ndc);

double compute_sse(std::span<const ColorPoint> points, std::span<const double> weights,
                   std::span<const ColorPoint> centers, std::span<const std::uint32_t> memberships);
double compute_sse(std::span<const ColorPoint> points, std::span<const ColorPoint> centers,
                   std::span<const std::uint32_t> memberships);

int repair_empty_clusters(std::span<const ColorPoint> points, std::span<const double> weights,
                          std::vector<ColorPoint> &centers, std::vector<std::uint32_t> &memberships);

ClusterState kmeans_full(std::span<const ColorPoint> points, std::vector<ColorPoint> init,
                         const ClusterOptions &options);

ClusterState wsm(std::span<const ColorPoint> points, std::span<const double> weights, std::vector<ColorPoint> init,
                 const ClusterOptions &options);

} // namespace quant

#endif
