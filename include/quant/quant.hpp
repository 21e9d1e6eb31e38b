// quant/quant.hpp -- the reference quantiser's C++ API (namespace quant) for
// the device hot path, served by libquant_b200.so over the C-ABI in cqg.h.
//
// This header re-declares the subset of the reference's public headers that
// the hot path touches, with the same names, fields, signatures and exception
// behaviour (citations: /root/reference/proj/include/quant/*.hpp), so code
// written against the reference (e.g. its CLI or benchmark harness) can be
// relinked against this library:
//   color.hpp      Rgb8, ColorPoint, dist2, channel_to_u8, to_rgb8, Palette
//   rng.hpp        Rng (mt19937_64 + portable draws), weighted_draw
//   image.hpp      RawImage (image I/O is outside the device path)
//   histogram.hpp  SamplingMode, HashParams, WeightedHistogram, build_histogram
//   kmeans.hpp     Termination, ClusterOptions, ClusterState, wsm, ...
//   init.hpp       SeedConfig, init_maximin, init_kmeanspp
//   metrics.hpp    MappingResult, map_pixels, mse, psnr_from_mse, QuantReport
//   pipeline.hpp   MethodSpec, parse_method, QuantizeConfig, run_quantize
// The per-point helpers (nearest_full, assign_point_sortmeans, ...) and the
// centre table are small host utilities kept for API compatibility; the data
// path (histogram, initialisation, Lloyd, mapping) always runs on the GPU.
#pragma once

#include <cmath>
#include <cstdint>
#include <optional>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace quant {

// ---- color.hpp:10-82 ------------------------------------------------------
struct Rgb8 {
    std::uint8_t r = 0, g = 0, b = 0;
    friend bool operator==(const Rgb8 &x, const Rgb8 &y) { return x.r == y.r && x.g == y.g && x.b == y.b; }
};

struct ColorPoint {
    double r = 0.0, g = 0.0, b = 0.0;
    ColorPoint() = default;
    ColorPoint(double r_, double g_, double b_) : r(r_), g(g_), b(b_) {}
    explicit ColorPoint(Rgb8 c) : r(c.r), g(c.g), b(c.b) {}
    ColorPoint &operator+=(const ColorPoint &o) { r += o.r; g += o.g; b += o.b; return *this; }
    friend ColorPoint operator+(ColorPoint x, const ColorPoint &y) { return x += y; }
    friend ColorPoint operator-(const ColorPoint &x, const ColorPoint &y) { return {x.r - y.r, x.g - y.g, x.b - y.b}; }
    friend ColorPoint operator*(const ColorPoint &x, double s) { return {x.r * s, x.g * s, x.b * s}; }
    friend bool operator==(const ColorPoint &x, const ColorPoint &y) { return x.r == y.r && x.g == y.g && x.b == y.b; }
};

double dist2(const ColorPoint &a, const ColorPoint &b);
double dist2(const ColorPoint &a, const Rgb8 &b);
std::uint8_t channel_to_u8(double v);
Rgb8 to_rgb8(const ColorPoint &c);

struct Palette {
    std::vector<ColorPoint> colors;
    bool truncated = false;
    std::size_t size() const { return colors.size(); }
};

// ---- rng.hpp:17-54 --------------------------------------------------------
class Rng {
  public:
    explicit Rng(std::uint64_t seed) : gen_(seed) {}
    std::uint64_t next_u64() { return gen_(); }
    std::uint64_t next_below(std::uint64_t n);
    double next_unit() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }

  private:
    std::mt19937_64 gen_;
};

std::size_t weighted_draw(std::span<const double> mass, Rng &rng);

// ---- image.hpp:13-24 ------------------------------------------------------
struct RawImage {
    int width = 0;
    int height = 0;
    std::vector<Rgb8> pixels;
    std::size_t pixel_count() const { return pixels.size(); }
    Rgb8 &at(int x, int y) { return pixels[static_cast<std::size_t>(y) * width + x]; }
    const Rgb8 &at(int x, int y) const { return pixels[static_cast<std::size_t>(y) * width + x]; }
};

// image.hpp:26-44: PPM (P6, maxval 255) on the host; PNG needs libpng, which
// this build does not link (load/save report it as unsupported).
struct LoadedImage {
    RawImage image;
    std::vector<std::string> warnings;
};
LoadedImage load_image(const std::string &path);
void save_image(const RawImage &image, const std::string &path);
void save_ppm(const RawImage &image, const std::string &path);

// ---- histogram.hpp:19-60 --------------------------------------------------
enum class SamplingMode { None, TwoToOne, Unique, TwoToOneUnique };
const char *sampling_mode_token(SamplingMode mode);
SamplingMode parse_sampling_mode(const std::string &token);

struct HashParams {
    std::uint64_t a[3] = {1, 1, 1};
    std::uint64_t m = 1;
};
std::uint64_t hash_color(Rgb8 c, const HashParams &p);
std::uint64_t next_prime_at_least(std::uint64_t n);
HashParams make_hash_params(std::size_t pixel_count, Rng &rng);

struct WeightedHistogram {
    std::vector<ColorPoint> colors;
    std::vector<double> weights;
    std::vector<std::uint32_t> counts;
    std::size_t source_pixel_count = 0;
    HashParams hash;
    std::size_t size() const { return colors.size(); }
};

std::vector<Rgb8> subsample_2to1(const RawImage &image);
WeightedHistogram build_histogram(std::span<const Rgb8> pixels, std::uint64_t seed);

// ---- kmeans.hpp:17-129 ----------------------------------------------------
struct Termination {
    double epsilon = 1e-3;
    int max_iterations = 100;
    std::optional<int> fixed_iterations;
};
bool check_convergence(double sse_prev, double sse_cur, double epsilon);

struct ClusterOptions {
    Termination term;
    bool record_history = false;
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
    std::vector<double> dist2;
    std::vector<std::uint32_t> order;
    double d2(std::size_t i, std::size_t j) const { return dist2[i * k + j]; }
    std::uint32_t order_at(std::size_t i, std::size_t n) const { return order[i * k + n]; }
};

// host utilities (single points / K x K), kept for API compatibility
CenterDistanceTable build_center_distance_table(std::span<const ColorPoint> centers);
std::uint32_t nearest_full(const ColorPoint &x, std::span<const ColorPoint> centers, std::uint64_t &ndc);
std::uint32_t assign_point_sortmeans(const ColorPoint &x, std::uint32_t prev, const CenterDistanceTable &table,
                                     std::span<const ColorPoint> centers, std::uint64_t &ndc);
std::uint32_t nearest_pruned_lowest_index(const ColorPoint &x, std::uint32_t hint, const CenterDistanceTable &table,
                                          std::span<const ColorPoint> centers, std::uint64_t &ndc);
double compute_sse(std::span<const ColorPoint> points, std::span<const double> weights,
                   std::span<const ColorPoint> centers, std::span<const std::uint32_t> memberships);

// Weighted sort-means on the device. The device keeps exact integer moments,
// so the substrate must be count-weighted: points on the 8-bit grid and
// weights[i] == count_i * (1.0 / P) for integer counts summing to P (every
// substrate run_quantize builds); other inputs throw std::invalid_argument.
ClusterState wsm(std::span<const ColorPoint> points, std::span<const double> weights,
                 std::vector<ColorPoint> init, const ClusterOptions &options);
// Same, straight from a histogram (no weight decoding).
ClusterState wsm(const WeightedHistogram &hist, std::vector<ColorPoint> init, const ClusterOptions &options);

// ---- init.hpp:17-72 -------------------------------------------------------
struct SeedConfig {
    int k = 8;
    std::uint64_t seed = 1;
    ColorPoint lbg_perturbation{0.255, 0.255, 0.255};
    Termination lbg_refine{};
    int density_grid = 8;
    bool maximin_weighted_first = true;
};
std::vector<ColorPoint> init_maximin(const WeightedHistogram &hist, const SeedConfig &cfg);
std::vector<ColorPoint> init_kmeanspp(const WeightedHistogram &hist, const SeedConfig &cfg);

// ---- precluster.hpp:16-34: the coarse grid the preclusterers read -------
struct CoarseHistogram {
    static constexpr int grid = 32;
    static constexpr std::size_t bins = 32768;
    std::vector<std::uint64_t> count;
    std::vector<std::int64_t> sum_r, sum_g, sum_b, sum_sq;
    CoarseHistogram() : count(bins, 0), sum_r(bins, 0), sum_g(bins, 0), sum_b(bins, 0), sum_sq(bins, 0) {}
    static std::size_t bin_index(int br, int bg, int bb) {
        return (static_cast<std::size_t>(br) * grid + bg) * grid + bb;
    }
    static std::size_t bin_of(Rgb8 c) { return bin_index(c.r >> 3, c.g >> 3, c.b >> 3); }
};
// on the device (cqg_coarse_histogram / _weighted)
CoarseHistogram build_coarse_histogram(std::span<const Rgb8> pixels);
CoarseHistogram build_coarse_histogram(const WeightedHistogram &hist);

// ---- metrics.hpp:14-57 ----------------------------------------------------
struct MappingResult {
    std::vector<std::uint32_t> indices;
    RawImage quantized;
    double mean_sq_dist = 0.0;
    std::uint64_t ndc = 0;
};
MappingResult map_pixels(const RawImage &image, const Palette &palette);
double mse(const RawImage &a, const RawImage &b);
double psnr_from_mse(double mse_value);

struct QuantReport {
    std::string image;
    std::string method;
    int k_requested = 0;
    int k_actual = 0;
    int run = 0;
    std::uint64_t seed = 0;
    SamplingMode sampling = SamplingMode::Unique;
    double mse = 0.0;
    double psnr = 0.0;
    int iterations = 0;
    double ndc_per_point_iter = 0.0;
    double time_ms = 0.0;
    std::vector<std::string> flags;
    std::string to_json() const;
    static const char *csv_header();
    std::string csv_row() const;
};

// ---- pipeline.hpp:19-53 ---------------------------------------------------
struct MethodSpec {
    bool refine = false;
    std::string base;
    std::string token() const { return refine ? "wsm-" + base : base; }
};
MethodSpec parse_method(const std::string &method, const std::string &init = "");
std::vector<std::string> all_method_tokens();

struct QuantizeConfig {
    MethodSpec method;
    int k = 8;
    SamplingMode sampling = SamplingMode::Unique;
    std::uint64_t seed = 1;
    Termination term;
    bool record_history = false;
    // Extension of this build: initial centres for initialisers outside the
    // device path (e.g. a preclusterer palette for "wsm-wu"); empty = use the
    // method's own device initialiser (mmx, kpp).
    std::vector<ColorPoint> init_centers;
};

struct QuantizeResult {
    Palette palette;
    MappingResult mapping;
    ClusterState state;
    QuantReport report;
    std::size_t substrate_points = 0;
};

QuantizeResult run_quantize(const RawImage &image, const QuantizeConfig &config);

// Device selection for the calling thread (default 0).
void set_device(int device);

} // namespace quant
