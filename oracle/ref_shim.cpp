// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libquantref.so).
// It lets the pytest suite, the golden-fixture generator and bench.py's
// reference arm drive the reference's own public API (quant::build_histogram,
// init_maximin / init_kmeanspp, wsm, map_pixels, run_quantize) on the same
// bytes the device path sees. No reference source is copied here; this file
// only includes the reference headers in place.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "quant/histogram.hpp"
#include "quant/init.hpp"
#include "quant/kmeans.hpp"
#include "quant/metrics.hpp"
#include "quant/pipeline.hpp"
#include "quant/precluster.hpp"
#include "test_support.hpp"

using namespace quant;

namespace {
thread_local std::string g_err;

int fail(const std::exception &e) {
    g_err = e.what();
    return -1;
}

RawImage make_image(const std::uint8_t *rgb, int w, int h) {
    RawImage img;
    img.width = w;
    img.height = h;
    img.pixels.resize(static_cast<std::size_t>(w) * h);
    std::memcpy(img.pixels.data(), rgb, img.pixels.size() * 3);
    return img;
}

// Histogram object equal to what build_histogram would return for these
// colours/counts (weights = count * (1/P), histogram.cpp:99-102).
WeightedHistogram make_hist(const std::uint32_t *colors, const std::uint32_t *counts, std::uint64_t n,
                            std::uint64_t P) {
    WeightedHistogram h;
    h.source_pixel_count = P;
    const double inv = 1.0 / static_cast<double>(P);
    for (std::uint64_t i = 0; i < n; ++i) {
        h.colors.emplace_back(static_cast<double>((colors[i] >> 16) & 255),
                              static_cast<double>((colors[i] >> 8) & 255),
                              static_cast<double>(colors[i] & 255));
        h.counts.push_back(counts[i]);
        h.weights.push_back(static_cast<double>(counts[i]) * inv);
    }
    return h;
}
} // namespace

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }

int ref_synthetic_photo(int w, int h, std::uint64_t seed, std::uint8_t *out) {
    RawImage img = testsup::synthetic_photo(w, h, seed);
    std::memcpy(out, img.pixels.data(), img.pixels.size() * 3);
    return 0;
}

std::int64_t ref_histogram(const std::uint8_t *rgb, std::uint64_t P, std::uint64_t seed,
                           std::uint32_t *colors, std::uint32_t *counts, double *weights) {
    try {
        std::vector<Rgb8> px(P);
        std::memcpy(px.data(), rgb, P * 3);
        WeightedHistogram h = build_histogram(px, seed);
        for (std::size_t i = 0; i < h.size(); ++i) {
            colors[i] = (static_cast<std::uint32_t>(h.colors[i].r) << 16) |
                        (static_cast<std::uint32_t>(h.colors[i].g) << 8) |
                        static_cast<std::uint32_t>(h.colors[i].b);
            counts[i] = h.counts[i];
            if (weights) weights[i] = h.weights[i];
        }
        return static_cast<std::int64_t>(h.size());
    } catch (const std::exception &e) {
        return fail(e);
    }
}

// quant::build_coarse_histogram (precluster.hpp:32-34), both overloads:
// from pixels (colors == nullptr) or from a weighted histogram. out: 5 x 32768
// (count | sum_r | sum_g | sum_b | sum_sq, as int64 bit patterns).
int ref_coarse_histogram(const std::uint8_t *rgb, std::uint64_t P, const std::uint32_t *colors,
                         const std::uint32_t *counts, std::uint64_t n, std::int64_t *out) {
    try {
        CoarseHistogram ch;
        if (!colors) {
            std::vector<Rgb8> px(P);
            if (P) std::memcpy(px.data(), rgb, P * 3);
            ch = build_coarse_histogram(std::span<const Rgb8>(px));
        } else {
            std::uint64_t total = 0;
            for (std::uint64_t i = 0; i < n; ++i) total += counts[i];
            ch = build_coarse_histogram(make_hist(colors, counts, n, total ? total : 1));
        }
        for (std::size_t b = 0; b < CoarseHistogram::bins; ++b) {
            out[b] = static_cast<std::int64_t>(ch.count[b]);
            out[CoarseHistogram::bins + b] = ch.sum_r[b];
            out[2 * CoarseHistogram::bins + b] = ch.sum_g[b];
            out[3 * CoarseHistogram::bins + b] = ch.sum_b[b];
            out[4 * CoarseHistogram::bins + b] = ch.sum_sq[b];
        }
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

// kind: 0 = mmx, 1 = kpp, 2 = wu (preclusterer palette, padded by maximin_pad)
int ref_init(int kind, const std::uint32_t *colors, const std::uint32_t *counts, std::uint64_t n,
             std::uint64_t P, int k, std::uint64_t seed, double *centers, int *k_out) {
    try {
        WeightedHistogram h = make_hist(colors, counts, n, P);
        SeedConfig cfg;
        cfg.k = k;
        cfg.seed = seed;
        std::vector<ColorPoint> c;
        if (kind == 0) c = init_maximin(h, cfg);
        else if (kind == 1) c = init_kmeanspp(h, cfg);
        else {
            Palette p = wu_quantize(build_coarse_histogram(h), k);
            c = p.colors;
            if (static_cast<int>(c.size()) < k) c = maximin_pad(h, std::move(c), k);
        }
        for (std::size_t i = 0; i < c.size(); ++i) {
            centers[3 * i] = c[i].r;
            centers[3 * i + 1] = c[i].g;
            centers[3 * i + 2] = c[i].b;
        }
        *k_out = static_cast<int>(c.size());
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_wsm(const std::uint32_t *colors, const std::uint32_t *counts, std::uint64_t n, std::uint64_t P,
            const double *init, int k, double eps, int max_it, int fixed_it, double *centers_out,
            std::uint32_t *labels_out, double *sse_trace, int *iters, std::uint64_t *ndc,
            int *repairs, std::uint32_t *hist_labels, double *hist_centers, double *seconds) {
    try {
        WeightedHistogram h = make_hist(colors, counts, n, P);
        std::vector<ColorPoint> c0;
        for (int i = 0; i < k; ++i) c0.emplace_back(init[3 * i], init[3 * i + 1], init[3 * i + 2]);
        ClusterOptions opt;
        opt.term.epsilon = eps;
        opt.term.max_iterations = max_it;
        if (fixed_it > 0) opt.term.fixed_iterations = fixed_it;
        opt.record_history = hist_labels != nullptr || hist_centers != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        ClusterState st = wsm(h.colors, h.weights, std::move(c0), opt);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        for (int i = 0; i < k; ++i) {
            centers_out[3 * i] = st.centers[i].r;
            centers_out[3 * i + 1] = st.centers[i].g;
            centers_out[3 * i + 2] = st.centers[i].b;
        }
        std::memcpy(labels_out, st.memberships.data(), n * 4);
        for (std::size_t i = 0; i < st.sse_trace.size(); ++i) sse_trace[i] = st.sse_trace[i];
        *iters = st.iterations;
        *ndc = st.ndc_total;
        *repairs = st.repair_count;
        for (std::size_t it = 0; it < st.history.size(); ++it) {
            if (hist_labels) std::memcpy(hist_labels + it * n, st.history[it].memberships.data(), n * 4);
            if (hist_centers)
                for (int i = 0; i < k; ++i) {
                    hist_centers[(it * k + i) * 3] = st.history[it].centers[i].r;
                    hist_centers[(it * k + i) * 3 + 1] = st.history[it].centers[i].g;
                    hist_centers[(it * k + i) * 3 + 2] = st.history[it].centers[i].b;
                }
        }
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_map_pixels(const std::uint8_t *rgb, int w, int h, const double *pal, int k,
                   std::uint32_t *indices, std::uint8_t *quant, double *mse, std::uint64_t *ndc,
                   double *seconds) {
    try {
        RawImage img = make_image(rgb, w, h);
        Palette p;
        for (int i = 0; i < k; ++i) p.colors.emplace_back(pal[3 * i], pal[3 * i + 1], pal[3 * i + 2]);
        const auto t0 = std::chrono::steady_clock::now();
        MappingResult m = map_pixels(img, p);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (indices) std::memcpy(indices, m.indices.data(), m.indices.size() * 4);
        if (quant) std::memcpy(quant, m.quantized.pixels.data(), m.quantized.pixels.size() * 3);
        *mse = m.mean_sq_dist;
        if (ndc) *ndc = m.ndc;
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

// Full reference pipeline; csv (>= 512 bytes) receives QuantReport::csv_row()
// with image name `name` and time_ms forced to 0 (bench zero_time, bench.cpp:87).
// stage_s (nullable, 4 doubles) receives histogram / init / wsm / map seconds
// measured by re-running the public stages separately (bench cpu baseline).
int ref_run_quantize_s(const std::uint8_t *rgb, int w, int h, const char *method, int k,
                       std::uint64_t seed, double eps, int max_it, int fixed_it, const char *name,
                       int run, double *palette, int *k_actual, int *iters, double *ndc_ppi,
                       double *mse, double *time_ms, char *csv, std::uint32_t *indices,
                       std::uint8_t *quant, const char *sampling);

int ref_run_quantize(const std::uint8_t *rgb, int w, int h, const char *method, int k,
                     std::uint64_t seed, double eps, int max_it, int fixed_it, const char *name,
                     int run, double *palette, int *k_actual, int *iters, double *ndc_ppi,
                     double *mse, double *time_ms, char *csv, std::uint32_t *indices,
                     std::uint8_t *quant) {
    return ref_run_quantize_s(rgb, w, h, method, k, seed, eps, max_it, fixed_it, name, run, palette, k_actual,
                              iters, ndc_ppi, mse, time_ms, csv, indices, quant, "unique");
}

// run_quantize with QuantizeConfig::sampling given by its token (none|2to1|unique|both)
int ref_run_quantize_s(const std::uint8_t *rgb, int w, int h, const char *method, int k,
                       std::uint64_t seed, double eps, int max_it, int fixed_it, const char *name,
                       int run, double *palette, int *k_actual, int *iters, double *ndc_ppi,
                       double *mse, double *time_ms, char *csv, std::uint32_t *indices,
                       std::uint8_t *quant, const char *sampling) {
    try {
        RawImage img = make_image(rgb, w, h);
        QuantizeConfig cfg;
        cfg.sampling = parse_sampling_mode(sampling ? sampling : "unique");
        cfg.method = parse_method(method);
        cfg.k = k;
        cfg.seed = seed;
        cfg.term.epsilon = eps;
        cfg.term.max_iterations = max_it;
        if (fixed_it > 0) cfg.term.fixed_iterations = fixed_it;
        QuantizeResult r = run_quantize(img, cfg);
        for (std::size_t i = 0; i < r.palette.size(); ++i) {
            palette[3 * i] = r.palette.colors[i].r;
            palette[3 * i + 1] = r.palette.colors[i].g;
            palette[3 * i + 2] = r.palette.colors[i].b;
        }
        *k_actual = r.report.k_actual;
        *iters = r.report.iterations;
        *ndc_ppi = r.report.ndc_per_point_iter;
        *mse = r.report.mse;
        *time_ms = r.report.time_ms;
        if (indices) std::memcpy(indices, r.mapping.indices.data(), r.mapping.indices.size() * 4);
        if (quant) std::memcpy(quant, r.mapping.quantized.pixels.data(), r.mapping.quantized.pixels.size() * 3);
        if (csv) {
            QuantReport rep = r.report;
            rep.image = name ? name : "";
            rep.run = run;
            rep.time_ms = 0.0;
            const std::string row = rep.csv_row();
            std::strncpy(csv, row.c_str(), 511);
            csv[511] = 0;
        }
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

// Stage-timed reference pipeline for the CPU baseline: build_histogram,
// init_maximin/init_kmeanspp, wsm, map_pixels, each through the public API.
int ref_time_pipeline(const std::uint8_t *rgb, int w, int h, int init_kind, int k, std::uint64_t seed,
                      double eps, int max_it, int fixed_it, double *stage_s, std::uint64_t *n_unique,
                      int *iters, double *mse) {
    try {
        using clk = std::chrono::steady_clock;
        RawImage img = make_image(rgb, w, h);
        const auto t0 = clk::now();
        WeightedHistogram hist = build_histogram(img.pixels, seed);
        const auto t1 = clk::now();
        SeedConfig sc;
        sc.k = k;
        sc.seed = seed;
        std::vector<ColorPoint> init = init_kind == 1 ? init_kmeanspp(hist, sc) : init_maximin(hist, sc);
        const auto t2 = clk::now();
        ClusterOptions opt;
        opt.term.epsilon = eps;
        opt.term.max_iterations = max_it;
        if (fixed_it > 0) opt.term.fixed_iterations = fixed_it;
        ClusterState st = wsm(hist.colors, hist.weights, std::move(init), opt);
        const auto t3 = clk::now();
        Palette pal;
        pal.colors = st.centers;
        MappingResult m = map_pixels(img, pal);
        const auto t4 = clk::now();
        stage_s[0] = std::chrono::duration<double>(t1 - t0).count();
        stage_s[1] = std::chrono::duration<double>(t2 - t1).count();
        stage_s[2] = std::chrono::duration<double>(t3 - t2).count();
        stage_s[3] = std::chrono::duration<double>(t4 - t3).count();
        *n_unique = hist.size();
        *iters = st.iterations;
        *mse = m.mean_sq_dist;
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

} // extern "C"

// ---- the general API: real points, arbitrary weights (kmeans.hpp / init.hpp)
namespace {
std::vector<ColorPoint> pts_of(const double *p, std::uint64_t n) {
    std::vector<ColorPoint> v;
    v.reserve(n);
    for (std::uint64_t i = 0; i < n; ++i) v.emplace_back(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
    return v;
}
void put_pts(const std::vector<ColorPoint> &v, double *out) {
    for (std::size_t i = 0; i < v.size(); ++i) {
        out[3 * i] = v[i].r;
        out[3 * i + 1] = v[i].g;
        out[3 * i + 2] = v[i].b;
    }
}
WeightedHistogram hist_of(const double *colors, const double *weights, std::uint64_t n) {
    WeightedHistogram h;
    h.colors = pts_of(colors, n);
    h.weights.assign(weights, weights + n);
    h.counts.assign(n, 1);
    h.source_pixel_count = n;
    return h;
}
} // namespace

extern "C" {
// wsm(points, weights, ...) or, with weights == NULL, kmeans_full(points, ...)
int ref_lloyd_general(const double *points, const double *weights, std::uint64_t n, const double *init, int k,
                      double eps, int max_it, int fixed_it, double *centers_out, std::uint32_t *labels_out,
                      double *sse_trace, int *iters, std::uint64_t *ndc, int *repairs, std::uint32_t *hist_labels,
                      double *hist_centers) {
    try {
        const std::vector<ColorPoint> pts = pts_of(points, n);
        std::vector<ColorPoint> c0 = pts_of(init, static_cast<std::uint64_t>(k));
        ClusterOptions opt;
        opt.term.epsilon = eps;
        opt.term.max_iterations = max_it;
        if (fixed_it > 0) opt.term.fixed_iterations = fixed_it;
        opt.record_history = hist_labels != nullptr || hist_centers != nullptr;
        ClusterState st = weights ? wsm(pts, std::span<const double>(weights, n), std::move(c0), opt)
                                  : kmeans_full(pts, std::move(c0), opt);
        put_pts(st.centers, centers_out);
        std::memcpy(labels_out, st.memberships.data(), n * 4);
        for (std::size_t i = 0; i < st.sse_trace.size(); ++i) sse_trace[i] = st.sse_trace[i];
        *iters = st.iterations;
        *ndc = st.ndc_total;
        *repairs = st.repair_count;
        for (std::size_t it = 0; it < st.history.size(); ++it) {
            if (hist_labels) std::memcpy(hist_labels + it * n, st.history[it].memberships.data(), n * 4);
            if (hist_centers) put_pts(st.history[it].centers, hist_centers + it * 3 * k);
        }
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_compute_sse(const double *points, const double *weights, std::uint64_t n, const double *centers, int k,
                    const std::uint32_t *labels, double *out) {
    try {
        const std::vector<ColorPoint> pts = pts_of(points, n), c = pts_of(centers, static_cast<std::uint64_t>(k));
        std::span<const std::uint32_t> m(labels, n);
        *out = weights ? compute_sse(pts, std::span<const double>(weights, n), c, m) : compute_sse(pts, c, m);
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_repair(const double *points, const double *weights, std::uint64_t n, double *centers, int k,
               std::uint32_t *labels, int *repairs) {
    try {
        const std::vector<ColorPoint> pts = pts_of(points, n);
        std::vector<ColorPoint> c = pts_of(centers, static_cast<std::uint64_t>(k));
        std::vector<std::uint32_t> m(labels, labels + n);
        *repairs = repair_empty_clusters(pts, std::span<const double>(weights, n), c, m);
        put_pts(c, centers);
        std::memcpy(labels, m.data(), n * 4);
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_center_table(const double *centers, int k, double *dist, std::uint32_t *order) {
    try {
        const std::vector<ColorPoint> c = pts_of(centers, static_cast<std::uint64_t>(k));
        const CenterDistanceTable t = build_center_distance_table(c);
        std::memcpy(dist, t.dist2.data(), t.dist2.size() * 8);
        std::memcpy(order, t.order.data(), t.order.size() * 4);
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_next_masses(const double *colors, const double *weights, std::uint64_t n, const double *centers, int k,
                    double *masses) {
    try {
        const WeightedHistogram h = hist_of(colors, weights, n);
        const std::vector<ColorPoint> c = pts_of(centers, static_cast<std::uint64_t>(k));
        const std::vector<double> m = kmeanspp_next_masses(h, c);
        std::memcpy(masses, m.data(), m.size() * 8);
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}

int ref_maximin_pad(const double *colors, const double *weights, std::uint64_t n, const double *centers, int k0,
                    int k, double *out, int *k_out) {
    try {
        const WeightedHistogram h = hist_of(colors, weights, n);
        std::vector<ColorPoint> c = pts_of(centers, static_cast<std::uint64_t>(k0));
        const std::vector<ColorPoint> r = maximin_pad(h, std::move(c), k);
        put_pts(r, out);
        *k_out = static_cast<int>(r.size());
        return 0;
    } catch (const std::exception &e) {
        return fail(e);
    }
}
} // extern "C"
