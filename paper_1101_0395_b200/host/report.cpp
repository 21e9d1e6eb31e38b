// report.cpp -- metrics.hpp and pipeline.hpp (reference src/metrics.cpp:15-150,
// src/pipeline.cpp:20-164). map_pixels and run_quantize run on the device
// (cqg_map, cqg_quantize); the report formats are frozen CSV / JSON.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <limits>

#include "context.hpp"

namespace quant {

using detail::check;
using detail::ctx;
using detail::flatten;
using detail::unflatten;

// ---- metrics (metrics.cpp) ------------------------------------------------
MappingResult map_pixels(const RawImage &image, const Palette &palette) {
    if (palette.colors.empty()) throw std::invalid_argument("map_pixels: empty palette");
    if (image.pixels.empty()) throw std::invalid_argument("map_pixels: empty image");
    MappingResult out;
    const std::size_t P = image.pixel_count();
    out.indices.resize(P);
    out.quantized.width = image.width;
    out.quantized.height = image.height;
    out.quantized.pixels.resize(P);
    const std::vector<double> pal = flatten(palette.colors);
    check(cqg_map(ctx(), reinterpret_cast<const std::uint8_t *>(image.pixels.data()), P, pal.data(),
                  static_cast<int>(palette.size()), out.indices.data(), 4,
                  reinterpret_cast<std::uint8_t *>(out.quantized.pixels.data()), &out.mean_sq_dist, &out.ndc));
    return out;
}

double mse(const RawImage &a, const RawImage &b) {
    if (a.width != b.width || a.height != b.height) throw std::invalid_argument("mse: image dimensions differ");
    if (a.pixels.empty()) throw std::invalid_argument("mse: empty images");
    std::uint64_t s = 0;
    for (std::size_t i = 0; i < a.pixels.size(); ++i) {
        const int dr = a.pixels[i].r - b.pixels[i].r, dg = a.pixels[i].g - b.pixels[i].g,
                  db = a.pixels[i].b - b.pixels[i].b;
        s += static_cast<std::uint64_t>(dr * dr + dg * dg + db * db);
    }
    return static_cast<double>(s) / static_cast<double>(a.pixels.size());
}

double psnr_from_mse(double v) {
    if (v < 0.0) throw std::invalid_argument("psnr_from_mse: negative mse");
    if (v == 0.0) return std::numeric_limits<double>::infinity();
    return 20.0 * std::log10(255.0 / std::sqrt(v));
}

namespace {
std::string fmt(const char *spec, double v) {
    char b[64];
    std::snprintf(b, sizeof b, spec, v);
    return b;
}
std::string jstr(const std::string &s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}
std::string jnum(double v) {
    if (std::isnan(v)) return "null";
    return fmt("%.17g", v);
}
} // namespace

const char *QuantReport::csv_header() {
    return "image,method,k,run,seed,sampling,mse,psnr,iterations,ndc_per_point_iter,time_ms,actual_k,flags";
}

std::string QuantReport::csv_row() const { // metrics.cpp:121-150
    std::string flagstr;
    for (const auto &f : flags) flagstr += (flagstr.empty() ? "" : ";") + f;
    std::string r = image + "," + method + "," + std::to_string(k_requested) + "," + std::to_string(run) + "," +
                    std::to_string(seed) + "," + sampling_mode_token(sampling) + ",";
    r += std::isnan(mse) ? "nan" : fmt("%.6f", mse);
    r += ",";
    r += std::isinf(psnr) ? "inf" : (std::isnan(psnr) ? "nan" : fmt("%.4f", psnr));
    r += "," + std::to_string(iterations) + "," + fmt("%.4f", ndc_per_point_iter) + "," + fmt("%.3f", time_ms) + "," +
         std::to_string(k_actual) + "," + flagstr;
    return r;
}

std::string QuantReport::to_json() const { // metrics.cpp:96-115 (keys sorted, 2-space indent)
    std::string f = "[";
    for (std::size_t i = 0; i < flags.size(); ++i) f += (i ? ", " : "") + jstr(flags[i]);
    f += "]";
    std::string o = "{\n";
    o += "  \"actual_k\": " + std::to_string(k_actual) + ",\n";
    o += "  \"flags\": " + f + ",\n";
    o += "  \"image\": " + jstr(image) + ",\n";
    o += "  \"iterations\": " + std::to_string(iterations) + ",\n";
    o += "  \"k\": " + std::to_string(k_requested) + ",\n";
    o += "  \"method\": " + jstr(method) + ",\n";
    o += "  \"mse\": " + jnum(mse) + ",\n";
    o += "  \"ndc_per_point_iter\": " + jnum(ndc_per_point_iter) + ",\n";
    o += "  \"psnr\": " + (std::isinf(psnr) ? std::string("\"inf\"") : jnum(psnr)) + ",\n";
    o += "  \"run\": " + std::to_string(run) + ",\n";
    o += "  \"sampling\": " + jstr(sampling_mode_token(sampling)) + ",\n";
    o += "  \"seed\": " + std::to_string(seed) + ",\n";
    o += "  \"time_ms\": " + jnum(time_ms) + "\n}";
    return o;
}

// ---- pipeline (pipeline.cpp) ----------------------------------------------
namespace {
const std::vector<std::string> kPre = {"mc", "ott", "oct", "wan", "wu", "bs"};
const std::vector<std::string> kInit = {"fgy", "lbg", "mmx", "den", "var", "sff", "kpp"};
bool has(const std::vector<std::string> &v, const std::string &s) { return std::find(v.begin(), v.end(), s) != v.end(); }
} // namespace

MethodSpec parse_method(const std::string &method, const std::string &init) { // pipeline.cpp:20-45
    MethodSpec s;
    if (method == "wsm") {
        s.refine = true;
        s.base = init.empty() ? "fgy" : init;
    } else if (method.rfind("wsm-", 0) == 0) {
        if (!init.empty())
            throw std::invalid_argument("method '" + method + "' already names its initializer; drop --init");
        s.refine = true;
        s.base = method.substr(4);
    } else {
        if (!init.empty()) throw std::invalid_argument("--init only applies to wsm methods, not '" + method + "'");
        s.base = method;
    }
    if (s.refine) {
        if (!has(kInit, s.base) && !has(kPre, s.base))
            throw std::invalid_argument("unknown initializer '" + s.base +
                                        "' (expected fgy|lbg|mmx|den|var|sff|kpp|mc|ott|oct|wan|wu|bs)");
    } else if (!has(kPre, s.base)) {
        throw std::invalid_argument("unknown method '" + method +
                                    "' (expected mc|ott|oct|wan|wu|bs, wsm, or wsm-<init>)");
    }
    return s;
}

std::vector<std::string> all_method_tokens() {
    std::vector<std::string> out = kPre;
    for (const auto &t : kInit) out.push_back("wsm-" + t);
    for (const auto &t : kPre) out.push_back("wsm-" + t);
    return out;
}

namespace {
void finish_report(QuantizeResult &out, const QuantizeConfig &config, double ms) {
    QuantReport &r = out.report;
    r.method = config.method.token();
    r.k_requested = config.k;
    r.k_actual = static_cast<int>(out.palette.size());
    r.seed = config.seed;
    r.sampling = config.sampling;
    r.mse = out.mapping.mean_sq_dist;
    r.psnr = psnr_from_mse(r.mse);
    r.iterations = out.state.iterations;
    r.ndc_per_point_iter = out.state.ndc_per_point_iter(out.substrate_points);
    r.time_ms = ms;
    if (out.state.repair_count > 0) r.flags.push_back("repairs:" + std::to_string(out.state.repair_count));
}

int device_init_kind(const QuantizeConfig &config) {
    if (config.method.base == "mmx") return CQG_INIT_MAXIMIN;
    if (config.method.base == "kpp") return CQG_INIT_KMEANSPP;
    throw std::invalid_argument("run_quantize: initializer '" + config.method.base +
                                "' is outside the device path; supply init_centers");
}

// record_history: the stages as separate device calls, so the engine can keep
// the per-iteration snapshots (pipeline.cpp:126-130 forwards the flag to wsm)
QuantizeResult quantize_with_history(const RawImage &image, const QuantizeConfig &config,
                                     std::span<const ColorPoint> init_centers) {
    QuantizeResult out;
    const bool sub = config.sampling == SamplingMode::TwoToOne || config.sampling == SamplingMode::TwoToOneUnique;
    const bool dedup = config.sampling == SamplingMode::Unique || config.sampling == SamplingMode::TwoToOneUnique;
    std::vector<Rgb8> sampled_storage;
    std::span<const Rgb8> sampled(image.pixels);
    if (sub) {
        sampled_storage = subsample_2to1(image);
        sampled = sampled_storage;
    }
    const WeightedHistogram hist = build_histogram(sampled, config.seed);
    std::vector<ColorPoint> init(init_centers.begin(), init_centers.end());
    if (init.empty()) {
        SeedConfig sc;
        sc.k = config.k;
        sc.seed = config.seed;
        init = device_init_kind(config) == CQG_INIT_MAXIMIN ? init_maximin(hist, sc) : init_kmeanspp(hist, sc);
    }
    ClusterOptions opts;
    opts.term = config.term;
    opts.record_history = true;
    if (dedup) {
        out.state = detail::lloyd_counts(detail::pack_all(hist.colors), hist.counts, hist.source_pixel_count, init, opts);
        out.substrate_points = hist.size();
    } else { // every sampled pixel, weight 1/S (pipeline.cpp:103-108)
        std::vector<std::uint32_t> packed(sampled.size()), ones(sampled.size(), 1u);
        for (std::size_t i = 0; i < sampled.size(); ++i)
            packed[i] = (std::uint32_t(sampled[i].r) << 16) | (std::uint32_t(sampled[i].g) << 8) | sampled[i].b;
        out.state = detail::lloyd_counts(packed, ones, sampled.size(), init, opts);
        out.substrate_points = sampled.size();
    }
    out.palette.colors = out.state.centers;
    out.mapping = map_pixels(image, out.palette);
    return out;
}

QuantizeResult quantize(const RawImage &image, const QuantizeConfig &config, std::span<const ColorPoint> init_centers) {
    if (image.pixels.empty()) throw std::invalid_argument("run_quantize: empty image");
    if (config.k < 1) throw std::invalid_argument("run_quantize: k must be at least 1");
    if (!config.method.refine)
        throw std::invalid_argument("run_quantize: standalone preclusterers are outside the device path");
    if (!init_centers.empty() && static_cast<int>(init_centers.size()) != config.k)
        throw std::invalid_argument("run_quantize: init_centers must hold k centres");
    const auto t0 = std::chrono::steady_clock::now();
    if (config.record_history) {
        QuantizeResult out = quantize_with_history(image, config, init_centers);
        finish_report(out, config, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        return out;
    }
    QuantizeResult out;
    const std::size_t P = image.pixel_count();
    const int k = config.k;
    cqg_quantize_cfg cfg{};
    cfg.k = k;
    cfg.seed = config.seed;
    ClusterOptions co;
    co.term = config.term;
    cfg.term = detail::to_term(co);
    cfg.index_bytes = 4;
    switch (config.sampling) { // pipeline.cpp:91-116
        case SamplingMode::None: cfg.sampling = CQG_SAMPLING_NONE; break;
        case SamplingMode::TwoToOne: cfg.sampling = CQG_SAMPLING_TWO_TO_ONE; break;
        case SamplingMode::TwoToOneUnique: cfg.sampling = CQG_SAMPLING_BOTH; break;
        default: cfg.sampling = CQG_SAMPLING_UNIQUE; break;
    }
    cfg.width = image.width;
    cfg.height = image.height;
    std::vector<double> init;
    if (!init_centers.empty()) {
        cfg.init_kind = CQG_INIT_GIVEN;
        init = flatten(init_centers);
    } else {
        cfg.init_kind = device_init_kind(config);
    }
    const int limit = cfg.term.fixed_iterations > 0 ? cfg.term.fixed_iterations : cfg.term.max_iterations;
    std::vector<double> pal(3 * static_cast<std::size_t>(k)), sse(std::max(limit, 1));
    std::vector<std::uint32_t> labels(P); // the substrate: <= 2^24 colours, or every sampled pixel
    out.mapping.indices.resize(P);
    out.mapping.quantized.width = image.width;
    out.mapping.quantized.height = image.height;
    out.mapping.quantized.pixels.resize(P);
    cqg_quantize_stats st{};
    check(cqg_quantize(ctx(), reinterpret_cast<const std::uint8_t *>(image.pixels.data()), P, &cfg,
                       init.empty() ? nullptr : init.data(), pal.data(), labels.data(), sse.data(),
                       out.mapping.indices.data(), reinterpret_cast<std::uint8_t *>(out.mapping.quantized.pixels.data()),
                       &st));
    const auto t1 = std::chrono::steady_clock::now();
    out.palette.colors = unflatten(pal.data(), static_cast<std::size_t>(k));
    out.mapping.mean_sq_dist = st.mean_sq_dist;
    out.mapping.ndc = st.map_ndc;
    out.state.centers = out.palette.colors;
    out.state.memberships.assign(labels.begin(), labels.begin() + static_cast<std::ptrdiff_t>(st.n_unique));
    out.state.sse_trace.assign(sse.begin(), sse.begin() + st.lloyd.iterations);
    out.state.iterations = st.lloyd.iterations;
    out.state.ndc_total = st.lloyd.ndc_total;
    out.state.repair_count = st.lloyd.repair_count;
    out.substrate_points = st.n_unique;
    finish_report(out, config, std::chrono::duration<double, std::milli>(t1 - t0).count());
    return out;
}
} // namespace

QuantizeResult run_quantize(const RawImage &image, const QuantizeConfig &config) {
    return quantize(image, config, {});
}

QuantizeResult run_quantize(const RawImage &image, const QuantizeConfig &config,
                            std::span<const ColorPoint> init_centers) {
    if (init_centers.empty()) throw std::invalid_argument("run_quantize: init_centers must hold k centres");
    return quantize(image, config, init_centers);
}

} // namespace quant
