// quant_b200.cpp -- the reference's quant:: C++ API (include/quant/quant.hpp)
// implemented over the C-ABI of libcqg.so. Semantics and exception messages
// follow the reference sources cited per function (/root/reference/proj/src).
#include "quant/quant.hpp"

#include <algorithm>
#include <functional>
#include <fstream>
#include <cstdlib>
#include <cerrno>
#include <cctype>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>

#include "cqg.h"

namespace quant {

namespace {

thread_local int t_device = 0;

struct CtxHolder {
    std::map<int, cqg_ctx *> ctx;
    ~CtxHolder() {
        for (auto &kv : ctx) cqg_destroy(kv.second);
    }
};
thread_local CtxHolder t_ctx;

cqg_ctx *ctx() {
    auto it = t_ctx.ctx.find(t_device);
    if (it != t_ctx.ctx.end()) return it->second;
    cqg_ctx *c = cqg_create(t_device);
    if (!c) throw std::runtime_error(std::string("libcqg: ") + cqg_last_error());
    t_ctx.ctx[t_device] = c;
    return c;
}

void check(int rc) {
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

std::vector<double> flatten(std::span<const ColorPoint> c) {
    std::vector<double> v(3 * c.size());
    for (std::size_t i = 0; i < c.size(); ++i) {
        v[3 * i] = c[i].r;
        v[3 * i + 1] = c[i].g;
        v[3 * i + 2] = c[i].b;
    }
    return v;
}

std::vector<ColorPoint> unflatten(const double *v, std::size_t k) {
    std::vector<ColorPoint> c(k);
    for (std::size_t i = 0; i < k; ++i) c[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
    return c;
}

cqg_term to_term(const ClusterOptions &o) {
    const Termination &t = o.term;
    if (t.fixed_iterations && *t.fixed_iterations <= 0)
        throw std::invalid_argument("clustering: fixed_iterations < 1"); // kmeans.cpp:187-188
    cqg_term ct{};
    ct.epsilon = t.epsilon;
    ct.max_iterations = t.max_iterations;
    ct.fixed_iterations = t.fixed_iterations ? *t.fixed_iterations : 0;
    ct.record_history = o.record_history ? 1 : 0;
    return ct;
}

ClusterState lloyd(const std::vector<std::uint32_t> &packed, const std::vector<std::uint32_t> &counts,
                   std::uint64_t P, std::vector<ColorPoint> init, const ClusterOptions &options) {
    const cqg_term term = to_term(options);
    const std::size_t n = packed.size(), k = init.size();
    const int limit = term.fixed_iterations > 0 ? term.fixed_iterations : std::max(term.max_iterations, 1);
    std::vector<double> in = flatten(init), cen(3 * std::max<std::size_t>(k, 1));
    std::vector<std::uint32_t> labels(std::max<std::size_t>(n, 1));
    std::vector<double> sse(limit);
    std::vector<std::uint32_t> hl;
    std::vector<double> hc;
    if (options.record_history) {
        hl.resize(static_cast<std::size_t>(limit) * n);
        hc.resize(static_cast<std::size_t>(limit) * 3 * k);
    }
    cqg_lloyd_stats st{};
    check(cqg_lloyd(ctx(), packed.data(), counts.data(), n, P, in.empty() ? nullptr : in.data(),
                    static_cast<int>(k), &term, cen.data(), labels.data(), sse.data(), &st,
                    hl.empty() ? nullptr : hl.data(), hc.empty() ? nullptr : hc.data()));
    ClusterState s;
    s.centers = unflatten(cen.data(), k);
    s.memberships.assign(labels.begin(), labels.begin() + static_cast<std::ptrdiff_t>(n));
    s.sse_trace.assign(sse.begin(), sse.begin() + st.iterations);
    s.iterations = st.iterations;
    s.ndc_total = st.ndc_total;
    s.repair_count = st.repair_count;
    if (options.record_history)
        for (int it = 0; it < st.iterations; ++it) {
            IterationSnapshot snap;
            snap.centers = unflatten(hc.data() + static_cast<std::size_t>(it) * 3 * k, k);
            snap.memberships.assign(hl.begin() + static_cast<std::ptrdiff_t>(it * n),
                                    hl.begin() + static_cast<std::ptrdiff_t>((it + 1) * n));
            s.history.push_back(std::move(snap));
        }
    return s;
}

struct DeviceHist {
    std::vector<std::uint32_t> packed, counts;
    std::uint64_t P = 0;
};

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

} // namespace

void set_device(int device) { t_device = device; }

// ---- colour ---------------------------------------------------------------
double dist2(const ColorPoint &a, const ColorPoint &b) {
    const double dr = a.r - b.r, dg = a.g - b.g, db = a.b - b.b;
    return dr * dr + dg * dg + db * db;
}
double dist2(const ColorPoint &a, const Rgb8 &b) { return dist2(a, ColorPoint(b)); }

std::uint8_t channel_to_u8(double v) { // color.hpp:63-68
    double r = std::floor(v + 0.5);
    if (r < 0.0) r = 0.0;
    if (r > 255.0) r = 255.0;
    return static_cast<std::uint8_t>(r);
}
Rgb8 to_rgb8(const ColorPoint &c) { return {channel_to_u8(c.r), channel_to_u8(c.g), channel_to_u8(c.b)}; }

// ---- rng ------------------------------------------------------------------
std::uint64_t Rng::next_below(std::uint64_t n) { // rng.hpp:25-33
    if (n == 0) throw std::invalid_argument("next_below: empty range");
    const std::uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    std::uint64_t x;
    do { x = gen_(); } while (x >= limit);
    return x % n;
}

std::size_t weighted_draw(std::span<const double> mass, Rng &rng) { // rng.hpp:43-54
    double total = 0.0;
    for (double m : mass) total += m;
    if (!(total > 0.0)) throw std::invalid_argument("weighted_draw: total mass must be positive");
    const double u = rng.next_unit() * total;
    double acc = 0.0;
    for (std::size_t i = 0; i + 1 < mass.size(); ++i) {
        acc += mass[i];
        if (u < acc) return i;
    }
    return mass.size() - 1;
}

// ---- histogram ------------------------------------------------------------
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
    DeviceHist d = device_hist(pixels);
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
    h.counts = std::move(d.counts);
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

// ---- PPM image I/O on the host (image.hpp:26-44; binary P6, maxval 255) ----
namespace {
[[noreturn]] void io_fail(const std::string &path, const std::string &what) {
    throw std::runtime_error(path + ": " + what);
}

// next whitespace-delimited header token; '#' comments run to end of line.
// The delimiter after the token is consumed (so after maxval exactly one
// whitespace byte separates the header from the raster).
bool ppm_token(std::istream &in, std::string &tok) {
    tok.clear();
    for (int c = in.get(); c != EOF; c = in.get()) {
        if (c == '#') {
            while (c != EOF && c != '\n') c = in.get();
            if (c == EOF) break;
            continue;
        }
        if (std::isspace(c)) {
            if (tok.empty()) continue;
            return true;
        }
        tok.push_back(static_cast<char>(c));
    }
    return !tok.empty();
}

long ppm_field(std::istream &in, const std::string &path, const char *field) {
    std::string tok;
    if (!ppm_token(in, tok)) io_fail(path, std::string("truncated PPM header (missing ") + field + ")");
    char *end = nullptr;
    errno = 0;
    const long v = std::strtol(tok.c_str(), &end, 10);
    if (tok.empty() || *end != '\0' || errno != 0 || std::isspace(static_cast<unsigned char>(tok[0])))
        io_fail(path, std::string("malformed PPM ") + field + " '" + tok + "'");
    return v;
}

bool ends_with_ci(const std::string &s, const char *suffix) {
    const std::size_t n = std::strlen(suffix);
    if (s.size() < n) return false;
    for (std::size_t i = 0; i < n; ++i)
        if (std::tolower(static_cast<unsigned char>(s[s.size() - n + i])) != suffix[i]) return false;
    return true;
}
} // namespace

LoadedImage load_image(const std::string &path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) io_fail(path, "cannot open file");
    char magic[2] = {0, 0};
    in.read(magic, 2);
    if (in.gcount() < 2) io_fail(path, "file too short to identify");
    if (magic[0] == '\x89' && magic[1] == 'P') io_fail(path, "PNG input needs libpng, which this build does not link");
    if (!(magic[0] == 'P' && magic[1] == '6'))
        io_fail(path, "unsupported format (expected binary PPM 'P6' or PNG)");
    const long w = ppm_field(in, path, "width");
    const long h = ppm_field(in, path, "height");
    const long maxval = ppm_field(in, path, "maxval");
    if (w <= 0 || h <= 0) io_fail(path, "non-positive PPM dimensions");
    if (maxval != 255) io_fail(path, "unsupported PPM maxval " + std::to_string(maxval) + " (only 255)");
    LoadedImage out;
    out.image.width = static_cast<int>(w);
    out.image.height = static_cast<int>(h);
    const std::size_t bytes = static_cast<std::size_t>(w) * static_cast<std::size_t>(h) * 3;
    out.image.pixels.resize(bytes / 3);
    in.read(reinterpret_cast<char *>(out.image.pixels.data()), static_cast<std::streamsize>(bytes));
    if (static_cast<std::size_t>(in.gcount()) != bytes)
        io_fail(path, "truncated PPM pixel data (expected " + std::to_string(bytes) + " bytes, got " +
                          std::to_string(in.gcount()) + ")");
    return out;
}

void save_ppm(const RawImage &image, const std::string &path) {
    if (image.width <= 0 || image.height <= 0 ||
        image.pixels.size() != static_cast<std::size_t>(image.width) * static_cast<std::size_t>(image.height))
        throw std::invalid_argument("save_ppm: inconsistent image dimensions");
    std::ofstream out(path, std::ios::binary);
    if (!out) io_fail(path, "cannot open file for writing");
    const std::string head = "P6\n" + std::to_string(image.width) + " " + std::to_string(image.height) + "\n255\n";
    out.write(head.data(), static_cast<std::streamsize>(head.size()));
    out.write(reinterpret_cast<const char *>(image.pixels.data()),
              static_cast<std::streamsize>(image.pixels.size() * 3));
    if (!out) io_fail(path, "write failed");
}

void save_image(const RawImage &image, const std::string &path) {
    if (ends_with_ci(path, ".ppm")) return save_ppm(image, path);
    if (ends_with_ci(path, ".png")) io_fail(path, "PNG output needs libpng, which this build does not link");
    io_fail(path, "unknown output extension (use .ppm or .png)");
}

// ---- kmeans host utilities (kmeans.cpp:9-114) -----------------------------
bool check_convergence(double sse_prev, double sse_cur, double epsilon) {
    if (sse_cur == 0.0) return true;
    return (sse_prev - sse_cur) / sse_cur <= epsilon;
}

CenterDistanceTable build_center_distance_table(std::span<const ColorPoint> centers) {
    const std::size_t k = centers.size();
    CenterDistanceTable t;
    t.k = k;
    t.dist2.resize(k * k);
    t.order.resize(k * k);
    for (std::size_t i = 0; i < k; ++i)
        for (std::size_t j = 0; j < k; ++j) t.dist2[i * k + j] = dist2(centers[i], centers[j]);
    for (std::size_t i = 0; i < k; ++i) {
        std::uint32_t *row = t.order.data() + i * k;
        const double *d = t.dist2.data() + i * k;
        for (std::size_t j = 0; j < k; ++j) row[j] = static_cast<std::uint32_t>(j);
        std::sort(row, row + k, [d](std::uint32_t a, std::uint32_t b) { return d[a] != d[b] ? d[a] < d[b] : a < b; });
        auto self = std::find(row, row + k, static_cast<std::uint32_t>(i));
        std::rotate(row, self, self + 1);
    }
    return t;
}

std::uint32_t nearest_full(const ColorPoint &x, std::span<const ColorPoint> c, std::uint64_t &ndc) {
    std::uint32_t best = 0;
    double bd = dist2(x, c[0]);
    ++ndc;
    for (std::size_t j = 1; j < c.size(); ++j, ++ndc) {
        const double d = dist2(x, c[j]);
        if (d < bd) { bd = d; best = static_cast<std::uint32_t>(j); }
    }
    return best;
}

std::uint32_t assign_point_sortmeans(const ColorPoint &x, std::uint32_t prev, const CenterDistanceTable &t,
                                     std::span<const ColorPoint> c, std::uint64_t &ndc) {
    const double pd = dist2(x, c[prev]);
    ++ndc;
    const double cut = 4.0 * pd;
    double bd = pd;
    std::uint32_t best = prev;
    for (std::size_t j = 1; j < t.k; ++j) {
        const std::uint32_t o = t.order_at(prev, j);
        if (t.d2(prev, o) >= cut) break;
        const double d = dist2(x, c[o]);
        ++ndc;
        if (d < bd) { bd = d; best = o; }
    }
    return best;
}

std::uint32_t nearest_pruned_lowest_index(const ColorPoint &x, std::uint32_t hint, const CenterDistanceTable &t,
                                          std::span<const ColorPoint> c, std::uint64_t &ndc) {
    const double pd = dist2(x, c[hint]);
    ++ndc;
    const double cut = 4.0 * pd;
    double bd = pd;
    std::uint32_t best = hint;
    for (std::size_t j = 1; j < t.k; ++j) {
        const std::uint32_t o = t.order_at(hint, j);
        if (t.d2(hint, o) > cut) break;
        const double d = dist2(x, c[o]);
        ++ndc;
        if (d < bd || (d == bd && o < best)) { bd = d; best = o; }
    }
    return best;
}

double compute_sse(std::span<const ColorPoint> points, std::span<const double> weights,
                   std::span<const ColorPoint> centers, std::span<const std::uint32_t> m) {
    double s = 0.0;
    for (std::size_t i = 0; i < points.size(); ++i) s += weights[i] * dist2(points[i], centers[m[i]]);
    return s;
}

// ---- wsm (kmeans.cpp:271-277) on the device -------------------------------
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
    // decode integer counts: w_i == c_i * (1/P) exactly (histogram.cpp:99-102)
    const double wmin = *std::min_element(weights.begin(), weights.end());
    std::vector<std::uint32_t> counts(n);
    std::uint64_t P = 0;
    for (int cmin = 1; cmin <= 256 && P == 0; ++cmin) {
        const std::uint64_t cand = static_cast<std::uint64_t>(std::llround(cmin / wmin));
        if (cand == 0) continue;
        const double inv = 1.0 / static_cast<double>(cand);
        std::uint64_t tot = 0;
        bool ok = true;
        for (std::size_t i = 0; i < n && ok; ++i) {
            const double c = std::nearbyint(weights[i] * static_cast<double>(cand));
            if (c < 1.0 || c > 4294967295.0 || c * inv != weights[i]) ok = false;
            counts[i] = static_cast<std::uint32_t>(c);
            tot += counts[i];
        }
        if (ok && tot == cand) P = cand;
    }
    if (P == 0) throw std::invalid_argument("wsm: device engine needs weights of the form count/P");
    std::vector<std::uint32_t> packed(n);
    for (std::size_t i = 0; i < n; ++i) {
        const ColorPoint &p = points[i];
        if (p.r != std::floor(p.r) || p.g != std::floor(p.g) || p.b != std::floor(p.b) || p.r < 0 || p.g < 0 ||
            p.b < 0 || p.r > 255 || p.g > 255 || p.b > 255)
            throw std::invalid_argument("wsm: device engine needs points on the 8-bit colour grid");
        packed[i] = pack(p);
    }
    return lloyd(packed, counts, P, std::move(init), options);
}

ClusterState wsm(const WeightedHistogram &hist, std::vector<ColorPoint> init, const ClusterOptions &options) {
    std::vector<std::uint32_t> packed(hist.size());
    for (std::size_t i = 0; i < hist.size(); ++i) packed[i] = pack(hist.colors[i]);
    return lloyd(packed, hist.counts, hist.source_pixel_count, std::move(init), options);
}

// ---- init (init.cpp:127-138, 295-314) on the device -----------------------
static std::vector<ColorPoint> run_init(int kind, const WeightedHistogram &hist, const SeedConfig &cfg) {
    std::vector<std::uint32_t> packed(hist.size());
    for (std::size_t i = 0; i < hist.size(); ++i) packed[i] = pack(hist.colors[i]);
    std::vector<double> out(3 * static_cast<std::size_t>(std::max(cfg.k, 1)));
    if (kind == CQG_INIT_MAXIMIN)
        check(cqg_init_maximin(ctx(), packed.data(), hist.counts.data(), hist.size(), hist.source_pixel_count, cfg.k,
                               cfg.seed, cfg.maximin_weighted_first ? 1 : 0, out.data()));
    else
        check(cqg_init_kmeanspp(ctx(), packed.data(), hist.counts.data(), hist.size(), hist.source_pixel_count,
                                cfg.k, cfg.seed, out.data()));
    return unflatten(out.data(), static_cast<std::size_t>(cfg.k));
}

std::vector<ColorPoint> init_maximin(const WeightedHistogram &hist, const SeedConfig &cfg) {
    return run_init(CQG_INIT_MAXIMIN, hist, cfg);
}
std::vector<ColorPoint> init_kmeanspp(const WeightedHistogram &hist, const SeedConfig &cfg) {
    return run_init(CQG_INIT_KMEANSPP, hist, cfg);
}

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

QuantizeResult run_quantize(const RawImage &image, const QuantizeConfig &config) { // pipeline.cpp:81-164
    if (image.pixels.empty()) throw std::invalid_argument("run_quantize: empty image");
    if (config.k < 1) throw std::invalid_argument("run_quantize: k must be at least 1");
    if (!config.method.refine)
        throw std::invalid_argument("run_quantize: standalone preclusterers are outside the device path");
    const auto t0 = std::chrono::steady_clock::now();
    QuantizeResult out;
    const std::size_t P = image.pixel_count();
    const int k = config.k;
    cqg_quantize_cfg cfg{};
    cfg.k = k;
    cfg.seed = config.seed;
    ClusterOptions co;
    co.term = config.term;
    cfg.term = to_term(co);
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
    if (!config.init_centers.empty()) {
        if (static_cast<int>(config.init_centers.size()) != k)
            throw std::invalid_argument("run_quantize: init_centers must hold k centres");
        cfg.init_kind = CQG_INIT_GIVEN;
        init = flatten(config.init_centers);
    } else if (config.method.base == "mmx") {
        cfg.init_kind = CQG_INIT_MAXIMIN;
    } else if (config.method.base == "kpp") {
        cfg.init_kind = CQG_INIT_KMEANSPP;
    } else {
        throw std::invalid_argument("run_quantize: initializer '" + config.method.base +
                                    "' is outside the device path; supply init_centers");
    }
    const int limit = cfg.term.fixed_iterations > 0 ? cfg.term.fixed_iterations : cfg.term.max_iterations;
    std::vector<double> pal(3 * static_cast<std::size_t>(k));
    std::vector<std::uint32_t> labels(P); // the substrate: <= 2^24 colours, or every sampled pixel
    std::vector<double> sse(std::max(limit, 1));
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
    QuantReport &r = out.report;
    r.method = config.method.token();
    r.k_requested = k;
    r.k_actual = k;
    r.seed = config.seed;
    r.sampling = config.sampling;
    r.mse = out.mapping.mean_sq_dist;
    r.psnr = psnr_from_mse(r.mse);
    r.iterations = out.state.iterations;
    r.ndc_per_point_iter = out.state.ndc_per_point_iter(out.substrate_points);
    r.time_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (out.state.repair_count > 0) r.flags.push_back("repairs:" + std::to_string(out.state.repair_count));
    return out;
}

} // namespace quant
