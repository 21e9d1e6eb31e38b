// test_dropin.cpp -- the reference's own style of checks (its doctest suites,
// proj/tests/test_*.cpp) run against libquant_b200.so through the C++ quant::
// API. Built by __graft_entry__.build() into tests/cpp/test_dropin; run by
// tests/test_gpu_cpp.py on a GPU box. Prints one line per case, exit 0 = pass.
//
//   argv[1] = tests/golden directory (acc_61.rgb, acc_62.rgb, sweep_a_rows.csv, wu_init.txt)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "quant/quant.hpp"

using namespace quant;

static int g_fail = 0;
#define CHECK(cond)                                                                     \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
            ++g_fail;                                                                   \
        }                                                                               \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                        \
    do {                                                                                \
        bool ok_ = false;                                                               \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const T &) {                                                           \
            ok_ = true;                                                                 \
        } catch (...) {                                                                 \
        }                                                                               \
        if (!ok_) {                                                                     \
            std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
            ++g_fail;                                                                   \
        }                                                                               \
    } while (0)

static RawImage load_rgb(const std::string &path, int w, int h) {
    RawImage img;
    img.width = w;
    img.height = h;
    img.pixels.resize(static_cast<std::size_t>(w) * h);
    std::ifstream f(path, std::ios::binary);
    f.read(reinterpret_cast<char *>(img.pixels.data()), static_cast<std::streamsize>(img.pixels.size() * 3));
    return img;
}

static void case_histogram_order() { // test_histogram.cpp:102-118
    const Rgb8 A{10, 20, 30}, B{200, 100, 50}, C{0, 0, 0};
    std::vector<Rgb8> px = {A, B, A, C, B, A};
    WeightedHistogram h = build_histogram(px, 1);
    CHECK(h.size() == 3);
    CHECK(h.source_pixel_count == 6);
    CHECK(h.colors[0] == ColorPoint(10, 20, 30));
    CHECK(h.colors[1] == ColorPoint(200, 100, 50));
    CHECK(h.colors[2] == ColorPoint(0, 0, 0));
    CHECK(h.counts[0] == 3 && h.counts[1] == 2 && h.counts[2] == 1);
    CHECK(h.weights[0] == 0.5);
    CHECK(h.hash.m == next_prime_at_least(12));
    CHECK_THROWS_AS(build_histogram(std::vector<Rgb8>{}, 1), std::invalid_argument);
}

static void case_wsm_semantics() { // test_kmeans.cpp:210-285
    std::vector<ColorPoint> pts = {{0, 0, 0}, {9, 0, 0}};
    std::vector<double> w = {0.5, 0.5};
    ClusterState st = wsm(pts, w, {{5, 0, 0}, {5, 0, 0}}, {});
    CHECK(st.repair_count == 1);
    CHECK(st.iterations == 1);
    CHECK(st.sse_trace.size() == 1 && st.sse_trace[0] == 0.0);
    std::vector<double> got = {st.centers[0].r, st.centers[1].r};
    std::sort(got.begin(), got.end());
    CHECK(got == (std::vector<double>{0.0, 9.0}));

    std::vector<ColorPoint> one = {{0, 0, 0}};
    std::vector<ColorPoint> three = {{0, 0, 0}, {1, 1, 1}, {2, 2, 2}};
    CHECK_THROWS_AS(wsm(pts, w, {}, {}), std::invalid_argument);
    CHECK_THROWS_AS(wsm(pts, w, three, {}), std::invalid_argument);
    CHECK_THROWS_AS(wsm(pts, std::vector<double>{0.5}, one, {}), std::invalid_argument);
    CHECK_THROWS_AS(wsm(pts, std::vector<double>{0.5, -0.5}, one, {}), std::invalid_argument);
    ClusterOptions bad;
    bad.term.epsilon = -1.0;
    CHECK_THROWS_AS(wsm(pts, w, one, bad), std::invalid_argument);
    bad.term.epsilon = 0.001;
    bad.term.max_iterations = 0;
    CHECK_THROWS_AS(wsm(pts, w, one, bad), std::invalid_argument);
    bad.term.max_iterations = 100;
    bad.term.fixed_iterations = 0;
    CHECK_THROWS_AS(wsm(pts, w, one, bad), std::invalid_argument);
}

static void case_histogram_equals_duplicates() { // test_kmeans.cpp:287-305 (weights = counts / P)
    std::vector<ColorPoint> hp = {{10, 0, 0}, {90, 0, 0}};
    std::vector<double> hw = {0.75, 0.25};
    ClusterOptions opt;
    opt.term.fixed_iterations = 3;
    ClusterState fast = wsm(hp, hw, {{0, 0, 0}, {100, 0, 0}}, opt);
    CHECK(fast.sse_trace.size() == 3);
    CHECK(fast.centers[0] == ColorPoint(10, 0, 0));
    CHECK(fast.centers[1] == ColorPoint(90, 0, 0));
    CHECK(fast.sse_trace[0] == 0.0 && fast.sse_trace[2] == 0.0);
}

static void case_mapping() { // test_metrics.cpp:66-92
    RawImage img;
    img.width = 1;
    img.height = 1;
    img.pixels = {{1, 0, 0}};
    Palette pal;
    pal.colors = {{2, 0, 0}, {0, 0, 0}};
    CHECK(map_pixels(img, pal).indices[0] == 0);
    std::swap(pal.colors[0], pal.colors[1]);
    CHECK(map_pixels(img, pal).indices[0] == 0);
    img.width = 2;
    img.pixels = {{0, 0, 0}, {1, 0, 0}};
    pal.colors = {{0.5, 0, 0}};
    MappingResult m = map_pixels(img, pal);
    CHECK(std::abs(m.mean_sq_dist - 0.25) <= 1e-12);
    CHECK(m.quantized.pixels[0].r == 1);
    CHECK_THROWS_AS(map_pixels(img, Palette{}), std::invalid_argument);
}

static void case_golden_rows(const std::string &dir) { // proj/tmp_acceptance/sweep_a.csv:2-13
    std::ifstream f(dir + "/sweep_a_rows.csv");
    std::string line;
    std::getline(f, line);
    std::multiset<std::string> want;
    while (std::getline(f, line))
        if (!line.empty() && line.find(",wu,") == std::string::npos) want.insert(line);
    std::ifstream wf(dir + "/wu_init.txt");
    std::vector<std::vector<ColorPoint>> wu(2);
    for (int s = 0; s < 2; ++s)
        for (int i = 0; i < 8; ++i) {
            double r, g, b;
            wf >> r >> g >> b;
            wu[s].push_back({r, g, b});
        }
    std::multiset<std::string> got;
    for (int s = 0; s < 2; ++s) {
        const int seed_img = 61 + s;
        RawImage img = load_rgb(dir + "/acc_" + std::to_string(seed_img) + ".rgb", 40, 40);
        for (const char *method : {"wsm-kpp", "wsm-wu"})
            for (int run = 0; run < 2; ++run) {
                QuantizeConfig cfg;
                cfg.method = parse_method(method);
                cfg.k = 8;
                cfg.seed = 3 + run;
                QuantizeResult r = std::string(method) == "wsm-wu" ? run_quantize(img, cfg, wu[s])
                                                                    : run_quantize(img, cfg);
                r.report.image = "acc_" + std::to_string(seed_img) + ".ppm";
                r.report.run = run;
                r.report.time_ms = 0.0;
                got.insert(r.report.csv_row());
            }
    }
    CHECK(got == want);
    if (got != want)
        for (const auto &g : got) std::printf("  got  %s\n", g.c_str());
}

static void case_report_format() { // test_metrics.cpp:94-125
    CHECK(std::string(QuantReport::csv_header()) ==
          "image,method,k,run,seed,sampling,mse,psnr,iterations,ndc_per_point_iter,time_ms,actual_k,flags");
    QuantReport r;
    r.image = "img.ppm";
    r.method = "wsm-wu";
    r.k_requested = 32;
    r.k_actual = 32;
    r.run = 2;
    r.seed = 3;
    r.mse = 71.25;
    r.psnr = 29.603;
    r.iterations = 14;
    r.ndc_per_point_iter = 3.9812;
    r.time_ms = 12.5;
    r.flags = {"repairs:1", "padded_init"};
    CHECK(r.csv_row() == "img.ppm,wsm-wu,32,2,3,unique,71.250000,29.6030,14,3.9812,12.500,32,repairs:1;padded_init");
    CHECK(r.to_json().find("\"psnr\": 29.603") != std::string::npos);
}

static void case_sampling_substrates() { // test_pipeline.cpp:106-134: the substrate per sampling mode
    RawImage img;
    img.width = 50;
    img.height = 40;
    img.pixels.resize(50 * 40);
    std::uint32_t st = 33;
    for (auto &p : img.pixels) { // a few repeated colours plus noise
        st = st * 1664525u + 1013904223u;
        const int c = (st >> 28) & 7;
        p = Rgb8{static_cast<std::uint8_t>(30 * c), static_cast<std::uint8_t>(200 - 20 * c),
                 static_cast<std::uint8_t>((st >> 16) & ((st >> 27) & 1 ? 255 : 3))};
    }
    QuantizeConfig cfg;
    cfg.method = parse_method("wsm-mmx");
    cfg.k = 16;
    cfg.sampling = SamplingMode::None;
    const QuantizeResult none = run_quantize(img, cfg);
    CHECK(none.substrate_points == img.pixels.size());
    CHECK(none.state.memberships.size() == img.pixels.size());
    cfg.sampling = SamplingMode::TwoToOne;
    const QuantizeResult half = run_quantize(img, cfg);
    CHECK(half.substrate_points == 25 * 20);
    cfg.sampling = SamplingMode::Unique;
    const QuantizeResult uniq = run_quantize(img, cfg);
    CHECK(uniq.substrate_points == build_histogram(img.pixels, cfg.seed).size());
    CHECK(uniq.substrate_points < img.pixels.size());
    cfg.sampling = SamplingMode::TwoToOneUnique;
    const QuantizeResult both = run_quantize(img, cfg);
    CHECK(both.substrate_points <= half.substrate_points);
    for (const QuantizeResult *r : {&none, &half, &uniq, &both}) {
        CHECK(r->palette.size() == 16);
        CHECK(r->report.mse > 0.0);
        CHECK(r->mapping.indices.size() == img.pixels.size());
    }
    CHECK(std::string(sampling_mode_token(both.report.sampling)) == "both");
}

static void case_coarse_histogram() { // precluster.cpp:13-47, both overloads, exact integers
    std::vector<Rgb8> px;
    std::uint64_t st = 12345;
    for (int i = 0; i < 5000; ++i) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        px.push_back(Rgb8{static_cast<std::uint8_t>(st >> 56), static_cast<std::uint8_t>(st >> 48),
                          static_cast<std::uint8_t>((st >> 40) & 0x3f)});
    }
    CoarseHistogram want;
    for (const Rgb8 &p : px) {
        const std::size_t b = CoarseHistogram::bin_of(p);
        want.count[b] += 1;
        want.sum_r[b] += p.r;
        want.sum_g[b] += p.g;
        want.sum_b[b] += p.b;
        want.sum_sq[b] += static_cast<std::int64_t>(p.r) * p.r + static_cast<std::int64_t>(p.g) * p.g +
                          static_cast<std::int64_t>(p.b) * p.b;
    }
    const CoarseHistogram a = build_coarse_histogram(std::span<const Rgb8>(px));
    const CoarseHistogram b = build_coarse_histogram(build_histogram(px, 1));
    for (const CoarseHistogram *g : {&a, &b}) {
        CHECK(g->count == want.count);
        CHECK(g->sum_r == want.sum_r && g->sum_g == want.sum_g && g->sum_b == want.sum_b);
        CHECK(g->sum_sq == want.sum_sq);
    }
    bool threw = false;
    try {
        build_coarse_histogram(std::span<const Rgb8>());
    } catch (const std::invalid_argument &e) {
        threw = std::string(e.what()) == "build_coarse_histogram: no pixels";
    }
    CHECK(threw);
}

static void case_ppm_roundtrip() { // image.hpp:41-42: "P6\n<w> <h>\n255\n" + raw RGB
    RawImage img;
    img.width = 3;
    img.height = 2;
    for (int i = 0; i < 6; ++i)
        img.pixels.push_back(Rgb8{static_cast<std::uint8_t>(i * 40), static_cast<std::uint8_t>(255 - i),
                                  static_cast<std::uint8_t>(i)});
    const std::string path = "/tmp/cqg_dropin_test.ppm";
    save_image(img, path);
    {
        std::FILE *f = std::fopen(path.c_str(), "rb");
        char head[12] = {};
        CHECK(f && std::fread(head, 1, 11, f) == 11);
        if (f) std::fclose(f);
        CHECK(std::string(head, 11) == "P6\n3 2\n255\n");
    }
    const LoadedImage back = load_image(path);
    CHECK(back.image.width == 3 && back.image.height == 2);
    CHECK(std::memcmp(back.image.pixels.data(), img.pixels.data(), 18) == 0);
    // a comment between header tokens; a truncated raster
    {
        std::FILE *f = std::fopen(path.c_str(), "wb");
        const char data[] = "P6 # c\n3 2\n255\nabc";
        std::fwrite(data, 1, sizeof(data) - 1, f);
        std::fclose(f);
    }
    bool threw = false;
    try {
        load_image(path);
    } catch (const std::runtime_error &e) {
        threw = std::string(e.what()) == path + ": truncated PPM pixel data (expected 18 bytes, got 3)";
    }
    CHECK(threw);
    std::remove(path.c_str());
}

// bench.hpp (bench.cpp:27-113): the sweep through the device run_quantize on
// the golden 40x40 images saved as PPM; zero_time reruns byte-identical; a
// method outside the device path ("wu") gives error rows and the sweep goes on.
// argv[2] (optional) receives the CSV for the comparison with the reference
// library's rows (tests/test_gpu_cpp.py).
static void case_bench_sweep(const std::string &dir, const std::string &csv_out) {
    const std::string tmp = "/tmp/cqg_bench_sweep";
    std::string mk = "mkdir -p " + tmp;
    CHECK(std::system(mk.c_str()) == 0);
    BenchConfig bc;
    for (int seed_img : {61, 62}) {
        RawImage img;
        img.width = img.height = 40;
        img.pixels.resize(1600);
        std::ifstream f(dir + "/acc_" + std::to_string(seed_img) + ".rgb", std::ios::binary);
        f.read(reinterpret_cast<char *>(img.pixels.data()), 1600 * 3);
        CHECK(f.gcount() == 1600 * 3);
        const std::string path = tmp + "/acc_" + std::to_string(seed_img) + ".ppm";
        save_ppm(img, path);
        bc.image_paths.push_back(path);
    }
    bc.methods = {"wsm-kpp", "wsm-mmx", "wu"};
    bc.ks = {4, 8};
    bc.runs = 2;
    bc.seed_base = 3;
    bc.zero_time = true;
    std::ostringstream log;
    const BenchResults a = run_bench(bc, &log);
    CHECK(a.rows.size() == 2u * 3u * 2u * 2u);
    CHECK(a.error_count == 8); // "wu": a standalone preclusterer, outside the device path
    const std::string c1 = tmp + "/a.csv", c2 = tmp + "/b.csv";
    write_bench_csv(a, c1);
    write_bench_csv(run_bench(bc, nullptr), c2);
    auto slurp = [](const std::string &p) {
        std::ifstream f(p, std::ios::binary);
        return std::string(std::istreambuf_iterator<char>(f), {});
    };
    CHECK(slurp(c1) == slurp(c2));
    CHECK(slurp(c1).rfind("image,method,k,run,seed,sampling,", 0) == 0);
    // the same sweep with its cells shared out over 4 worker threads (a device context of 32 SMs
    // each): same rows, same CSV, same log
    set_bench_workers(4, 32);
    std::ostringstream log4;
    const BenchResults a4 = run_bench(bc, &log4);
    set_bench_workers(1);
    const std::string c4 = tmp + "/w4.csv";
    write_bench_csv(a4, c4);
    CHECK(slurp(c1) == slurp(c4));
    CHECK(log.str() == log4.str());
    CHECK(a4.error_count == a.error_count);
    const RankSummary rs = rank_aggregate(a);
    CHECK(rs.methods == std::vector<std::string>({"wsm-kpp", "wsm-mmx"})); // error rows do not rank
    if (!csv_out.empty()) write_bench_csv(a, csv_out);
}

int main(int argc, char **argv) {
    const std::string dir = argc > 1 ? argv[1] : "tests/golden";
    const std::string csv_out = argc > 2 ? argv[2] : "";
    struct Case {
        const char *name;
        void (*fn)();
    } cases[] = {{"histogram_order", case_histogram_order},
                 {"wsm_semantics", case_wsm_semantics},
                 {"histogram_equals_duplicates", case_histogram_equals_duplicates},
                 {"mapping", case_mapping},
                 {"report_format", case_report_format},
                 {"sampling_substrates", case_sampling_substrates},
                 {"coarse_histogram", case_coarse_histogram},
                 {"ppm_roundtrip", case_ppm_roundtrip}};
    for (const auto &c : cases) {
        const int before = g_fail;
        try {
            c.fn();
        } catch (const std::exception &e) {
            std::printf("  exception: %s\n", e.what());
            ++g_fail;
        }
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
    }
    {
        const int before = g_fail;
        try {
            case_golden_rows(dir);
        } catch (const std::exception &e) {
            std::printf("  exception: %s\n", e.what());
            ++g_fail;
        }
        std::printf("%s golden_rows\n", g_fail == before ? "PASS" : "FAIL");
    }
    {
        const int before = g_fail;
        try {
            case_bench_sweep(dir, csv_out);
        } catch (const std::exception &e) {
            std::printf("  exception: %s\n", e.what());
            ++g_fail;
        }
        std::printf("%s bench_sweep\n", g_fail == before ? "PASS" : "FAIL");
    }
    std::printf("%d failure(s)\n", g_fail);
    return g_fail == 0 ? 0 : 1;
}
