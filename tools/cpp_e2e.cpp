// End-to-end timing through the C++ drop-in (libquant_b200.so), the way a caller of the
// reference library uses it: pageable std::vector buffers, the full QuantizeResult returned.
//   cpp_e2e <image.ppm> <k> <method> <reps> <copies> <workers> <sms_per_worker>
// (a) quant::run_quantize on one host thread, `reps` calls;
// (b) quant::run_bench over `copies` copies of the image with 1 worker and with `workers`
//     worker threads (set_bench_workers), zero_time rows compared.
// Prints one JSON object. Built by paper_1101_0395_b200/_build.py; run by bench.py.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "quant/quant.hpp"

using namespace quant;
using clk = std::chrono::steady_clock;

static double ms_since(clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }

int main(int argc, char **argv) {
    if (argc < 8) {
        std::fprintf(stderr, "usage: cpp_e2e image.ppm k method reps copies workers sms_per_worker\n");
        return 2;
    }
    const std::string path = argv[1], method = argv[3];
    const int k = std::atoi(argv[2]), reps = std::atoi(argv[4]), copies = std::atoi(argv[5]),
              workers = std::atoi(argv[6]), sms = std::atoi(argv[7]);
    set_bench_workers(workers, sms); // before the first CUDA call: it also asks for 32 hardware queues
    set_bench_workers(1);
    const LoadedImage li = load_image(path);
    const double P = static_cast<double>(li.image.pixel_count());
    QuantizeConfig qc;
    qc.method = parse_method(method);
    qc.k = k;
    qc.seed = 202;
    for (int i = 0; i < 3; ++i) run_quantize(li.image, qc);
    const auto t0 = clk::now();
    double mse = 0.0;
    int iters = 0;
    for (int i = 0; i < reps; ++i) {
        const QuantizeResult r = run_quantize(li.image, qc);
        mse = r.report.mse;
        iters = r.state.iterations;
    }
    const double one_ms = ms_since(t0) / reps;

    BenchConfig bc;
    bc.image_paths.assign(static_cast<std::size_t>(copies), path);
    bc.methods = {method};
    bc.ks = {k};
    bc.runs = 1;
    bc.seed_base = 202;
    bc.zero_time = true;
    run_bench(bc, nullptr);
    const auto t1 = clk::now();
    const BenchResults b1 = run_bench(bc, nullptr);
    const double sweep1_ms = ms_since(t1);
    set_bench_workers(workers, sms);
    run_bench(bc, nullptr);
    const auto t2 = clk::now();
    const BenchResults bw = run_bench(bc, nullptr);
    const double sweepw_ms = ms_since(t2);
    bool same = b1.rows.size() == bw.rows.size() && b1.error_count == 0 && bw.error_count == 0;
    for (std::size_t i = 0; same && i < b1.rows.size(); ++i) same = b1.rows[i].csv_row() == bw.rows[i].csv_row();
    std::printf("{\"image\": \"%dx%d\", \"k\": %d, \"method\": \"%s\", \"iterations\": %d, \"mse\": %.17g, "
                "\"run_quantize\": {\"ms_per_call\": %.4f, \"mpixel_s\": %.2f, \"calls\": %d}, "
                "\"run_bench\": {\"images\": %d, \"one_worker_ms\": %.3f, \"one_worker_mpixel_s\": %.2f, "
                "\"workers\": %d, \"sms_per_worker\": %d, \"workers_ms\": %.3f, \"workers_mpixel_s\": %.2f, "
                "\"rows_equal\": %s, \"note\": \"wall clock, PPM load included\"}}\n",
                li.image.width, li.image.height, k, method.c_str(), iters, mse, one_ms, P / one_ms / 1e3, reps, copies,
                sweep1_ms, copies * P / sweep1_ms / 1e3, workers, sms, sweepw_ms, copies * P / sweepw_ms / 1e3,
                same ? "true" : "false");
    return same ? 0 : 1;
}
