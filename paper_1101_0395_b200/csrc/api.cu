// api.cu -- the extern "C" boundary of libcqg.so (declared in include/cqg.h).
//
// Validation mirrors the reference's exception sites and messages so the C++
// wrapper (quant:: API) can rethrow the same exception type and text:
//   histogram.cpp:70, init.cpp:15-19, kmeans.cpp:175-188 and :275,
//   metrics.cpp:16-17, pipeline.cpp:82-83.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "cqg_internal.cuh"

#include <map>
#include <mutex>

namespace {
thread_local std::string g_last_error;

// Results bound for pageable caller memory travel through the context's pinned
// staging buffers (copy_out) and are handed over here, at the end of the call:
// a cudaMemcpyAsync into pageable memory is staged by the driver under a
// device-wide lock and stalls the other contexts of a concurrent batch (cfg2,
// 16 images through 8 contexts, palette into a pageable array: 6.2 -> 9.2 ms;
// the C++ drop-in's std::vector outputs: 16 images in 23 ms).
struct PendingOut {
    cqg_ctx *ctx;
    void *dst;
    const void *src;
    size_t bytes;
};
thread_local std::vector<PendingOut> g_pending_out;

void finish_pending_out(bool ok) {
    if (g_pending_out.empty()) return;
    std::vector<PendingOut> todo;
    todo.swap(g_pending_out);
    for (const auto &p : todo) p.ctx->stage_out_used = 0;
    if (!ok) return;
    cudaStream_t last = nullptr;
    bool have = false;
    for (const auto &p : todo) {
        if (!have || p.ctx->stream != last) {
            if (cudaStreamSynchronize(p.ctx->stream) != cudaSuccess) cqg::fail(CQG_E_RUNTIME, "copy to host failed");
            last = p.ctx->stream;
            have = true;
        }
        std::memcpy(p.dst, p.src, p.bytes);
    }
}

template <class F>
int guarded(F &&f) {
    try {
        f();
        finish_pending_out(true);
        return CQG_OK;
    } catch (const cqg::Error &e) {
        finish_pending_out(false);
        g_last_error = e.msg;
        return e.code;
    } catch (const std::exception &e) {
        finish_pending_out(false);
        g_last_error = e.what();
        return CQG_E_RUNTIME;
    }
}

void use_device(cqg_ctx *ctx) {
    if (!ctx) cqg::fail(CQG_E_INVALID, "null cqg context");
    CQG_CUDA(cudaSetDevice(ctx->device));
    ctx->stage_in_used = 0; // every entry point synchronises its stream before it returns
}

void validate_k_init(int k, uint64_t n) {
    if (k < 1) cqg::fail(CQG_E_INVALID, "initialization: k must be at least 1");
    if ((uint64_t)k > n)
        cqg::fail(CQG_E_INVALID, "initialization: k (" + std::to_string(k) + ") exceeds distinct colors (" +
                                     std::to_string(n) + ")");
}

void validate_run(uint64_t n, int k, const cqg_term &t) {
    if (k <= 0) cqg::fail(CQG_E_INVALID, "clustering: no initial centers");
    if (n == 0) cqg::fail(CQG_E_INVALID, "clustering: no points");
    if ((uint64_t)k > n)
        cqg::fail(CQG_E_INVALID, "clustering: k (" + std::to_string(k) + ") exceeds number of points (" +
                                     std::to_string(n) + ")");
    if (t.epsilon < 0.0) cqg::fail(CQG_E_INVALID, "clustering: negative epsilon");
    if (t.max_iterations <= 0) cqg::fail(CQG_E_INVALID, "clustering: max_iterations < 1");
    if (k > 4096) cqg::fail(CQG_E_INVALID, "clustering: k > 4096 is not supported by the device engine");
}

void validate_pixels(uint64_t P, const char *who) {
    if (P >= (1ull << 32)) cqg::fail(CQG_E_INVALID, std::string(who) + ": more than 2^32-1 pixels");
}

struct Timer {
    // stage boundaries as events on the stream, read after the pipeline's own
    // final synchronisation (no host synchronisation between stages); the
    // events belong to the context (created once, not per call)
    cqg_ctx *ctx;
    bool on;
    cudaEvent_t *ev;
    int n = 0;
    Timer(cqg_ctx *c, bool enable) : ctx(c), on(enable), ev(c->stage_ev) {
        if (on) {
            if (!ev[0])
                for (int i = 0; i < 8; ++i) cudaEventCreate(&ev[i]);
            cudaEventRecord(ev[n++], ctx->stream);
        }
    }
    int lap() {
        if (!on || n >= 8) return 0;
        cudaEventRecord(ev[n], ctx->stream);
        return n++;
    }
    double ms(int i) const { // stage ending at lap i; call after the stream is synchronised
        if (!on || i <= 0) return 0.0;
        float t = 0.f;
        cudaEventElapsedTime(&t, ev[i - 1], ev[i]);
        return t;
    }
    ~Timer() = default;
};

} // namespace

namespace cqg {

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

void launched(cqg_ctx *ctx, int n) { ctx->launches += (unsigned long long)n; }

static int take_event(cqg_ctx *ctx) {
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        CQG_CUDA(cudaEventCreate(&e));
        ctx->ev_pool.push_back(e);
    }
    return (int)ctx->ev_used++;
}

int prof_begin(cqg_ctx *ctx) {
    if (!ctx->prof_on) return -1;
    const int e = take_event(ctx);
    CQG_CUDA(cudaEventRecord(ctx->ev_pool[e], ctx->stream));
    return e;
}

int prof_end(cqg_ctx *ctx, int cat, int begin, double units) {
    if (!ctx->prof_on || begin < 0) return -1;
    const int e = take_event(ctx);
    CQG_CUDA(cudaEventRecord(ctx->ev_pool[e], ctx->stream));
    ctx->prof_recs.push_back({cat, begin, e, units});
    return (int)ctx->prof_recs.size() - 1;
}

void prof_add_units(cqg_ctx *ctx, int rec, double units) {
    if (rec >= 0 && rec < (int)ctx->prof_recs.size()) ctx->prof_recs[rec].units += units;
}

static void prof_drain(cqg_ctx *ctx) {
    if (ctx->prof_recs.empty()) {
        ctx->ev_used = 0;
        return;
    }
    CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (const auto &r : ctx->prof_recs) {
        float ms = 0.f;
        CQG_CUDA(cudaEventElapsedTime(&ms, ctx->ev_pool[r.e0], ctx->ev_pool[r.e1]));
        ctx->prof_ms[r.cat] += ms;
        ctx->prof_units[r.cat] += r.units;
        ctx->prof_launches[r.cat] += 1;
    }
    ctx->prof_recs.clear();
    ctx->ev_used = 0;
}

static bool is_pageable_host(const void *p) {
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return attr.type == cudaMemoryTypeUnregistered;
}

// transfers up to this size go through pinned staging when the caller's memory is pageable
constexpr size_t kStageMax = 8u << 20; // larger ones keep the driver's pipelined pageable path

static void *next_stage(std::vector<HostBuf> &bufs, size_t &used, size_t bytes) {
    if (used == bufs.size()) bufs.emplace_back();
    return bufs[used++].ensure(bytes);
}

const void *stage_in(cqg_ctx *ctx, const void *user, size_t bytes, DevBuf &buf) {
    if (is_device_ptr(user)) return user;
    void *d = buf.ensure(bytes);
    const void *src = user;
    if (bytes <= kStageMax && is_pageable_host(user)) {
        void *h = next_stage(ctx->stage_in, ctx->stage_in_used, bytes);
        std::memcpy(h, user, bytes);
        src = h;
    }
    CQG_CUDA(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return d;
}

void copy_out(cqg_ctx *ctx, void *user, const void *dev, size_t bytes) {
    if (!user || bytes == 0 || user == dev) return;
    if (bytes <= kStageMax && is_pageable_host(user)) {
        void *h = next_stage(ctx->stage_out, ctx->stage_out_used, bytes);
        CQG_CUDA(cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        g_pending_out.push_back({ctx, user, h, bytes});
        return;
    }
    CQG_CUDA(cudaMemcpyAsync(user, dev, bytes, cudaMemcpyDefault, ctx->stream));
}

uint64_t read_scalar_u32(cqg_ctx *ctx, const uint32_t *dev) {
    uint32_t *h = static_cast<uint32_t *>(ctx->pinned.ensure(4096));
    CQG_CUDA(cudaMemcpyAsync(h, dev, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    return *h;
}

// pick the caller's buffer when it is device memory, else a context buffer
template <class T>
T *out_buf(void *user, DevBuf &buf, size_t count) {
    if (user && is_device_ptr(user)) return static_cast<T *>(user);
    return static_cast<T *>(buf.ensure(count * sizeof(T)));
}

// histogram into device buffers; returns N'
static uint64_t histogram_into(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t P, uint32_t *colors_d,
                               uint32_t *counts_d, uint32_t *first_d) {
    uint32_t *n_dev = static_cast<uint32_t *>(ctx->scal.ensure(256)) + 32;
    histogram_dev(ctx, rgb_d, P, colors_d, counts_d, first_d, n_dev);
    return read_scalar_u32(ctx, n_dev);
}

} // namespace cqg

using namespace cqg;

extern "C" {

const char *cqg_version(void) { return "cqg 0.1 (sm_100a)"; }

const char *cqg_last_error(void) { return g_last_error.c_str(); }

cqg_ctx *cqg_create(int device) {
    cqg_ctx *ctx = nullptr;
    const int rc = guarded([&] {
        int count = 0;
        CQG_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) fail(CQG_E_INVALID, "cqg_create: no CUDA device " + std::to_string(device));
        CQG_CUDA(cudaSetDevice(device));
        cudaDeviceProp prop{};
        CQG_CUDA(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            fail(CQG_E_CUDA, std::string("cqg_create: device ") + prop.name + " is not sm_100 (Blackwell)");
        ctx = new cqg_ctx();
        ctx->device = device;
        ctx->num_sms = prop.multiProcessorCount;
        ctx->dev_sms = prop.multiProcessorCount;
        CQG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
        CQG_CUDA(cudaStreamCreateWithFlags(&ctx->aux, cudaStreamNonBlocking));
        CQG_CUDA(cudaEventCreateWithFlags(&ctx->aux_fork, cudaEventDisableTiming));
        CQG_CUDA(cudaEventCreateWithFlags(&ctx->aux_join, cudaEventDisableTiming));
        CQG_CUDA(cudaEventCreateWithFlags(&ctx->lloyd_join, cudaEventDisableTiming));
        CQG_CUDA(cudaEventCreateWithFlags(&ctx->lloyd_fork, cudaEventDisableTiming));
        CQG_CUDA(cudaEventCreateWithFlags(&ctx->walk_fork, cudaEventDisableTiming));
        CQG_CUDA(cudaEventCreateWithFlags(&ctx->walk_join, cudaEventDisableTiming));
        CQG_CUDA(cudaStreamCreateWithFlags(&ctx->aux2, cudaStreamNonBlocking));
        const char *ng = getenv("CQG_NO_GRAPH");
        ctx->use_graphs = !(ng && ng[0] == '1');
        const char *nc = getenv("CQG_NO_CLUSTER_INIT");
        ctx->use_cluster_init = !(nc && nc[0] == '1');
        const char *cn = getenv("CQG_CLUSTER_NT");
        if (cn) ctx->cluster_nt = atoi(cn);
        const char *fs = getenv("CQG_DBG_INIT_FORCE_SEQ");
        if (fs) ctx->dbg_init_force_seq = atoi(fs);
        const char *nt = getenv("CQG_NO_INIT_TILE");
        ctx->use_init_tile = !(nt && nt[0] == '1');
        const char *tm = getenv("CQG_INIT_TILE_MIN");
        if (tm) ctx->init_tile_min = strtoull(tm, nullptr, 10);
        const char *np = getenv("CQG_NO_PRUNE");
        ctx->use_prune = !(np && np[0] == '1');
        const char *nn = getenv("CQG_NO_NDC_CODE");
        ctx->use_ndc_code = !(nn && nn[0] == '1');
        const char *nf = getenv("CQG_NO_FILTER_LIST");
        ctx->use_filter_list = !(nf && nf[0] == '1');
        const char *nw = getenv("CQG_DBG_NDC_WIN");
        if (nw) ctx->dbg_ndc_win = atoi(nw);
    });
    if (rc != CQG_OK) {
        delete ctx;
        return nullptr;
    }
    return ctx;
}

void cqg_destroy(cqg_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    release_graphs(ctx);
    shard_release(ctx);
    DevBuf *bufs[] = {&ctx->tab, &ctx->list, &ctx->bitmap, &ctx->wordpref, &ctx->scal, &ctx->img,
                      &ctx->colors, &ctx->counts, &ctx->first, &ctx->labels, &ctx->cen, &ctx->fcen,
                      &ctx->dtab, &ctx->dsorted, &ctx->order, &ctx->mom, &ctx->queue, &ctx->ndc,
                      &ctx->status, &ctx->sizes, &ctx->red, &ctx->hist_labels, &ctx->hist_centers,
                      &ctx->sse, &ctx->lut, &ctx->idx_out, &ctx->q_out, &ctx->mom_map, &ctx->coarse, &ctx->mind2,
                      &ctx->initpart, &ctx->initsel, &ctx->unit_draws, &ctx->inittile, &ctx->mom_g, &ctx->partial, &ctx->shard_log,
                      &ctx->bnd, &ctx->shift, &ctx->dcode, &ctx->rowmin, &ctx->snap_cen, &ctx->snap_lab, &ctx->ndc_keys, &ctx->dmom, &ctx->survivors,
                      &ctx->sub_img, &ctx->raw_col, &ctx->raw_cnt,
                      &ctx->full_col, &ctx->full_cnt, &ctx->map_rows, &ctx->map_lab, &ctx->pcnt, &ctx->pent, &ctx->pseg};
    for (DevBuf *b : bufs) b->release();
    ctx->pinned.release();
    ctx->pinned_nu.release();
    for (HostBuf &h : ctx->stage_out) h.release();
    for (HostBuf &h : ctx->stage_in) h.release();
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    for (cudaEvent_t e : ctx->stage_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->aux) {
        cudaStreamSynchronize(ctx->aux);
        cudaStreamDestroy(ctx->aux);
        if (ctx->aux2) {
            cudaStreamSynchronize(ctx->aux2);
            cudaStreamDestroy(ctx->aux2);
        }
        cudaEventDestroy(ctx->aux_fork);
        cudaEventDestroy(ctx->aux_join);
        cudaEventDestroy(ctx->lloyd_join);
        cudaEventDestroy(ctx->lloyd_fork);
        cudaEventDestroy(ctx->walk_fork);
        cudaEventDestroy(ctx->walk_join);
    }
    delete ctx;
}

int cqg_set_stream(cqg_ctx *ctx, void *stream) {
    return guarded([&] {
        use_device(ctx);
        if (!stream) {
            if (!ctx->own_stream) {
                CQG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
                ctx->own_stream = true;
            }
            return;
        }
        if (ctx->own_stream) {
            cudaStreamSynchronize(ctx->stream);
            cudaStreamDestroy(ctx->stream);
        }
        release_graphs(ctx);
        ctx->stream = static_cast<cudaStream_t>(stream);
        ctx->own_stream = false;
    });
}

uint64_t cqg_launch_count(const cqg_ctx *ctx) { return ctx ? ctx->launches : 0; }

int cqg_set_sm_budget(cqg_ctx *ctx, int sms) {
    return guarded([&] {
        if (!ctx) fail(CQG_E_INVALID, "cqg_set_sm_budget: null context");
        if (sms < 0) fail(CQG_E_INVALID, "cqg_set_sm_budget: negative SM count");
        use_device(ctx);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
        ctx->num_sms = (sms == 0 || sms >= ctx->dev_sms) ? ctx->dev_sms : (sms < 16 ? 16 : sms);
        release_graphs(ctx); // captured launch geometries follow the budget
    });
}

int cqg_set_profiling(cqg_ctx *ctx, int on) {
    return guarded([&] {
        use_device(ctx);
        prof_drain(ctx);
        ctx->prof_on = on != 0;
    });
}

int cqg_read_profile(cqg_ctx *ctx, cqg_profile *out, int reset) {
    return guarded([&] {
        use_device(ctx);
        prof_drain(ctx);
        if (out) {
            for (int i = 0; i < CQG_PROF_N; ++i) {
                out->ms[i] = ctx->prof_ms[i];
                out->units[i] = ctx->prof_units[i];
                out->launches[i] = ctx->prof_launches[i];
            }
        }
        if (reset) {
            for (int i = 0; i < CQG_PROF_N; ++i) {
                ctx->prof_ms[i] = 0;
                ctx->prof_units[i] = 0;
                ctx->prof_launches[i] = 0;
            }
        }
    });
}

int cqg_bench_sweep(cqg_ctx *ctx, int reps, double *ms_per_launch, double *units_per_launch) {
    return guarded([&] {
        use_device(ctx);
        if (!ctx->have_last_sweep) fail(CQG_E_INVALID, "cqg_bench_sweep: no Lloyd run on this context yet");
        if (reps < 1) reps = 1;
        double ms = 0.0, units = 0.0;
        bench_sweep_dev(ctx, reps, &ms, &units);
        if (ms_per_launch) *ms_per_launch = ms;
        if (units_per_launch) *units_per_launch = units;
    });
}

int cqg_histogram(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, uint32_t *colors, uint32_t *counts,
                  uint32_t *first, uint64_t *n_unique) {
    return guarded([&] {
        use_device(ctx);
        if (P == 0 || !rgb) fail(CQG_E_INVALID, "build_histogram: no pixels");
        validate_pixels(P, "build_histogram");
        const uint64_t cap = P < (1ull << 24) ? P : (1ull << 24);
        const uint8_t *rgb_d = static_cast<const uint8_t *>(stage_in(ctx, rgb, P * 3, ctx->img));
        uint32_t *col_d = out_buf<uint32_t>(colors, ctx->colors, cap);
        uint32_t *cnt_d = out_buf<uint32_t>(counts, ctx->counts, cap);
        uint32_t *fst_d = first ? out_buf<uint32_t>(first, ctx->first, cap) : nullptr;
        const uint64_t n = histogram_into(ctx, rgb_d, P, col_d, cnt_d, fst_d);
        copy_out(ctx, colors, col_d, n * 4);
        copy_out(ctx, counts, cnt_d, n * 4);
        if (first) copy_out(ctx, first, fst_d, n * 4);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (n_unique) *n_unique = n;
    });
}

static void init_common(cqg_ctx *ctx, int kind, const uint32_t *colors, const uint32_t *counts, uint64_t n,
                        uint64_t P, int k, uint64_t seed, int weighted_first, double *centers) {
    use_device(ctx);
    validate_k_init(k, n);
    if (P == 0) fail(CQG_E_INVALID, "initialization: zero source pixel count");
    const uint32_t *col_d = static_cast<const uint32_t *>(stage_in(ctx, colors, n * 4, ctx->colors));
    const uint32_t *cnt_d = static_cast<const uint32_t *>(stage_in(ctx, counts, n * 4, ctx->counts));
    double *cen_d = out_buf<double>(centers, ctx->cen, 3 * (size_t)k);
    if (kind == CQG_INIT_MAXIMIN) init_maximin_dev(ctx, col_d, cnt_d, n, P, k, seed, weighted_first, cen_d);
    else init_kmeanspp_dev(ctx, col_d, cnt_d, n, P, k, seed, cen_d);
    copy_out(ctx, centers, cen_d, 24 * (size_t)k);
    CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    CQG_CUDA(cudaGetLastError());
}

int cqg_init_maximin(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n, uint64_t P,
                     int k, uint64_t seed, int weighted_first, double *centers) {
    return guarded([&] { init_common(ctx, CQG_INIT_MAXIMIN, colors, counts, n, P, k, seed, weighted_first, centers); });
}

int cqg_init_kmeanspp(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n, uint64_t P,
                      int k, uint64_t seed, double *centers) {
    return guarded([&] { init_common(ctx, CQG_INIT_KMEANSPP, colors, counts, n, P, k, seed, 1, centers); });
}

int cqg_lloyd(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n, uint64_t P,
              const double *init, int k, const cqg_term *term, double *centers, uint32_t *labels,
              double *sse_trace, cqg_lloyd_stats *stats, uint32_t *hist_labels, double *hist_centers) {
    return guarded([&] {
        use_device(ctx);
        if (!term) fail(CQG_E_INVALID, "clustering: null termination");
        validate_run(n, k, *term);
        if (!init || !centers || !sse_trace) fail(CQG_E_INVALID, "cqg_lloyd: null output");
        if (P == 0) fail(CQG_E_INVALID, "wsm: weights must be positive");
        if (!is_device_ptr(counts)) {
            uint64_t tot = 0;
            for (uint64_t i = 0; i < n; ++i) {
                if (counts[i] == 0) fail(CQG_E_INVALID, "wsm: weights must be positive");
                tot += counts[i];
            }
            if (tot > P) fail(CQG_E_INVALID, "cqg_lloyd: counts exceed the source pixel count");
        }
        const uint32_t *col_d = static_cast<const uint32_t *>(stage_in(ctx, colors, n * 4, ctx->colors));
        const uint32_t *cnt_d = static_cast<const uint32_t *>(stage_in(ctx, counts, n * 4, ctx->counts));
        const double *init_d = static_cast<const double *>(stage_in(ctx, init, 24 * (size_t)k, ctx->initsel));
        uint32_t *lab_d = out_buf<uint32_t>(labels, ctx->labels, n);
        double *cen_d = out_buf<double>(centers, ctx->cen, 3 * (size_t)k);
        if (cen_d == init_d) fail(CQG_E_INVALID, "cqg_lloyd: centers must not alias init");
        LloydOut o = lloyd_dev(ctx, col_d, cnt_d, n, P, init_d, k, *term, lab_d, cen_d, sse_trace,
                               hist_labels, hist_centers);
        copy_out(ctx, centers, cen_d, 24 * (size_t)k);
        copy_out(ctx, labels, lab_d, 4 * n);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (stats) {
            stats->iterations = o.iterations;
            stats->repair_count = o.repairs;
            stats->ndc_total = o.ndc;
            stats->n_points = n;
            stats->flagged_total = o.flagged;
            stats->swept_total = o.swept;
        }
    });
}

int cqg_lloyd_exact(cqg_ctx *ctx, const double *points, const double *weights, uint64_t n, const double *init,
                    int k, const cqg_term *term, double *centers, uint32_t *labels, double *sse_trace,
                    cqg_lloyd_stats *stats, uint32_t *hist_labels, double *hist_centers) {
    return guarded([&] {
        use_device(ctx);
        if (!term) fail(CQG_E_INVALID, "clustering: null termination");
        validate_run(n, k, *term); // kmeans.cpp:173-188
        if (term->fixed_iterations < 0) fail(CQG_E_INVALID, "clustering: fixed_iterations < 1");
        if (!points || !init || !centers || !sse_trace) fail(CQG_E_INVALID, "cqg_lloyd_exact: null argument");
        const double *pts_d = static_cast<const double *>(stage_in(ctx, points, 24 * n, ctx->raw_col));
        const double *w_d = nullptr;
        if (weights) {
            if (!is_device_ptr(weights))
                for (uint64_t i = 0; i < n; ++i)
                    if (!(weights[i] > 0.0)) fail(CQG_E_INVALID, "wsm: weights must be positive"); // kmeans.cpp:275
            w_d = static_cast<const double *>(stage_in(ctx, weights, 8 * n, ctx->raw_cnt));
        }
        const double *init_d = static_cast<const double *>(stage_in(ctx, init, 24 * (size_t)k, ctx->initsel));
        uint32_t *lab_d = out_buf<uint32_t>(labels, ctx->labels, n);
        double *cen_d = out_buf<double>(centers, ctx->cen, 3 * (size_t)k);
        if (cen_d == init_d) fail(CQG_E_INVALID, "cqg_lloyd_exact: centers must not alias init");
        const ExactOut o = exact_lloyd_dev(ctx, pts_d, w_d, n, init_d, k, *term, weights != nullptr, lab_d, cen_d,
                                           sse_trace, hist_labels, hist_centers);
        copy_out(ctx, centers, cen_d, 24 * (size_t)k);
        copy_out(ctx, labels, lab_d, 4 * n);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (stats) {
            *stats = cqg_lloyd_stats{};
            stats->iterations = o.iterations;
            stats->repair_count = o.repairs;
            stats->ndc_total = o.ndc;
            stats->n_points = n;
            stats->swept_total = n * (uint64_t)o.iterations;
        }
    });
}

int cqg_compute_sse(cqg_ctx *ctx, const double *points, const double *weights, uint64_t n, const double *centers,
                    int k, const uint32_t *labels, double *sse) {
    return guarded([&] {
        use_device(ctx);
        if (!sse) fail(CQG_E_INVALID, "compute_sse: null output");
        if (n == 0) {
            *sse = 0.0;
            return;
        }
        if (!points || !centers || !labels || k < 1) fail(CQG_E_INVALID, "compute_sse: null argument");
        const double *pts_d = static_cast<const double *>(stage_in(ctx, points, 24 * n, ctx->raw_col));
        const double *w_d = weights ? static_cast<const double *>(stage_in(ctx, weights, 8 * n, ctx->raw_cnt)) : nullptr;
        const double *cen_d = static_cast<const double *>(stage_in(ctx, centers, 24 * (size_t)k, ctx->initsel));
        const uint32_t *lab_d = static_cast<const uint32_t *>(stage_in(ctx, labels, 4 * n, ctx->labels));
        double *scratch = static_cast<double *>(ctx->ndc.ensure(64)) + 4;
        *sse = exact_sse_dev(ctx, pts_d, w_d, n, cen_d, lab_d, scratch);
    });
}

int cqg_repair_empty_clusters(cqg_ctx *ctx, const double *points, const double *weights, uint64_t n,
                              double *centers, int k, uint32_t *labels, int *repairs) {
    return guarded([&] {
        use_device(ctx);
        if (!points || !weights || !centers || !labels || k < 1 || n == 0)
            fail(CQG_E_INVALID, "repair_empty_clusters: empty input");
        const double *pts_d = static_cast<const double *>(stage_in(ctx, points, 24 * n, ctx->raw_col));
        const double *w_d = static_cast<const double *>(stage_in(ctx, weights, 8 * n, ctx->raw_cnt));
        double *cen_d = out_buf<double>(centers, ctx->cen, 3 * (size_t)k);
        uint32_t *lab_d = out_buf<uint32_t>(labels, ctx->labels, n);
        if (cen_d != centers) CQG_CUDA(cudaMemcpyAsync(cen_d, centers, 24 * (size_t)k, cudaMemcpyDefault, ctx->stream));
        if (lab_d != labels) CQG_CUDA(cudaMemcpyAsync(lab_d, labels, 4 * n, cudaMemcpyDefault, ctx->stream));
        const int r = exact_repair_dev(ctx, pts_d, w_d, n, cen_d, k, lab_d);
        copy_out(ctx, centers, cen_d, 24 * (size_t)k);
        copy_out(ctx, labels, lab_d, 4 * n);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (repairs) *repairs = r;
    });
}

int cqg_center_table(cqg_ctx *ctx, const double *centers, int k, double *dist2, uint32_t *order) {
    return guarded([&] {
        use_device(ctx);
        if (k < 1) {
            return;
        }
        if (!centers || !dist2 || !order) fail(CQG_E_INVALID, "build_center_distance_table: null argument");
        if (k > 4096) fail(CQG_E_INVALID, "build_center_distance_table: k > 4096 is not supported");
        const double *cen_d = static_cast<const double *>(stage_in(ctx, centers, 24 * (size_t)k, ctx->initsel));
        double *dist_d = out_buf<double>(dist2, ctx->dtab, (size_t)k * k);
        uint32_t *ord_d = out_buf<uint32_t>(order, ctx->order, (size_t)k * k);
        exact_table_dev(ctx, cen_d, k, dist_d, ord_d);
        copy_out(ctx, dist2, dist_d, 8 * (size_t)k * k);
        copy_out(ctx, order, ord_d, 4 * (size_t)k * k);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cqg_kmeanspp_next_masses(cqg_ctx *ctx, const double *colors, const double *weights, uint64_t n,
                             const double *centers, int k, double *masses) {
    return guarded([&] {
        use_device(ctx);
        if (n == 0) return;
        if (!colors || !weights || !masses || (k > 0 && !centers))
            fail(CQG_E_INVALID, "kmeanspp_next_masses: null argument");
        if (k <= 0) { // init.cpp:318: the weights themselves
            CQG_CUDA(cudaMemcpyAsync(masses, weights, 8 * n, cudaMemcpyDefault, ctx->stream));
            CQG_CUDA(cudaStreamSynchronize(ctx->stream));
            return;
        }
        const double *pts_d = static_cast<const double *>(stage_in(ctx, colors, 24 * n, ctx->raw_col));
        const double *w_d = static_cast<const double *>(stage_in(ctx, weights, 8 * n, ctx->raw_cnt));
        const double *cen_d = static_cast<const double *>(stage_in(ctx, centers, 24 * (size_t)k, ctx->initsel));
        double *m_d = out_buf<double>(masses, ctx->first, n);
        exact_next_masses_dev(ctx, pts_d, w_d, n, cen_d, k, m_d);
        copy_out(ctx, masses, m_d, 8 * n);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cqg_maximin_pad(cqg_ctx *ctx, const double *colors, uint64_t n, const double *centers, int k0, int k,
                    double *out) {
    return guarded([&] {
        use_device(ctx);
        validate_k_init(k, n); // init.cpp:325 (validate_k)
        if (k0 < 1 || !centers) fail(CQG_E_INVALID, "maximin_pad: need at least one center");
        if (!out || !colors) fail(CQG_E_INVALID, "maximin_pad: null argument");
        const int kk = k0 > k ? k0 : k;
        double *cen_d = out_buf<double>(out, ctx->cen, 3 * (size_t)kk);
        CQG_CUDA(cudaMemcpyAsync(cen_d, centers, 24 * (size_t)k0, cudaMemcpyDefault, ctx->stream));
        if (k0 < k) {
            const double *pts_d = static_cast<const double *>(stage_in(ctx, colors, 24 * n, ctx->raw_col));
            exact_maximin_pad_dev(ctx, pts_d, n, cen_d, k0, k);
        }
        copy_out(ctx, out, cen_d, 24 * (size_t)kk);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cqg_shard_begin(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n_local, uint64_t P,
                    const double *init, int k, const cqg_term *term) {
    return guarded([&] {
        use_device(ctx);
        if (!term) fail(CQG_E_INVALID, "clustering: null termination");
        if (k <= 0) fail(CQG_E_INVALID, "clustering: no initial centers");
        if (term->epsilon < 0.0) fail(CQG_E_INVALID, "clustering: negative epsilon");
        if (term->max_iterations <= 0) fail(CQG_E_INVALID, "clustering: max_iterations < 1");
        if (k > 1024) fail(CQG_E_INVALID, "clustering: k > 1024 is not supported by the sharded engine");
        if (P == 0) fail(CQG_E_INVALID, "wsm: weights must be positive");
        const uint32_t *col_d = n_local ? static_cast<const uint32_t *>(stage_in(ctx, colors, n_local * 4, ctx->colors))
                                        : static_cast<const uint32_t *>(ctx->colors.ensure(4));
        const uint32_t *cnt_d = n_local ? static_cast<const uint32_t *>(stage_in(ctx, counts, n_local * 4, ctx->counts))
                                        : static_cast<const uint32_t *>(ctx->counts.ensure(4));
        const double *init_d = static_cast<const double *>(stage_in(ctx, init, 24 * (size_t)k, ctx->initsel));
        shard_begin_dev(ctx, col_d, cnt_d, n_local, P, init_d, k, *term);
    });
}

static int shard_partial(cqg_ctx *ctx, int64_t *partial, bool run) {
    return guarded([&] {
        use_device(ctx);
        const size_t bytes = 8 * (5 * (size_t)shard_k(ctx) + 2);
        long long *d = is_device_ptr(partial) ? reinterpret_cast<long long *>(partial)
                                              : static_cast<long long *>(ctx->partial.ensure(bytes));
        shard_assign_dev(ctx, d, run);
        copy_out(ctx, partial, d, bytes);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cqg_shard_assign(cqg_ctx *ctx, int64_t *partial) { return shard_partial(ctx, partial, true); }
int cqg_shard_moments(cqg_ctx *ctx, int64_t *partial) { return shard_partial(ctx, partial, false); }

int cqg_shard_finalize(cqg_ctx *ctx, const int64_t *global, int *state, double *sse) {
    return guarded([&] {
        use_device(ctx);
        const size_t bytes = 8 * (5 * (size_t)shard_k(ctx) + 2);
        const long long *g = static_cast<const long long *>(stage_in(ctx, global, bytes, ctx->partial));
        const int st = shard_finalize_dev(ctx, g, sse);
        if (state) *state = st;
    });
}

int cqg_shard_finalize_async(cqg_ctx *ctx, const int64_t *global) {
    return guarded([&] {
        use_device(ctx);
        if (!is_device_ptr(global)) fail(CQG_E_INVALID, "cqg_shard_finalize_async: global must be device memory");
        shard_finalize_async_dev(ctx, reinterpret_cast<const long long *>(global));
    });
}

int cqg_shard_status(cqg_ctx *ctx, int *state, int *iterations) {
    return guarded([&] {
        use_device(ctx);
        const int st = shard_status_dev(ctx, iterations);
        if (state) *state = st;
    });
}

int cqg_shard_sizes(cqg_ctx *ctx, uint32_t *sizes) {
    return guarded([&] {
        use_device(ctx);
        const size_t bytes = 4 * (size_t)shard_k(ctx);
        uint32_t *d = out_buf<uint32_t>(sizes, ctx->sizes, (size_t)shard_k(ctx));
        shard_sizes_dev(ctx, d);
        copy_out(ctx, sizes, d, bytes);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cqg_shard_donor(cqg_ctx *ctx, const uint32_t *global_sizes, int fallback, double *value, uint64_t *local_index,
                    uint32_t *colour, uint32_t *label) {
    return guarded([&] {
        use_device(ctx);
        const uint32_t *g = static_cast<const uint32_t *>(
            stage_in(ctx, global_sizes, 4 * (size_t)shard_k(ctx), ctx->status));
        double v;
        uint64_t i;
        uint32_t c, l;
        shard_donor_dev(ctx, g, fallback, &v, &i, &c, &l);
        if (value) *value = v;
        if (local_index) *local_index = i;
        if (colour) *colour = c;
        if (label) *label = l;
    });
}

int cqg_shard_move(cqg_ctx *ctx, uint64_t local_index, int e, uint32_t colour) {
    return guarded([&] {
        use_device(ctx);
        if (e < 0 || e >= shard_k(ctx)) fail(CQG_E_INVALID, "cqg_shard_move: cluster out of range");
        shard_move_dev(ctx, local_index, e, colour);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cqg_shard_end(cqg_ctx *ctx, double *centers, uint32_t *labels, double *sse_trace, int *iterations) {
    return guarded([&] {
        use_device(ctx);
        const int it = shard_end_dev(ctx, centers, labels, sse_trace);
        if (iterations) *iterations = it;
    });
}

static void coarse_out(cqg_ctx *ctx, const unsigned long long *tab, uint64_t *count, int64_t *sum_r,
                       int64_t *sum_g, int64_t *sum_b, int64_t *sum_sq) {
    void *outs[5] = {count, sum_r, sum_g, sum_b, sum_sq};
    for (int f = 0; f < 5; ++f) copy_out(ctx, outs[f], tab + (size_t)f * 32768, sizeof(uint64_t) * 32768);
    CQG_CUDA(cudaStreamSynchronize(ctx->stream));
}

int cqg_coarse_histogram(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, uint64_t *count, int64_t *sum_r,
                         int64_t *sum_g, int64_t *sum_b, int64_t *sum_sq) {
    return guarded([&] {
        use_device(ctx);
        if (P == 0 || !rgb) fail(CQG_E_INVALID, "build_coarse_histogram: no pixels");
        if (!count || !sum_r || !sum_g || !sum_b || !sum_sq) fail(CQG_E_INVALID, "build_coarse_histogram: null output");
        validate_pixels(P, "build_coarse_histogram");
        // the distinct colours and their counts first (the same device
        // histogram as build_histogram), then 5 reductions per colour
        const uint64_t cap = P < (1ull << 24) ? P : (1ull << 24);
        const uint8_t *rgb_d = static_cast<const uint8_t *>(stage_in(ctx, rgb, P * 3, ctx->img));
        uint32_t *col_d = static_cast<uint32_t *>(ctx->colors.ensure(cap * 4));
        uint32_t *cnt_d = static_cast<uint32_t *>(ctx->counts.ensure(cap * 4));
        const uint64_t n = histogram_into(ctx, rgb_d, P, col_d, cnt_d, nullptr);
        unsigned long long *tab = static_cast<unsigned long long *>(ctx->coarse.ensure(sizeof(uint64_t) * 5 * 32768));
        coarse_hist_dev(ctx, col_d, cnt_d, n, tab);
        coarse_out(ctx, tab, count, sum_r, sum_g, sum_b, sum_sq);
    });
}

int cqg_coarse_histogram_weighted(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n,
                                  uint64_t *count, int64_t *sum_r, int64_t *sum_g, int64_t *sum_b,
                                  int64_t *sum_sq) {
    return guarded([&] {
        use_device(ctx);
        if (n == 0 || !colors || !counts) fail(CQG_E_INVALID, "build_coarse_histogram: empty histogram");
        if (!count || !sum_r || !sum_g || !sum_b || !sum_sq) fail(CQG_E_INVALID, "build_coarse_histogram: null output");
        const uint32_t *col_d = static_cast<const uint32_t *>(stage_in(ctx, colors, n * 4, ctx->raw_col));
        const uint32_t *cnt_d = static_cast<const uint32_t *>(stage_in(ctx, counts, n * 4, ctx->raw_cnt));
        unsigned long long *tab = static_cast<unsigned long long *>(ctx->coarse.ensure(sizeof(uint64_t) * 5 * 32768));
        coarse_hist_dev(ctx, col_d, cnt_d, n, tab);
        coarse_out(ctx, tab, count, sum_r, sum_g, sum_b, sum_sq);
    });
}

int cqg_map(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, const double *palette, int k, void *indices,
            int index_bytes, uint8_t *quantized, double *mean_sq_dist, uint64_t *ndc) {
    return guarded([&] {
        use_device(ctx);
        if (k < 1 || !palette) fail(CQG_E_INVALID, "map_pixels: empty palette");
        if (P == 0 || !rgb) fail(CQG_E_INVALID, "map_pixels: empty image");
        validate_pixels(P, "map_pixels");
        if (k > 4096) fail(CQG_E_INVALID, "map_pixels: palettes above 4096 entries are not supported");
        if (index_bytes != 1 && index_bytes != 4) fail(CQG_E_INVALID, "map_pixels: index_bytes must be 1 or 4");
        if (index_bytes == 1 && k > 256) fail(CQG_E_INVALID, "map_pixels: 8-bit indices need k <= 256");
        const uint64_t cap = P < (1ull << 24) ? P : (1ull << 24);
        const uint8_t *rgb_d = static_cast<const uint8_t *>(stage_in(ctx, rgb, P * 3, ctx->img));
        const double *pal_d = static_cast<const double *>(stage_in(ctx, palette, 24 * (size_t)k, ctx->initsel));
        uint32_t *col_d = static_cast<uint32_t *>(ctx->colors.ensure(cap * 4));
        uint32_t *cnt_d = static_cast<uint32_t *>(ctx->counts.ensure(cap * 4));
        const uint64_t n = histogram_into(ctx, rgb_d, P, col_d, cnt_d, nullptr);
        void *idx_d = indices ? out_buf<uint8_t>(indices, ctx->idx_out, P * (size_t)index_bytes) : nullptr;
        uint8_t *q_d = quantized ? out_buf<uint8_t>(quantized, ctx->q_out, P * 3) : nullptr;
        unsigned long long *ndc_h =
            ndc ? reinterpret_cast<unsigned long long *>(static_cast<char *>(ctx->pinned.ensure(4096)) + 3072) : nullptr;
        const double mse = map_dev(ctx, rgb_d, P, col_d, cnt_d, n, pal_d, k, idx_d, index_bytes, q_d, nullptr, nullptr,
                                   ndc_h);
        copy_out(ctx, indices, idx_d, P * (size_t)index_bytes);
        copy_out(ctx, quantized, q_d, P * 3);
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
        if (mean_sq_dist) *mean_sq_dist = mse;
        if (ndc) *ndc = *ndc_h;
    });
}

int cqg_quantize(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, const cqg_quantize_cfg *cfg, const double *init,
                 double *palette, uint32_t *labels, double *sse_trace, void *indices, uint8_t *quantized,
                 cqg_quantize_stats *stats) {
    return guarded([&] {
        use_device(ctx);
        if (P == 0 || !rgb) fail(CQG_E_INVALID, "run_quantize: empty image");
        if (!cfg) fail(CQG_E_INVALID, "run_quantize: null config");
        const int k = cfg->k;
        if (k < 1) fail(CQG_E_INVALID, "run_quantize: k must be at least 1");
        validate_pixels(P, "run_quantize");
        if (!palette) fail(CQG_E_INVALID, "run_quantize: null palette output");
        if (cfg->index_bytes != 1 && cfg->index_bytes != 4)
            fail(CQG_E_INVALID, "map_pixels: index_bytes must be 1 or 4");
        const int ib = cfg->index_bytes;
        if (ib == 1 && k > 256) fail(CQG_E_INVALID, "map_pixels: 8-bit indices need k <= 256");
        const int mode = cfg->sampling;
        if (mode < CQG_SAMPLING_UNIQUE || mode > CQG_SAMPLING_BOTH)
            fail(CQG_E_INVALID, "run_quantize: unknown sampling mode");
        const bool sub = mode == CQG_SAMPLING_TWO_TO_ONE || mode == CQG_SAMPLING_BOTH; // pipeline.cpp:91-92
        const bool dedup = mode == CQG_SAMPLING_UNIQUE || mode == CQG_SAMPLING_BOTH;   // pipeline.cpp:93-94
        if (sub && (cfg->width < 1 || cfg->height < 1 || (uint64_t)cfg->width * cfg->height != P))
            fail(CQG_E_INVALID, "run_quantize: 2:1 sampling needs width * height == pixel count");
        Timer tm(ctx, stats != nullptr && ctx->prof_on); // stage events only when profiling
        const uint8_t *rgb_d = static_cast<const uint8_t *>(stage_in(ctx, rgb, P * 3, ctx->img));
        // the sampled pixels (S of them) and their histogram (initialisers, dedup substrate)
        const uint8_t *smp_d = rgb_d;
        uint64_t S = P;
        if (sub) {
            S = (uint64_t)((cfg->width + 1) / 2) * ((cfg->height + 1) / 2);
            uint8_t *o = static_cast<uint8_t *>(ctx->sub_img.ensure(3 * S + 16));
            subsample_2to1_dev(ctx, rgb_d, cfg->width, cfg->height, o);
            smp_d = o;
        }
        const uint64_t cap = S < (1ull << 24) ? S : (1ull << 24);
        uint32_t *col_d = static_cast<uint32_t *>(ctx->colors.ensure(cap * 4));
        uint32_t *cnt_d = static_cast<uint32_t *>(ctx->counts.ensure(cap * 4));
        const uint64_t n = histogram_into(ctx, smp_d, S, col_d, cnt_d, nullptr);
        const int t_hist = tm.lap();

        double *init_d = static_cast<double *>(ctx->initsel.ensure(24 * (size_t)k + 64));
        if (cfg->init_kind == CQG_INIT_GIVEN) {
            if (!init) fail(CQG_E_INVALID, "run_quantize: initial centres required");
            CQG_CUDA(cudaMemcpyAsync(init_d, init, 24 * (size_t)k, cudaMemcpyDefault, ctx->stream));
        } else {
            validate_k_init(k, n);
            double *tmp = static_cast<double *>(ctx->hist_centers.ensure(24 * (size_t)k));
            if (cfg->init_kind == CQG_INIT_MAXIMIN) init_maximin_dev(ctx, col_d, cnt_d, n, S, k, cfg->seed, 1, tmp);
            else if (cfg->init_kind == CQG_INIT_KMEANSPP) init_kmeanspp_dev(ctx, col_d, cnt_d, n, S, k, cfg->seed, tmp);
            else fail(CQG_E_INVALID, "run_quantize: unknown initializer kind");
            CQG_CUDA(cudaMemcpyAsync(init_d, tmp, 24 * (size_t)k, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        const int t_init = tm.lap();

        // substrate: the distinct colours (count weights) or every sampled pixel (count 1, weight 1/S)
        const uint32_t *sub_col = col_d, *sub_cnt = cnt_d;
        uint64_t ns = n;
        if (!dedup) {
            uint32_t *rc = static_cast<uint32_t *>(ctx->raw_col.ensure(S * 4 + 16));
            uint32_t *rn = static_cast<uint32_t *>(ctx->raw_cnt.ensure(S * 4 + 16));
            pack_pixels_dev(ctx, smp_d, S, rc, rn);
            sub_col = rc;
            sub_cnt = rn;
            ns = S;
        }
        cqg_term term = cfg->term;
        term.record_history = 0;
        validate_run(ns, k, term);
        uint32_t *lab_d = static_cast<uint32_t *>(ctx->labels.ensure((ns > cap ? ns : cap) * 4));
        double *cen_d = static_cast<double *>(ctx->cen.ensure(24 * (size_t)k));
        const int limit = term.fixed_iterations > 0 ? term.fixed_iterations : term.max_iterations;
        double *sse_h = static_cast<double *>(ctx->pinned.ensure(4096 + 8 * (size_t)limit)) + 512;
        // the persistent Lloyd kernel's status is checked after the pipeline's
        // final synchronisation (not before the mapping is enqueued); the
        // subsampled modes read a histogram count in between, so they do not defer
        const bool defer = !sub;
        LloydOut o = lloyd_dev(ctx, sub_col, sub_cnt, ns, S, init_d, k, term, lab_d, cen_d, sse_h, nullptr, nullptr,
                               defer);
        if (!o.pending && sse_trace) std::memcpy(sse_trace, sse_h, 8 * (size_t)o.iterations);
        const int t_lloyd = tm.lap();

        // mapping over the full image needs its distinct colours: the histogram
        // above unless the image was subsampled
        const uint32_t *map_col = col_d, *map_cnt = cnt_d;
        uint64_t nm = n;
        if (sub) {
            const uint64_t capf = P < (1ull << 24) ? P : (1ull << 24);
            uint32_t *fc = static_cast<uint32_t *>(ctx->full_col.ensure(capf * 4));
            uint32_t *fn = static_cast<uint32_t *>(ctx->full_cnt.ensure(capf * 4));
            nm = histogram_into(ctx, rgb_d, P, fc, fn, nullptr);
            map_col = fc;
            map_cnt = fn;
        }
        void *idx_d = indices ? out_buf<uint8_t>(indices, ctx->idx_out, P * (size_t)ib) : nullptr;
        uint8_t *q_d = quantized ? out_buf<uint8_t>(quantized, ctx->q_out, P * 3) : nullptr;
        double *mse_h = static_cast<double *>(ctx->pinned.ensure(4096)) + 256; // bytes 2048.. (free here)
        unsigned long long *mndc_h = reinterpret_cast<unsigned long long *>(mse_h + 1); // MappingResult::ndc
        auto map_and_copy = [&]() {
            // 'unique': the mapping's colours are Lloyd's substrate, so its bounds prune the mapping sweep
            map_dev(ctx, rgb_d, P, map_col, map_cnt, nm, cen_d, k, idx_d, ib, q_d, mse_h,
                    mode == CQG_SAMPLING_UNIQUE ? &o : nullptr, mndc_h);
            copy_out(ctx, palette, cen_d, 24 * (size_t)k);
            copy_out(ctx, labels, lab_d, 4 * ns);
            copy_out(ctx, indices, idx_d, P * (size_t)ib);
            copy_out(ctx, quantized, q_d, P * 3);
            // the deferred Lloyd NDC ran on the side stream beside the mapping
            if (o.pending) CQG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->lloyd_join, 0));
            CQG_CUDA(cudaStreamSynchronize(ctx->stream)); // the pipeline's last synchronisation
        };
        map_and_copy();
        if (o.pending) {
            if (lloyd_finish(ctx, o, ns, k) != 1) {
                // an empty cluster: the synchronous loop (with repairs), then the mapping again
                o = lloyd_dev(ctx, sub_col, sub_cnt, ns, S, init_d, k, term, lab_d, cen_d, sse_h, nullptr, nullptr);
                map_and_copy();
            }
            if (sse_trace) std::memcpy(sse_trace, sse_h, 8 * (size_t)o.iterations);
        }
        const double mse = *mse_h;
        const int t_map = tm.lap();
        if (stats) {
            stats->n_unique = ns;
            stats->lloyd.iterations = o.iterations;
            stats->lloyd.repair_count = o.repairs;
            stats->lloyd.ndc_total = o.ndc;
            stats->lloyd.n_points = ns;
            stats->lloyd.flagged_total = o.flagged;
            stats->lloyd.swept_total = o.swept;
            stats->mean_sq_dist = mse;
            stats->map_ndc = *mndc_h;
            if (tm.on) CQG_CUDA(cudaEventSynchronize(tm.ev[t_map]));
            stats->ms_histogram = tm.ms(t_hist);
            stats->ms_init = tm.ms(t_init);
            stats->ms_lloyd = tm.ms(t_lloyd);
            stats->ms_map = tm.ms(t_map);
        }
    });
}

} // extern "C"

namespace cqg {
cudaError_t launch_cooperative(cqg_ctx *ctx, const void *kern, dim3 grid, dim3 block, void **args, size_t smem) {
    // Two cooperative kernels sized for the whole device could each get part
    // of the SMs and wait in their grid barriers forever, so whole-device
    // launches are chained (each waits for every earlier cooperative launch).
    // Contexts with an SM budget (cqg_set_sm_budget; budgets summing to at
    // most the device) fit side by side: they wait only for the last
    // whole-device launch.
    struct Chain {
        cudaEvent_t full = nullptr;                         // last whole-device launch
        std::map<const cqg_ctx *, cudaEvent_t> budgeted;    // last launch per budgeted context
    };
    static std::mutex mu;
    static std::map<int, Chain> chains;
    std::lock_guard<std::mutex> lock(mu);
    Chain &c = chains[ctx->device];
    const bool budget = ctx->num_sms < ctx->dev_sms;
    cudaError_t e;
    if (c.full && (e = cudaStreamWaitEvent(ctx->stream, c.full, 0)) != cudaSuccess) return e;
    if (!budget)
        for (auto &kv : c.budgeted)
            if ((e = cudaStreamWaitEvent(ctx->stream, kv.second, 0)) != cudaSuccess) return e;
    cudaEvent_t &ev = budget ? c.budgeted[ctx] : c.full;
    if (!ev && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaLaunchCooperativeKernel(kern, grid, block, args, smem, ctx->stream)) != cudaSuccess) return e;
    return cudaEventRecord(ev, ctx->stream);
}
} // namespace cqg

namespace cqg {
cudaError_t ensure_smem(const void *kern, size_t bytes) {
    // cudaFuncSetAttribute applies to the current device's context only, so
    // the cache is keyed on (device, kernel)
    int dev = 0;
    cudaError_t ge = cudaGetDevice(&dev);
    if (ge != cudaSuccess) return ge;
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, size_t> cur;
    std::lock_guard<std::mutex> lock(mu);
    size_t &c = cur[{dev, kern}];
    if (bytes <= c) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) c = bytes;
    return e;
}
} // namespace cqg
