/*
 * cqg.h -- C-ABI of the B200-native colour-quantiser hot path (libcqg.so).
 *
 * The reference (arXiv 1101.0395 artifact, /root/reference/proj) exposes its
 * hot path only as the C++ library API in proj/include/quant/*.hpp (no FFI,
 * plugin or operator registry: SURVEY.md §8(b)). Each entry point below
 * replaces one of those functions for the count-weighted ("unique" sampling)
 * path and keeps its argument meaning and error behaviour:
 *
 *   cqg_histogram      quant::build_histogram   include/quant/histogram.hpp:57
 *                                               (src/histogram.cpp:69-104)
 *   cqg_init_maximin   quant::init_maximin      include/quant/init.hpp:40
 *                                               (src/init.cpp:37-52,127-138)
 *   cqg_init_kmeanspp  quant::init_kmeanspp     include/quant/init.hpp:60
 *                                               (src/init.cpp:295-314)
 *   cqg_lloyd          quant::wsm               include/quant/kmeans.hpp:128-129
 *                                               (src/kmeans.cpp:173-277)
 *   cqg_map            quant::map_pixels        include/quant/metrics.hpp:28
 *                                               (src/metrics.cpp:15-55)
 *   cqg_coarse_histogram[_weighted]
 *                      quant::build_coarse_histogram include/quant/precluster.hpp:32-34
 *                                               (src/precluster.cpp:13-47)
 *   cqg_quantize       quant::run_quantize      include/quant/pipeline.hpp:53
 *                                               (src/pipeline.cpp:81-164), for
 *                                               methods wsm-mmx / wsm-kpp and
 *                                               caller-supplied initial centres
 *
 * Plain pointers and sizes only. Every pointer argument may be host memory
 * (pageable or pinned) or device memory of the context's device; the library
 * detects which (cudaPointerGetAttributes) and copies only what is needed.
 * All work is ordered on the context's stream; every call returns after its
 * results are visible at the output pointers.
 *
 * Errors: every function returns CQG_OK (0) or a CQG_E_* code; the message is
 * available from cqg_last_error() (thread-local). CQG_E_INVALID corresponds to
 * the reference's std::invalid_argument sites and carries the same message text
 * (e.g. "clustering: k (9) exceeds number of points (4)", kmeans.cpp:178-181);
 * CQG_E_RUNTIME corresponds to std::runtime_error (kmeans.cpp:159).
 *
 * Colours are packed 0x00RRGGBB in uint32; images are interleaved 8-bit RGB,
 * row-major, 3 bytes per pixel (quant::RawImage, image.hpp:13-24).
 * Centres / palettes are K x 3 doubles (r, g, b) as quant::ColorPoint.
 */
#ifndef CQG_H
#define CQG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CQG_OK 0
#define CQG_E_INVALID 1 /* std::invalid_argument in the reference */
#define CQG_E_RUNTIME 2 /* std::runtime_error in the reference */
#define CQG_E_CUDA 3    /* CUDA failure (no device, launch error, ...) */
#define CQG_E_NOMEM 4   /* device or pinned allocation failed */

#define CQG_INIT_MAXIMIN 0  /* "mmx" (init.cpp:127) */
#define CQG_INIT_KMEANSPP 1 /* "kpp" (init.cpp:295) */
#define CQG_INIT_GIVEN 2    /* caller supplies K initial centres */

typedef struct cqg_ctx cqg_ctx;

/* quant::Termination (kmeans.hpp:17-21) + ClusterOptions::record_history (:28-35).
 * fixed_iterations <= 0 means "not set" (std::optional empty). */
typedef struct {
    double epsilon;
    int max_iterations;
    int fixed_iterations;
    int record_history;
} cqg_term;

/* Scalar fields of quant::ClusterState (kmeans.hpp:42-56). */
typedef struct {
    int iterations;
    int repair_count;
    uint64_t ndc_total;
    uint64_t n_points;
    uint64_t flagged_total; /* points replayed in exact FP64 (diagnostic) */
    uint64_t swept_total;   /* points evaluated against every centre, summed over iterations;
                               the rest were proven to keep their label by distance bounds */
} cqg_lloyd_stats;

typedef struct {
    int init_kind; /* CQG_INIT_* */
    int k;
    uint64_t seed;
    cqg_term term;
    int index_bytes; /* 4: uint32 per pixel (MappingResult::indices layout); 1: uint8 (K <= 256) */
    int sampling;    /* CQG_SAMPLING_* (QuantizeConfig::sampling, pipeline.cpp:91-116) */
    int width, height; /* image shape, required by the 2:1 modes (subsample_2to1, histogram.cpp:60-67) */
} cqg_quantize_cfg;

/* QuantizeConfig::sampling. UNIQUE (the CLI default) clusters the distinct
 * colours with count weights; NONE / TWO_TO_ONE cluster the (sub)sampled pixels
 * themselves with weights 1/S; BOTH clusters the distinct colours of the 2:1
 * subsample. Initialisers always read the histogram of the sampled pixels, and
 * the mapping always covers the full image. */
enum { CQG_SAMPLING_UNIQUE = 0, CQG_SAMPLING_NONE = 1, CQG_SAMPLING_TWO_TO_ONE = 2, CQG_SAMPLING_BOTH = 3 };

typedef struct {
    uint64_t n_unique;   /* substrate_points (pipeline.cpp:117) */
    cqg_lloyd_stats lloyd;
    double mean_sq_dist; /* QuantReport::mse (pipeline.cpp:155) */
    uint64_t map_ndc;    /* MappingResult::ndc (metrics.cpp:36-48): distances the reference's pruned lookup evaluates */
    double ms_histogram, ms_init, ms_lloyd, ms_map; /* device time per stage (CUDA events), filled when
                                                      kernel profiling is on (cqg_set_profiling), else 0 */
} cqg_quantize_stats;

/* ---- context ------------------------------------------------------------ */
cqg_ctx *cqg_create(int device);
void cqg_destroy(cqg_ctx *ctx);
const char *cqg_last_error(void);
/* Use an existing cudaStream_t (NULL = the context's own stream). */
int cqg_set_stream(cqg_ctx *ctx, void *cuda_stream);
/* Restrict the context's grids to `sms` streaming multiprocessors (0: the
 * whole device). Contexts whose budgets sum to at most the device's SM count
 * may run their cooperative (grid-barrier) kernels concurrently, e.g. one
 * context per host thread and stream quantizing a batch of images; budgeted
 * contexts are ordered only behind whole-device cooperative launches. */
int cqg_set_sm_budget(cqg_ctx *ctx, int sms);
/* Number of library kernels launched by this context so far (bench evidence). */
uint64_t cqg_launch_count(const cqg_ctx *ctx);
const char *cqg_version(void);

/* ---- kernel-level profiling (bench evidence) -------------------------------
 * When enabled, the library brackets its hot kernels with CUDA events on the
 * launching stream and accumulates per category: device milliseconds, launch
 * count and algorithmic work units (distances for the sweeps, bytes for the
 * byte-bound kernels). */
#define CQG_PROF_SWEEP 0     /* Lloyd sweep (units: unique colours x K) */
#define CQG_PROF_MAPSWEEP 1  /* mapping sweep per distinct colour (units: N' x K) */
#define CQG_PROF_HIST 2      /* histogram stage (units: 3P + 8N' bytes) */
#define CQG_PROF_PIXEL 3     /* pixel mapping kernel (units: bytes moved) */
#define CQG_PROF_INIT 4      /* initialiser kernel (units: N' x (K-1) distance updates) */
#define CQG_PROF_REPLAY 5    /* exact FP64 replays (units: queued points) */
#define CQG_PROF_NDC 6       /* per-point distance-count (NDC) pass (units: points) */
#define CQG_PROF_LLOYD 7     /* whole Lloyd loop launches (persistent kernel / graph): units = N' x K x iterations */
#define CQG_PROF_MAPNDC 8    /* mapping distance count (MappingResult::ndc) (units: distinct colours) */
#define CQG_PROF_N 9
typedef struct {
    double ms[CQG_PROF_N];
    double units[CQG_PROF_N];
    uint64_t launches[CQG_PROF_N];
} cqg_profile;
int cqg_set_profiling(cqg_ctx *ctx, int on);
int cqg_read_profile(cqg_ctx *ctx, cqg_profile *out, int reset);
/* Kernel microbenchmark on the context's last Lloyd state: `reps` back-to-back
 * launches of the WALK-mode sweep kernel, bracketed by CUDA events on the
 * context stream. Returns the average device ms per launch and the
 * algorithmic units per launch (unique colours x K). Perturbs the context's
 * Lloyd scratch state (call after the results have been read). */
int cqg_bench_sweep(cqg_ctx *ctx, int reps, double *ms_per_launch, double *units_per_launch);

/* ---- stage 1: unique colours in first-occurrence order -------------------
 * rgb: P*3 bytes. colors/counts/first: capacity min(P, 2^24) each; `first`
 * (pixel index of first sight) may be NULL. *n_unique receives N'. Weights are
 * counts[i] * (1.0 / P) exactly as histogram.cpp:99-102. */
int cqg_histogram(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, uint32_t *colors,
                  uint32_t *counts, uint32_t *first, uint64_t *n_unique);

/* ---- initialisers (bit-exact with init.cpp for the same histogram) ------- */
int cqg_init_maximin(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n,
                     uint64_t P, int k, uint64_t seed, int weighted_first, double *centers);
int cqg_init_kmeanspp(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n,
                      uint64_t P, int k, uint64_t seed, double *centers);

/* ---- stages 2+3: weighted sort-means over the count-weighted histogram ----
 * Weights are counts[i]/P (P = source pixel count). init: k x 3. Outputs:
 * centers (k x 3), labels (n, post-repair memberships), sse_trace (capacity
 * fixed_iterations or max_iterations), stats. hist_labels (iters x n) and
 * hist_centers (iters x k x 3) are filled when term->record_history != 0 and
 * the pointers are non-NULL (ClusterState::history, pre-repair snapshots). */
int cqg_lloyd(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n,
              uint64_t P, const double *init, int k, const cqg_term *term, double *centers,
              uint32_t *labels, double *sse_trace, cqg_lloyd_stats *stats,
              uint32_t *hist_labels, double *hist_centers);

/* ---- the general Lloyd loop: real points, arbitrary weights (exact FP64) ----
 * quant::wsm for weights that are not count/P or points off the 8-bit grid
 * (kmeans.hpp:128-129), and quant::kmeans_full (kmeans.hpp:119) when weights
 * is NULL (unit weights, full scan every iteration, no repair: an empty
 * cluster keeps its centre). points: n x 3 doubles; weights: n (positive) or
 * NULL. Every output -- labels, centres, sse_trace, iterations, ndc_total,
 * repair_count, history -- is bit-identical to the reference's run_lloyd
 * (kmeans.cpp:192-260): its sequential FP64 sums are reproduced in order on
 * the device. Not a throughput path (per-iteration host round trips). */
int cqg_lloyd_exact(cqg_ctx *ctx, const double *points, const double *weights, uint64_t n, const double *init,
                    int k, const cqg_term *term, double *centers, uint32_t *labels, double *sse_trace,
                    cqg_lloyd_stats *stats, uint32_t *hist_labels, double *hist_centers);
/* API helpers of kmeans.hpp / init.hpp on the device, same arithmetic order:
 *   cqg_compute_sse            compute_sse (kmeans.hpp:99-105; weights NULL = unit overload)
 *   cqg_repair_empty_clusters  repair_empty_clusters (kmeans.hpp:112-115): centres, labels in/out
 *   cqg_center_table           build_center_distance_table (kmeans.hpp:73): k x k dist2, order
 *   cqg_kmeanspp_next_masses   kmeanspp_next_masses (init.hpp:65-66): weights x min dist2 to the
 *                              k chosen centres (k = 0: the weights)
 *   cqg_maximin_pad            maximin_pad (init.hpp:71-72): extend k0 centres to k by maximin picks */
int cqg_compute_sse(cqg_ctx *ctx, const double *points, const double *weights, uint64_t n, const double *centers,
                    int k, const uint32_t *labels, double *sse);
int cqg_repair_empty_clusters(cqg_ctx *ctx, const double *points, const double *weights, uint64_t n,
                              double *centers, int k, uint32_t *labels, int *repairs);
int cqg_center_table(cqg_ctx *ctx, const double *centers, int k, double *dist2, uint32_t *order);
int cqg_kmeanspp_next_masses(cqg_ctx *ctx, const double *colors, const double *weights, uint64_t n,
                             const double *centers, int k, double *masses);
int cqg_maximin_pad(cqg_ctx *ctx, const double *colors, uint64_t n, const double *centers, int k0, int k,
                    double *out);

/* ---- stages 2+3, sharded over ranks (one huge image) -------
 * Each rank holds a contiguous slice of the unique colours. Per iteration:
 *   cqg_shard_assign   local assignment (FULL first, then NDC + WALK sweep +
 *                      exact replay) and the rank's cumulative local moments
 *                      -> partial[5K+2] int64 = {K x (n, s_r, s_g, s_b, q),
 *                      local NDC of this iteration, local near-tie replays}
 *   (caller)           allreduce(partial, SUM) over the ranks (NCCL / gloo)
 *   cqg_shard_finalize centres / SSE / termination / walk table from the global
 *                      moments; identical on every rank. *state: 0 continue,
 *                      1 done, 2 empty cluster (run the repair protocol, then
 *                      allreduce cqg_shard_moments and finalize again).
 * partial/global may be host or device memory. P is the global pixel count. */
int cqg_shard_begin(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n_local,
                    uint64_t P, const double *init, int k, const cqg_term *term);
int cqg_shard_assign(cqg_ctx *ctx, int64_t *partial);
int cqg_shard_moments(cqg_ctx *ctx, int64_t *partial);
int cqg_shard_finalize(cqg_ctx *ctx, const int64_t *global, int *state, double *sse);
/* The same without a host round trip (global: device memory): the state is
 * logged on the device and the next cqg_shard_assign walks as if the run went
 * on. cqg_shard_status reads the log once: *state 0 = every logged iteration
 * continued, 1 = the last one finished the run, 2 = an empty cluster or an
 * early stop occurred (redo the run with cqg_shard_finalize). For fixed
 * iteration counts (BASELINE cfg5) the loop needs no per-iteration sync. */
int cqg_shard_finalize_async(cqg_ctx *ctx, const int64_t *global);
int cqg_shard_status(cqg_ctx *ctx, int *state, int *iterations);
/* repair protocol helpers (kmeans.cpp:124-169 across ranks) */
int cqg_shard_sizes(cqg_ctx *ctx, uint32_t *sizes);
int cqg_shard_donor(cqg_ctx *ctx, const uint32_t *global_sizes, int fallback, double *value,
                    uint64_t *local_index, uint32_t *colour, uint32_t *label);
int cqg_shard_move(cqg_ctx *ctx, uint64_t local_index, int e, uint32_t colour);
int cqg_shard_end(cqg_ctx *ctx, double *centers, uint32_t *labels, double *sse_trace, int *iterations);

/* ---- stage 4: exact lowest-index nearest palette entry per pixel + MSE ----
 * indices: P entries of index_bytes (4 = uint32 as MappingResult::indices,
 * 1 = uint8, requires k <= 256); may be NULL. quantized: P*3 bytes (palette
 * rendered with channel_to_u8, color.hpp:63-72); may be NULL. ndc (may be
 * NULL: not computed) receives MappingResult::ndc, the number of distances the
 * reference's hint-seeded pruned lookup evaluates (metrics.cpp:36-48,
 * kmeans.cpp:81-105). */
int cqg_map(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, const double *palette, int k,
            void *indices, int index_bytes, uint8_t *quantized, double *mean_sq_dist, uint64_t *ndc);

/* ---- coarse 32x32x32 histogram (quant::build_coarse_histogram,
 * include/quant/precluster.hpp:32-34; src/precluster.cpp:13-47): the
 * preclusterers' input (median cut / Wan / Wu, the CLI's default wsm-wu).
 * Bin (r>>3, g>>3, b>>3) in r-major order; per bin the pixel count and the
 * exact sums of r, g, b and r^2+g^2+b^2 over the ORIGINAL 8-bit values. Each
 * output array holds CQG_COARSE_BINS entries (host or device pointers). */
#define CQG_COARSE_BINS 32768
/* from an image (rgb: P x 3 bytes); "build_coarse_histogram: no pixels" */
int cqg_coarse_histogram(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, uint64_t *count, int64_t *sum_r,
                         int64_t *sum_g, int64_t *sum_b, int64_t *sum_sq);
/* from a weighted histogram (packed 0x00RRGGBB colours, counts, n entries);
 * "build_coarse_histogram: empty histogram" */
int cqg_coarse_histogram_weighted(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n,
                                  uint64_t *count, int64_t *sum_r, int64_t *sum_g, int64_t *sum_b,
                                  int64_t *sum_sq);

/* ---- whole hot path: histogram -> init -> wsm -> map --------------------
 * init: required for CQG_INIT_GIVEN (k x 3), ignored otherwise. palette: k x 3.
 * labels (capacity: the substrate -- min(P,2^24) colours, or P pixels for NONE),
 * sse_trace, indices, quantized may be NULL. stats->n_unique is the substrate size. */
int cqg_quantize(cqg_ctx *ctx, const uint8_t *rgb, uint64_t P, const cqg_quantize_cfg *cfg,
                 const double *init, double *palette, uint32_t *labels, double *sse_trace,
                 void *indices, uint8_t *quantized, cqg_quantize_stats *stats);

#ifdef __cplusplus
}
#endif

#endif /* CQG_H */
