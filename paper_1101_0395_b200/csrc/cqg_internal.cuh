// cqg_internal.cuh -- shared context, buffers, error plumbing and exact-FP64
// device helpers for libcqg.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "cqg.h"

namespace cqg {

// ---------------------------------------------------------------------------
// errors: thrown inside the library, converted to CQG_E_* at the C boundary

struct Error {
    int code;
    std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string &msg) { throw Error{code, msg}; }

#define CQG_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess)                                                            \
            ::cqg::fail(CQG_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// ---------------------------------------------------------------------------
// grow-only device buffers owned by a context

struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    void *ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes < 256 ? 256 : bytes;
        if (cudaMalloc(&p, want) != cudaSuccess) {
            cudaGetLastError();
            fail(CQG_E_NOMEM, "device allocation of " + std::to_string(want) + " bytes failed");
        }
        cap = want;
        return p;
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct HostBuf {
    void *p = nullptr;
    size_t cap = 0;
    void *ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t want = bytes < 256 ? 256 : bytes;
        if (cudaMallocHost(&p, want) != cudaSuccess) {
            cudaGetLastError();
            fail(CQG_E_NOMEM, "pinned allocation failed");
        }
        cap = want;
        return p;
    }
    template <class T>
    T *as() const { return static_cast<T *>(p); }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
};

// Per-iteration device status written by the finalize kernel and read back by
// the host loop (one small D2H per Lloyd iteration).
struct IterStatus {
    int32_t state;      // 0 continue, 1 done, 2 empty cluster -> repair needed
    int32_t iteration;
    uint32_t n_flagged; // FP64 replays this iteration
    uint32_t pad;
    double sse;
};

// Moments of one cluster over the count-weighted substrate: n = sum count,
// s = sum count*x (per channel), q = sum count*|x|^2. Exact integers.
struct Moments {
    unsigned long long n;
    long long s[3];
    unsigned long long q;
};

} // namespace cqg

struct cqg_ctx {
    int device = 0;
    int num_sms = 148;     // grid sizing: the device's SMs, or the cqg_set_sm_budget slice
    int dev_sms = 148;     // the device's SMs (size limits of the persistent kernel)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t aux = nullptr;            // side stream for independent work (mapping NDC)
    cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
    cudaStream_t aux2 = nullptr;           // second side stream: the persistent Lloyd loop's NDC pass
    cudaEvent_t lloyd_fork = nullptr, lloyd_join = nullptr; // ... forked after the loop, done
    cudaEvent_t walk_fork = nullptr, walk_join = nullptr;   // large WALK iterations: NDC beside the stay-test pass
    cudaEvent_t stage_ev[8] = {}; // cqg_quantize stage timing (created once per context)
    unsigned long long launches = 0;

    // stage 1 scratch
    cqg::DevBuf tab;       // 2^24 x uint2 {count, ~first_index}; kept all-zero between calls
    cqg::DevBuf list;      // unique colours in arrival order
    cqg::DevBuf bitmap;    // P bits: first-occurrence marks
    cqg::DevBuf wordpref;  // per-bitmap-block exclusive prefix
    cqg::DevBuf scal;      // small device scalars (counters)
    cqg::DevBuf pcnt, pent, pseg; // large images: per-colour counts (2^24), bucketed pixel entries, bucket offsets
    // input / substrate staging
    cqg::DevBuf img;       // image bytes when the caller passes host memory
    cqg::DevBuf colors, counts, first;
    // Lloyd state
    cqg::DevBuf labels, cen, fcen, dtab, dsorted, order, mom, queue, ndc, status, sizes, red;
    cqg::DevBuf hist_labels, hist_centers, sse;
    cqg::DevBuf bnd, shift, dcode;
    cqg::DevBuf rowmin, snap_cen, snap_lab, ndc_keys, dmom;
    cqg::DevBuf survivors; // WALK survivor list of filter_list_kernel (+ its counter) // persistent Lloyd: stay-test row minima, deferred-NDC snapshots
    cqg::DevBuf sub_img, raw_col, raw_cnt, full_col, full_cnt; // sampling modes     // distance-bound pruning: per-point (ub, lb), centre moves
    cqg::DevBuf mom_g, partial, shard_log; // sharded Lloyd: global moments, packed partials, state log
    void *shard = nullptr;      // cqg::ShardState (lloyd.cu)
    // mapping
    cqg::DevBuf lut, idx_out, q_out, mom_map, map_rows, map_lab;
    cqg::DevBuf coarse; // 5 x 32768 u64 coarse histogram (cqg_coarse_histogram)
    // init
    cqg::DevBuf mind2, initpart, initsel, unit_draws, inittile;
    cqg::HostBuf pinned;   // status readback and small results
    cqg::HostBuf pinned_nu; // initialiser unit draws (an async H2D source: no host-blocking copy)
    // pageable caller memory is reached through pinned staging buffers (copy_out / stage_in): one
    // grow-only buffer per transfer of a call, in call order, so a repeated call reuses them
    std::vector<cqg::HostBuf> stage_out, stage_in;
    size_t stage_out_used = 0, stage_in_used = 0;

    // cached CUDA graph of the Lloyd WHILE loop (lloyd.cu)
    bool use_graphs = true;
    bool use_cluster_init = true;
    int dbg_init_force_seq = 0; // tests only: CQG_DBG_INIT_FORCE_SEQ=1|2 drives the register cluster kernel's sequential paths
    int dbg_ndc_win = 0; // tests only: CQG_DBG_NDC_WIN=n caps the persistent loop's deferred-NDC window (relaunches)
    int cluster_nt = 0; // cluster init CTA size: 0 fewest padded slots, else forced (CQG_CLUSTER_NT=512..1024)
    bool use_init_tile = true; // colour-space tiles with box pruning for large-N init (CQG_NO_INIT_TILE=1: off)
    uint64_t init_tile_min = 1ull << 20; // ... from this many points (CQG_INIT_TILE_MIN; below, the record layout is as fast)
    bool use_ndc_code = true; // shared-memory code table for the NDC count (CQG_NO_NDC_CODE=1: off)
    bool use_prune = true; // distance-bound pruning of the WALK sweep (CQG_NO_PRUNE=1: off)
    bool use_filter_list = true; // large substrates: stay-test pass + survivor-list sweep (CQG_NO_FILTER_LIST=1: off)
    bool lloyd_prune_pending = false; // the deferred Lloyd run pruned (lloyd_finish)
    cudaGraphExec_t loop_exec = nullptr;
    cudaGraph_t loop_graph = nullptr;
    std::vector<uint64_t> loop_key;
    // kernel-level profiling (cqg_set_profiling)
    bool prof_on = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct ProfRec {
        int cat;
        int e0, e1;
        double units;
    };
    std::vector<ProfRec> prof_recs;
    double prof_ms[CQG_PROF_N] = {};
    // last Lloyd sweep launch (for cqg_bench_sweep)
    unsigned char last_sweep[512] = {};
    bool have_last_sweep = false;
    double prof_units[CQG_PROF_N] = {};
    unsigned long long prof_launches[CQG_PROF_N] = {};
};

namespace cqg {

// ---------------------------------------------------------------------------
// exact FP64 helpers: no FMA contraction, so results equal the reference's
// dist2 (color.hpp:47-59: ((dr*dr)+(dg*dg))+(db*db)) bit for bit.

__device__ __forceinline__ double d2_exact(double xr, double xg, double xb, double cr, double cg,
                                           double cb) {
    const double dr = __dsub_rn(xr, cr), dg = __dsub_rn(xg, cg), db = __dsub_rn(xb, cb);
    return __dadd_rn(__dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dg, dg)), __dmul_rn(db, db));
}

// correctly rounded unsigned 128-bit -> double (same contract as the oracle)
__device__ __forceinline__ double u128_to_double(unsigned __int128 x) {
    const unsigned long long hi = (unsigned long long)(x >> 64);
    if (hi == 0) return __ull2double_rn((unsigned long long)x);
    const int s = 64 - __clzll((long long)hi);
    unsigned long long v = (unsigned long long)(x >> s);
    const unsigned __int128 lostmask = (((unsigned __int128)1) << s) - 1;
    if ((x & lostmask) != 0) v |= 1ULL;
    return __dmul_rn(__ull2double_rn(v), __longlong_as_double((long long)(1023 + s) << 52)); // exact: x 2^s
}

// (n*Q - |S|^2) / n for one cluster, exact numerator (cluster_sse_exact in the oracle)
__device__ __forceinline__ double cluster_sse_exact(unsigned long long n, const long long *s,
                                                    unsigned long long q) {
    const unsigned __int128 nq = (unsigned __int128)n * q;
    const unsigned __int128 ss = (unsigned __int128)((__int128)s[0] * s[0]) +
                                 (unsigned __int128)((__int128)s[1] * s[1]) +
                                 (unsigned __int128)((__int128)s[2] * s[2]);
    return __ddiv_rn(u128_to_double(nq - ss), __ull2double_rn(n));
}

// Programmatic dependent launch: a kernel launched with launch_pdl starts
// while the previous kernel on the stream drains and waits here for its
// results (a no-op without the launch attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the next kernel on the stream launch now (its blocks wait in pdl_wait
// until this grid has completed and its memory is visible)
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CQG_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

__host__ __device__ __forceinline__ unsigned ceil_div(unsigned long long a, unsigned long long b) {
    return (unsigned)((a + b - 1) / b);
}

// host-side helpers implemented in api.cu
bool is_device_ptr(const void *p);
// profiling: prof_begin records a start event (returns -1 when profiling is off)
int prof_begin(cqg_ctx *ctx);
int prof_end(cqg_ctx *ctx, int cat, int begin, double units); // returns the record index (or -1)
void prof_add_units(cqg_ctx *ctx, int rec, double units);
void launched(cqg_ctx *ctx, int n = 1);
void release_graphs(cqg_ctx *ctx);
// copy `bytes` from user pointer (host or device) into a device buffer and
// return a device pointer that holds the data (the user pointer itself when
// it is already device memory).
const void *stage_in(cqg_ctx *ctx, const void *user, size_t bytes, DevBuf &buf);
void copy_out(cqg_ctx *ctx, void *user, const void *dev, size_t bytes);

// stage implementations (device pointers only; n_dev is a device scalar)
void histogram_dev(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t P, uint32_t *colors_d,
                   uint32_t *counts_d, uint32_t *first_d, uint32_t *n_dev);
uint64_t read_scalar_u32(cqg_ctx *ctx, const uint32_t *dev);

struct LloydOut {
    int iterations = 0;
    int repairs = 0;
    unsigned long long ndc = 0;
    unsigned long long flagged = 0;
    unsigned long long swept = 0; // points through the full centre loop, all iterations
    // final state for a bound-pruned mapping of the same substrate (bnd null: none)
    const uint32_t *labels = nullptr;
    float2 *bnd = nullptr;
    const float *shift = nullptr;
    const double *dsorted = nullptr;
    const uint16_t *dcode = nullptr; // 16-bit codes of dsorted (K <= 256), or null
    const double *rowmin = nullptr;  // nearest-other-centre distances (when dsorted is null)
    const Moments *mom = nullptr;
    int Kpow = 0;
    // deferred completion (lloyd_dev(..., allow_defer)): the persistent kernel
    // and its status read-back are enqueued, nothing synchronised yet; after
    // the caller's own synchronisation lloyd_finish() fills the counters
    bool pending = false;
    int prof_rec = -1;
};
// Raise (never lower) a kernel's dynamic shared-memory limit. The attribute is
// per function and process-wide: contexts on several host threads launching
// the same kernel with different K must not undo each other's setting.
cudaError_t ensure_smem(const void *kern, size_t bytes);

// Cooperative launches from several contexts/streams of one process are
// chained through one event per device: two partially resident grids that
// each wait in grid.sync() for the other's SMs would deadlock.
cudaError_t launch_cooperative(cqg_ctx *ctx, const void *kern, dim3 grid, dim3 block, void **args, size_t smem);

// After a deferred lloyd_dev and a stream synchronisation: iterations, NDC,
// counters from the pinned read-back; returns the final state (1 done, 2 an
// empty cluster: the caller reruns lloyd_dev without deferral, which repairs).
int lloyd_finish(cqg_ctx *ctx, LloydOut &out, uint64_t n, int K);
LloydOut lloyd_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n,
                   uint64_t P, const double *init_d, int k, const cqg_term &term, uint32_t *labels_d,
                   double *centers_d, double *sse_host, uint32_t *hist_labels_user,
                   double *hist_centers_user, bool allow_defer = false);

void bench_sweep_dev(cqg_ctx *ctx, int reps, double *ms, double *units);

// exact.cu: the reference's Lloyd loop for arbitrary real points and weights
// (w_d null = unit weights), bit-identical to run_lloyd; device pointers
struct ExactOut {
    int iterations = 0;
    int repairs = 0;
    unsigned long long ndc = 0;
};
ExactOut exact_lloyd_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, const double *init_d,
                         int K, const cqg_term &term, bool prune_repair, uint32_t *lab_d, double *cen_d,
                         double *sse_host, uint32_t *hist_labels_user, double *hist_centers_user);
void exact_table_dev(cqg_ctx *ctx, const double *cen_d, int K, double *dist_d, uint32_t *order_d);
double exact_sse_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, const double *cen_d,
                     const uint32_t *lab_d, double *scratch_d);
int exact_repair_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, double *cen_d, int K,
                     uint32_t *lab_d);
void exact_next_masses_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, const double *cen_d,
                           int k0, double *mass_d);
void exact_maximin_pad_dev(cqg_ctx *ctx, const double *pts_d, uint64_t n, double *cen_d, int k0, int k);
// sharded Lloyd (lloyd.cu); device pointers unless noted
void shard_begin_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n, uint64_t P,
                     const double *init_d, int K, const cqg_term &term);
void shard_assign_dev(cqg_ctx *ctx, long long *partial_d, bool run);
int shard_finalize_dev(cqg_ctx *ctx, const long long *global_d, double *sse);
void shard_finalize_async_dev(cqg_ctx *ctx, const long long *global_d);
int shard_status_dev(cqg_ctx *ctx, int *iterations);
void shard_sizes_dev(cqg_ctx *ctx, uint32_t *sizes_d);
void shard_donor_dev(cqg_ctx *ctx, const uint32_t *gsizes_d, int fallback, double *value, uint64_t *index,
                     uint32_t *colour, uint32_t *label);
void shard_move_dev(cqg_ctx *ctx, uint64_t index, int e, uint32_t colour);
int shard_end_dev(cqg_ctx *ctx, double *centers_user, uint32_t *labels_user, double *sse_user);
void shard_release(cqg_ctx *ctx);
int shard_k(cqg_ctx *ctx);
uint64_t shard_n(cqg_ctx *ctx);
void subsample_2to1_dev(cqg_ctx *ctx, const uint8_t *rgb_d, int w, int h, uint8_t *out_d);
void pack_pixels_dev(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t S, uint32_t *colors_d, uint32_t *counts_d);
// lloyd: the run that produced pal_d on this same substrate (colors_d, counts_d),
// or null; with its distance bounds the mapping sweep only re-examines the
// points whose label can change (MODE_MAPW).
void coarse_hist_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n,
                     unsigned long long *tab_d);
double map_dev(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t P, const uint32_t *colors_d,
               const uint32_t *counts_d, uint64_t n, const double *pal_d, int k, void *indices_d,
               int index_bytes, uint8_t *quant_d,
               double *mse_async = nullptr, const LloydOut *lloyd = nullptr,
               unsigned long long *ndc_async = nullptr); // MappingResult::ndc (pinned host), null: skip

void init_maximin_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n,
                      uint64_t P, int k, uint64_t seed, int weighted_first, double *centers_d);
void init_kmeanspp_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d,
                       uint64_t n, uint64_t P, int k, uint64_t seed, double *centers_d);

} // namespace cqg
