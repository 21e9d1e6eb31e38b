// lloyd.cu -- stages 2+3: weighted sort-means on the device.
//
// Replaces quant::wsm / run_lloyd (reference src/kmeans.cpp:173-277) for
// count-weighted substrates. Per iteration (all on the context stream):
//   sweep<FULL|WALK>   FP32 argmin + near-tie queue + NDC + moment deltas
//   replay<FULL|WALK>  exact FP64 reference assignment for queued points
//   finalize           centres = S/n (FP64), SSE from int128 moments,
//                      termination test (kmeans.cpp:249-257) -> IterStatus
//   fc / table         FP32 centre table + bound, K x K walk table
// The host reads one 24-byte IterStatus per iteration. Empty clusters (rare)
// are repaired by a host-driven loop of device kernels that reproduces
// repair_empty_clusters (kmeans.cpp:124-169) exactly.
#include <algorithm>
#include <cstring>

#include "sweep.cuh"

namespace cqg {

// ---------------------------------------------------------------------------
__global__ void fc_kernel(const double *cen, int K, int Kp, float *fc, float *tau) {
    __shared__ float s_max[32];
    __shared__ int s_neg[32];
    float cm = 0.f;
    int neg = 0;
    for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
        if (k < K) {
            const double r = cen[3 * k], g = cen[3 * k + 1], b = cen[3 * k + 2];
            fc[k] = __double2float_rn(__dmul_rn(-2.0, r));
            fc[Kp + k] = __double2float_rn(__dmul_rn(-2.0, g));
            fc[2 * Kp + k] = __double2float_rn(__dmul_rn(-2.0, b));
            fc[3 * Kp + k] = __double2float_rn(
                __dadd_rn(__dadd_rn(__dmul_rn(r, r), __dmul_rn(g, g)), __dmul_rn(b, b)));
            cm = fmaxf(cm, __double2float_ru(fmax(fabs(r), fmax(fabs(g), fabs(b)))));
            neg |= (r < 0.0) | (g < 0.0) | (b < 0.0);
        } else {
            fc[k] = 0.f;
            fc[Kp + k] = 0.f;
            fc[2 * Kp + k] = 0.f;
            fc[3 * Kp + k] = 1.0e30f;
        }
    }
    for (int o = 16; o; o >>= 1) {
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        neg |= __shfl_xor_sync(0xffffffffu, neg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_max[threadIdx.x >> 5] = cm;
        s_neg[threadIdx.x >> 5] = neg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double C = 0.0;
        int anyneg = 0;
        for (int i = 0; i < (int)((blockDim.x + 31) / 32); ++i) {
            C = fmax(C, (double)s_max[i]);
            anyneg |= s_neg[i];
        }
        const double u = 0x1.0p-24, X = 255.0;
        const double cc_err = u * 3.0 * C * C;
        const double m2c_err = u * 2.0 * X * 3.0 * C;
        // all partial sums lie in [0, cc + xx] when x, c >= 0; otherwise a
        // looser magnitude bound applies
        const double M = anyneg ? 3.0 * C * C + 3.0 * X * X + 6.0 * X * C : 3.0 * C * C + 3.0 * X * X;
        const double E = cc_err + m2c_err + 4.0 * u * M;
        tau[0] = (float)(2.0 * E * 1.0625 + 1.0e-3);
        tau[1] = 0x1.0p-14f; // covers the 8 truncated mantissa bits of both keys
    }
}

__global__ void table_kernel(const double *cen, int K, double *dtab, double *dsorted, uint32_t *order) {
    extern __shared__ double s_d[]; // K doubles + K ints
    int *s_rank = reinterpret_cast<int *>(s_d + K);
    const int i = blockIdx.x;
    const double cr = cen[3 * i], cg = cen[3 * i + 1], cb = cen[3 * i + 2];
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        const double d = d2_exact(cr, cg, cb, cen[3 * j], cen[3 * j + 1], cen[3 * j + 2]);
        s_d[j] = d;
        dtab[(size_t)i * K + j] = d;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        const double d = s_d[j];
        int rank = 0;
        for (int t = 0; t < K; ++t) {
            const double e = s_d[t];
            rank += (e < d) || (e == d && t < j);
        }
        s_rank[j] = rank;
    }
    __syncthreads();
    const int rself = s_rank[i];
    for (int j = threadIdx.x; j < K; j += blockDim.x) {
        const int rk = s_rank[j];
        const int pos = (j == i) ? 0 : (rk < rself ? rk + 1 : rk);
        order[(size_t)i * K + pos] = (uint32_t)j;
        dsorted[(size_t)i * K + pos] = s_d[j];
    }
}

namespace {

// Centres from moments, SSE, termination. One block.
__global__ void finalize_kernel(Moments *mom, double *cen, int K, uint64_t P, int iter, double eps,
                                int limit, int fixed, double *sse_arr, IterStatus *st,
                                const uint32_t *qn, unsigned long long *ndc, uint64_t n_points) {
    extern __shared__ double s_a[];
    __shared__ int s_empty;
    if (threadIdx.x == 0) s_empty = 0;
    __syncthreads();
    int empty = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) empty |= (mom[k].n == 0);
    if (empty) atomicOr(&s_empty, 1);
    __syncthreads();
    if (s_empty) {
        if (threadIdx.x == 0) {
            st->state = 2;
            st->iteration = iter;
            st->n_flagged = *qn;
        }
        return;
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const Moments m = mom[k];
        const double nd = __ull2double_rn(m.n);
        cen[3 * k] = __ddiv_rn(__ll2double_rn(m.s[0]), nd);
        cen[3 * k + 1] = __ddiv_rn(__ll2double_rn(m.s[1]), nd);
        cen[3 * k + 2] = __ddiv_rn(__ll2double_rn(m.s[2]), nd);
        s_a[k] = cluster_sse_exact(m.n, m.s, m.q);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int k = 0; k < K; ++k) tot = __dadd_rn(tot, s_a[k]);
        const double sse = __ddiv_rn(tot, __ull2double_rn(P));
        sse_arr[iter - 1] = sse;
        int done;
        if (fixed > 0) {
            done = iter >= limit;
        } else {
            done = (sse == 0.0);
            if (!done && iter >= 2) {
                const double prev = sse_arr[iter - 2];
                done = __ddiv_rn(__dsub_rn(prev, sse), sse) <= eps;
            }
            if (!done && iter >= limit) done = 1;
        }
        if (iter == 1) *ndc += (unsigned long long)n_points * (unsigned long long)K;
        st->state = done ? 1 : 0;
        st->iteration = iter;
        st->n_flagged = *qn;
        st->sse = sse;
    }
}

// ---- repair helpers (kmeans.cpp:124-169) ----------------------------------

__global__ void sizes_kernel(const uint32_t *labels, uint64_t n, uint32_t *sizes) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&sizes[labels[i]], 1u);
}

struct ValIdx {
    double v;
    unsigned long long i;
};

__device__ __forceinline__ ValIdx better(ValIdx a, ValIdx b) {
    // larger value wins; equal values -> lower index (strict > scan from 0)
    if (a.v > b.v) return a;
    if (b.v > a.v) return b;
    return a.i <= b.i ? a : b;
}

// donor candidates: weights[i] * dist2(points[i], centers[m[i]]) with
// weights = count * (1/P) (histogram.cpp:99-102); or, when fallback != 0, the
// lowest index whose cluster has >= 2 points (value 1, others -1).
__global__ void argmax_kernel(const uint32_t *colors, const uint32_t *counts, const uint32_t *labels,
                              uint64_t n, const double *cen, double inv, const uint32_t *sizes,
                              int fallback, ValIdx *part) {
    ValIdx best{-2.0, ~0ull};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = labels[i];
        double v;
        if (fallback) {
            v = sizes[m] >= 2 ? 1.0 : -1.0;
        } else {
            const uint32_t c = colors[i];
            const double w = __dmul_rn((double)counts[i], inv);
            v = __dmul_rn(w, d2_exact((double)((c >> 16) & 255u), (double)((c >> 8) & 255u),
                                      (double)(c & 255u), cen[3 * m], cen[3 * m + 1], cen[3 * m + 2]));
        }
        best = better(best, ValIdx{v, i});
    }
    __shared__ ValIdx s[256];
    s[threadIdx.x] = best;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if ((int)threadIdx.x < o) s[threadIdx.x] = better(s[threadIdx.x], s[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void argmax_final(ValIdx *part, int nparts) {
    if (threadIdx.x == 0) {
        ValIdx b = part[0];
        for (int i = 1; i < nparts; ++i) b = better(b, part[i]);
        part[0] = b;
    }
}

// move point `donor` into empty cluster e: labels, centre, moments, sizes
__global__ void apply_move_kernel(const uint32_t *colors, const uint32_t *counts, uint32_t *labels,
                                  double *cen, Moments *mom, uint32_t *sizes, uint64_t donor, int e) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const uint32_t old = labels[donor];
    const uint32_t c = colors[donor], cnt = counts[donor];
    const uint32_t r = (c >> 16) & 255u, g = (c >> 8) & 255u, b = c & 255u;
    const long long sc = (long long)cnt;
    const long long qq = (long long)(r * r + g * g + b * b);
    mom[old].n -= (unsigned long long)sc;
    mom[old].s[0] -= sc * r;
    mom[old].s[1] -= sc * g;
    mom[old].s[2] -= sc * b;
    mom[old].q -= (unsigned long long)(sc * qq);
    mom[e].n += (unsigned long long)sc;
    mom[e].s[0] += sc * r;
    mom[e].s[1] += sc * g;
    mom[e].s[2] += sc * b;
    mom[e].q += (unsigned long long)(sc * qq);
    labels[donor] = (uint32_t)e;
    cen[3 * e] = (double)r;
    cen[3 * e + 1] = (double)g;
    cen[3 * e + 2] = (double)b;
    sizes[old] -= 1;
    sizes[e] += 1;
}

int pick_grid(cqg_ctx *ctx, uint64_t work, int per_block, int per_sm) {
    uint64_t g = (work + per_block - 1) / per_block;
    const uint64_t gmax = (uint64_t)ctx->num_sms * per_sm;
    if (g > gmax) g = gmax;
    if (g < 1) g = 1;
    return (int)g;
}

} // namespace

size_t sweep_smem_bytes(int K, int Kp) {
    return (size_t)4 * Kp * sizeof(float) + (size_t)K * kAccPerCluster * sizeof(uint32_t);
}

template <int MODE>
static void launch_sweep_mode(cqg_ctx *ctx, const SweepArgs &a) {
    const size_t smem = sweep_smem_bytes(a.K, a.Kp);
    const uint64_t n = a.n;
    const int pb = prof_begin(ctx);
    if (a.K > 256) {
        auto kern = sweep_wide_kernel<MODE>;
        CQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int grid = pick_grid(ctx, n, kSweepThreads, 4);
        kern<<<grid, kSweepThreads, smem, ctx->stream>>>(a);
    } else {
        // choose points-per-thread so the grid still covers every SM twice
        const uint64_t per_sm2 = (uint64_t)ctx->num_sms * 2;
        if (n >= per_sm2 * kSweepThreads * 8) {
            auto kern = sweep_kernel<MODE, 8>;
            CQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kern<<<pick_grid(ctx, n, kSweepThreads * 8, 4), kSweepThreads, smem, ctx->stream>>>(a);
        } else if (n >= per_sm2 * kSweepThreads * 4) {
            auto kern = sweep_kernel<MODE, 4>;
            CQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kern<<<pick_grid(ctx, n, kSweepThreads * 4, 4), kSweepThreads, smem, ctx->stream>>>(a);
        } else if (n >= per_sm2 * kSweepThreads * 2) {
            auto kern = sweep_kernel<MODE, 2>;
            CQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kern<<<pick_grid(ctx, n, kSweepThreads * 2, 4), kSweepThreads, smem, ctx->stream>>>(a);
        } else {
            auto kern = sweep_kernel<MODE, 1>;
            CQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            kern<<<pick_grid(ctx, n, kSweepThreads, 4), kSweepThreads, smem, ctx->stream>>>(a);
        }
    }
    prof_end(ctx, MODE == MODE_MAP ? CQG_PROF_MAPSWEEP : CQG_PROF_SWEEP, pb, (double)n * (double)a.K);
    const int pr = prof_begin(ctx);
    replay_kernel<MODE><<<pick_grid(ctx, n / 64 + 1, 128, 2), 128, 0, ctx->stream>>>(a);
    prof_end(ctx, CQG_PROF_REPLAY, pr, 0.0);
    CQG_CUDA(cudaGetLastError());
    launched(ctx, 2);
}

void launch_sweep(cqg_ctx *ctx, int mode, const SweepArgs &a) {
    if (mode == MODE_FULL) launch_sweep_mode<MODE_FULL>(ctx, a);
    else if (mode == MODE_WALK) launch_sweep_mode<MODE_WALK>(ctx, a);
    else launch_sweep_mode<MODE_MAP>(ctx, a);
}

// ---------------------------------------------------------------------------

static int repair_loop(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n,
                       uint64_t P, int K, uint32_t *labels, double *cen, Moments *mom) {
    cudaStream_t s = ctx->stream;
    uint32_t *sizes = static_cast<uint32_t *>(ctx->sizes.ensure((size_t)K * 4));
    const int nparts = pick_grid(ctx, n, 256, 2);
    ValIdx *part = static_cast<ValIdx *>(ctx->red.ensure(sizeof(ValIdx) * (size_t)nparts));
    CQG_CUDA(cudaMemsetAsync(sizes, 0, (size_t)K * 4, s));
    sizes_kernel<<<nparts, 256, 0, s>>>(labels, n, sizes);
    launched(ctx);
    std::vector<uint32_t> hsz(K);
    CQG_CUDA(cudaMemcpyAsync(hsz.data(), sizes, (size_t)K * 4, cudaMemcpyDeviceToHost, s));
    CQG_CUDA(cudaStreamSynchronize(s));
    const double inv = 1.0 / static_cast<double>(P);
    int repairs = 0;
    ValIdx *hres = static_cast<ValIdx *>(ctx->pinned.ensure(4096));
    for (;;) {
        int e = -1;
        for (int k = 0; k < K; ++k)
            if (hsz[k] == 0) {
                e = k;
                break;
            }
        if (e < 0) break;
        argmax_kernel<<<nparts, 256, 0, s>>>(colors, counts, labels, n, cen, inv, sizes, 0, part);
        argmax_final<<<1, 32, 0, s>>>(part, nparts);
        launched(ctx, 2);
        CQG_CUDA(cudaMemcpyAsync(hres, part, sizeof(ValIdx), cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaStreamSynchronize(s));
        ValIdx best = *hres;
        if (!(best.v > 0.0)) {
            argmax_kernel<<<nparts, 256, 0, s>>>(colors, counts, labels, n, cen, inv, sizes, 1, part);
            argmax_final<<<1, 32, 0, s>>>(part, nparts);
            launched(ctx, 2);
            CQG_CUDA(cudaMemcpyAsync(hres, part, sizeof(ValIdx), cudaMemcpyDeviceToHost, s));
            CQG_CUDA(cudaStreamSynchronize(s));
            best = *hres;
            if (!(best.v > 0.0)) fail(CQG_E_RUNTIME, "repair_empty_clusters: more clusters than points");
        }
        uint32_t old = 0;
        CQG_CUDA(cudaMemcpyAsync(&hres[1], labels + best.i, 4, cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaStreamSynchronize(s));
        std::memcpy(&old, &hres[1], 4);
        apply_move_kernel<<<1, 32, 0, s>>>(colors, counts, labels, cen, mom, sizes, best.i, e);
        launched(ctx);
        hsz[old] -= 1;
        hsz[e] += 1;
        ++repairs;
    }
    return repairs;
}

LloydOut lloyd_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n,
                   uint64_t P, const double *init_d, int K, const cqg_term &term, uint32_t *labels_d,
                   double *centers_d, double *sse_host, uint32_t *hist_labels_user,
                   double *hist_centers_user) {
    cudaStream_t s = ctx->stream;
    const int Kp = (K + 3) & ~3;
    const int limit = term.fixed_iterations > 0 ? term.fixed_iterations : term.max_iterations;
    double *cen = centers_d;
    CQG_CUDA(cudaMemcpyAsync(cen, init_d, sizeof(double) * 3 * K, cudaMemcpyDeviceToDevice, s));
    float *fc = static_cast<float *>(ctx->fcen.ensure(sizeof(float) * (4 * (size_t)Kp + 8)));
    float *tau = fc + 4 * Kp;
    double *dtab = static_cast<double *>(ctx->dtab.ensure(sizeof(double) * (size_t)K * K));
    double *dsorted = static_cast<double *>(ctx->dsorted.ensure(sizeof(double) * (size_t)K * K));
    uint32_t *order = static_cast<uint32_t *>(ctx->order.ensure(sizeof(uint32_t) * (size_t)K * K));
    Moments *mom = static_cast<Moments *>(ctx->mom.ensure(sizeof(Moments) * (size_t)K));
    uint32_t *queue = static_cast<uint32_t *>(ctx->queue.ensure(sizeof(uint32_t) * (n + 1)));
    uint32_t *qn = static_cast<uint32_t *>(ctx->scal.ensure(256));
    unsigned long long *ndc = reinterpret_cast<unsigned long long *>(qn + 8);
    IterStatus *st = reinterpret_cast<IterStatus *>(qn + 16);
    double *sse_d = static_cast<double *>(ctx->sse.ensure(sizeof(double) * (size_t)(limit + 1)));
    IterStatus *hst = static_cast<IterStatus *>(ctx->pinned.ensure(4096));
    const bool hist = term.record_history && (hist_labels_user || hist_centers_user);
    uint32_t *hl_d = nullptr;
    double *hc_d = nullptr;
    if (hist) {
        hl_d = static_cast<uint32_t *>(ctx->hist_labels.ensure(sizeof(uint32_t) * n * (size_t)limit));
        hc_d = static_cast<double *>(ctx->hist_centers.ensure(sizeof(double) * 3 * (size_t)K * limit));
    }

    CQG_CUDA(cudaMemsetAsync(mom, 0, sizeof(Moments) * (size_t)K, s));
    CQG_CUDA(cudaMemsetAsync(ndc, 0, 8, s));
    fc_kernel<<<1, 256, 0, s>>>(cen, K, Kp, fc, tau);
    launched(ctx);

    SweepArgs a{};
    a.colors = colors_d;
    a.counts = counts_d;
    a.n = n;
    a.labels = labels_d;
    a.fc = fc;
    a.cen = cen;
    a.dtab = dtab;
    a.dsorted = dsorted;
    a.order = order;
    a.tau = tau;
    a.queue = queue;
    a.qn = qn;
    a.mom = mom;
    a.ndc = ndc;
    a.K = K;
    a.Kp = Kp;

    LloydOut out;
    const int fin_threads = K >= 1024 ? 1024 : ((K + 31) / 32) * 32;
    const size_t table_smem = (size_t)K * (sizeof(double) + sizeof(int));
    if (table_smem > 48 * 1024)
        CQG_CUDA(cudaFuncSetAttribute(table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)table_smem));
    if ((size_t)K * 8 > 48 * 1024)
        CQG_CUDA(cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, K * 8));
    int iter = 1;
    for (;; ++iter) {
        CQG_CUDA(cudaMemsetAsync(qn, 0, 4, s));
        launch_sweep(ctx, iter == 1 ? MODE_FULL : MODE_WALK, a);
        if (hist) {
            if (hist_labels_user)
                CQG_CUDA(cudaMemcpyAsync(hl_d + (size_t)(iter - 1) * n, labels_d, 4 * n,
                                         cudaMemcpyDeviceToDevice, s));
            if (hist_centers_user)
                CQG_CUDA(cudaMemcpyAsync(hc_d + (size_t)(iter - 1) * 3 * K, cen, 24 * (size_t)K,
                                         cudaMemcpyDeviceToDevice, s));
        }
        finalize_kernel<<<1, fin_threads, (size_t)K * 8, s>>>(mom, cen, K, P, iter, term.epsilon, limit,
                                                              term.fixed_iterations, sse_d, st, qn, ndc, n);
        launched(ctx);
        CQG_CUDA(cudaMemcpyAsync(hst, st, sizeof(IterStatus), cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaStreamSynchronize(s));
        out.flagged += hst->n_flagged;
        if (hst->state == 2) {
            out.repairs += repair_loop(ctx, colors_d, counts_d, n, P, K, labels_d, cen, mom);
            finalize_kernel<<<1, fin_threads, (size_t)K * 8, s>>>(mom, cen, K, P, iter, term.epsilon, limit,
                                                                  term.fixed_iterations, sse_d, st, qn, ndc, n);
            launched(ctx);
            CQG_CUDA(cudaMemcpyAsync(hst, st, sizeof(IterStatus), cudaMemcpyDeviceToHost, s));
            CQG_CUDA(cudaStreamSynchronize(s));
            if (hst->state == 2) fail(CQG_E_RUNTIME, "repair left an empty cluster");
        }
        if (hst->state == 1) break;
        fc_kernel<<<1, 256, 0, s>>>(cen, K, Kp, fc, tau);
        table_kernel<<<K, 256, table_smem, s>>>(cen, K, dtab, dsorted, order);
        launched(ctx, 2);
    }
    out.iterations = iter;
    CQG_CUDA(cudaMemcpyAsync(sse_host, sse_d, sizeof(double) * iter, cudaMemcpyDefault, s));
    CQG_CUDA(cudaMemcpyAsync(&out.ndc, ndc, 8, cudaMemcpyDeviceToHost, s));
    if (hist) {
        if (hist_labels_user) copy_out(ctx, hist_labels_user, hl_d, sizeof(uint32_t) * n * (size_t)iter);
        if (hist_centers_user) copy_out(ctx, hist_centers_user, hc_d, 24 * (size_t)K * iter);
    }
    CQG_CUDA(cudaStreamSynchronize(s));
    return out;
}

} // namespace cqg
