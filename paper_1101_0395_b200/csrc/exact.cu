// exact.cu -- the reference's Lloyd loop for arbitrary inputs, on the device.
//
// The hot path (lloyd.cu) clusters count-weighted colours on the 8-bit grid
// with exact integer moments. The reference's public API also takes real
// points with arbitrary positive weights (wsm, kmeans.hpp:128-129; its unit
// tests use random weights, tests/test_kmeans.cpp:193-208) and offers the
// unpruned, unrepaired reference engine kmeans_full (kmeans.hpp:119). This
// file runs that general case with the reference's own arithmetic order, so
// every output is bit-identical to run_lloyd (src/kmeans.cpp:192-260):
//
//   ex_table_kernel    build_center_distance_table (kmeans.cpp:14-38): one
//                      block per row, bitonic sort of (dist2, index), self
//                      rotated to the front
//   ex_assign_kernel   nearest_full (:40-54) or assign_point_sortmeans (:56-79),
//                      one point per thread, FP64 without contraction; NDC
//   repair             repair_empty_clusters (:124-169): host-driven loop over
//                      empty clusters, donor = parallel (max w*d2, lowest
//                      index) argmax, fallback = lowest index in a cluster of
//                      size >= 2
//   ex_update_kernel   weighted means: one thread per cluster accumulates its
//                      members in point order (the reference's sequential
//                      sum_r[m] += w*x.r chains, kmeans.cpp:228-243)
//   ex_sse_kernel      compute_sse (:107-122): terms in parallel, ONE
//                      sequential FP64 chain in point order
//
// The same kernels serve the API helpers compute_sse, repair_empty_clusters,
// build_center_distance_table, kmeanspp_next_masses and maximin_pad
// (init.cpp:316-335). Not a throughput path: per-iteration host round trips
// and O(n) sequential chains are the price of reproducing sequential FP64 sums.
#include <cstring>
#include <vector>

#include "cqg_internal.cuh"

namespace cqg {
namespace {

__device__ __forceinline__ double pd2(const double *x, const double *c) {
    return d2_exact(x[0], x[1], x[2], c[0], c[1], c[2]);
}

struct ValIdx64 {
    double v;
    unsigned long long i;
};

// row i of the centre table: dist2 in index order, walk order sorted by
// (dist2, index) with self forced to the front (std::rotate, kmeans.cpp:32-35)
__global__ void __launch_bounds__(256) ex_table_kernel(const double *__restrict__ cen, int K, int Kpow,
                                                       double *__restrict__ dist, uint32_t *__restrict__ order) {
    extern __shared__ unsigned long long s_key[];
    int *s_idx = reinterpret_cast<int *>(s_key + Kpow);
    __shared__ int s_self;
    const int i = blockIdx.x;
    for (int j = threadIdx.x; j < Kpow; j += blockDim.x) {
        if (j < K) {
            const double d = pd2(cen + 3 * i, cen + 3 * j);
            dist[(size_t)i * K + j] = d;
            s_key[j] = (unsigned long long)__double_as_longlong(d); // d >= 0: bits order like values
        } else {
            s_key[j] = ~0ull;
        }
        s_idx[j] = j;
    }
    __syncthreads();
    for (int size = 2; size <= Kpow; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (Kpow >> 1); t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = s_key[lo], b = s_key[hi];
                const int ia = s_idx[lo], ib = s_idx[hi];
                const bool gt = a > b || (a == b && ia > ib);
                if (gt == up) {
                    s_key[lo] = b;
                    s_key[hi] = a;
                    s_idx[lo] = ib;
                    s_idx[hi] = ia;
                }
            }
            __syncthreads();
        }
    for (int p = threadIdx.x; p < K; p += blockDim.x)
        if (s_idx[p] == i) s_self = p;
    __syncthreads();
    const int ps = s_self;
    for (int p = threadIdx.x; p < K; p += blockDim.x) {
        const int np = p < ps ? p + 1 : (p == ps ? 0 : p);
        order[(size_t)i * K + np] = (uint32_t)s_idx[p];
    }
}

__device__ __forceinline__ void add_ndc(unsigned long long local, unsigned long long *ndc) {
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(ndc, local);
}

// nearest_full (full != 0) or assign_point_sortmeans with the previous labels
__global__ void __launch_bounds__(256) ex_assign_kernel(const double *__restrict__ pts, uint64_t n,
                                                        const double *__restrict__ cen_g, int K,
                                                        const double *__restrict__ dist,
                                                        const uint32_t *__restrict__ order,
                                                        uint32_t *__restrict__ labels, int full,
                                                        unsigned long long *ndc) {
    extern __shared__ double s_c[];
    const bool sm = K <= 2048;
    if (sm)
        for (int j = threadIdx.x; j < 3 * K; j += blockDim.x) s_c[j] = cen_g[j];
    __syncthreads();
    const double *cen = sm ? s_c : cen_g;
    unsigned long long local = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double *x = pts + 3 * i;
        uint32_t best;
        if (full) {
            best = 0;
            double bd = pd2(x, cen);
            for (int j = 1; j < K; ++j) {
                const double d = pd2(x, cen + 3 * j);
                if (d < bd) {
                    bd = d;
                    best = (uint32_t)j;
                }
            }
            local += (unsigned long long)K;
        } else {
            const uint32_t prev = labels[i];
            const double *drow = dist + (size_t)prev * K;
            const uint32_t *orow = order + (size_t)prev * K;
            const double pdist = pd2(x, cen + 3 * prev);
            const double cut = __dmul_rn(4.0, pdist);
            double bd = pdist;
            best = prev;
            unsigned long long c = 1;
            for (int j = 1; j < K; ++j) {
                const uint32_t t = orow[j];
                if (drow[t] >= cut) break;
                const double d = pd2(x, cen + 3 * t);
                ++c;
                if (d < bd) {
                    bd = d;
                    best = t;
                }
            }
            local += c;
        }
        labels[i] = best;
    }
    add_ndc(local, ndc);
}

__global__ void ex_sizes_kernel(const uint32_t *__restrict__ labels, uint64_t n, uint32_t *__restrict__ sizes) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(sizes + labels[i], 1u);
}

__device__ __forceinline__ bool vi_better(const ValIdx64 &a, const ValIdx64 &b) {
    return a.v > b.v || (a.v == b.v && a.i < b.i);
}

// largest w_i * d2(x_i, c_{m_i}); equal values -> lowest index (the reference's
// strict '>' scan from index 0, kmeans.cpp:138-145). Block partials.
__global__ void __launch_bounds__(256) ex_donor_kernel(const double *__restrict__ pts, const double *__restrict__ w,
                                                       uint64_t n, const double *__restrict__ cen,
                                                       const uint32_t *__restrict__ labels, ValIdx64 *part) {
    ValIdx64 best{-1.0, ~0ull};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double d = pd2(pts + 3 * i, cen + 3 * labels[i]);
        const ValIdx64 c{w ? __dmul_rn(w[i], d) : d, i};
        if (vi_better(c, best)) best = c;
    }
    __shared__ ValIdx64 s[256];
    s[threadIdx.x] = best;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if ((int)threadIdx.x < o && vi_better(s[threadIdx.x + o], s[threadIdx.x])) s[threadIdx.x] = s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void ex_donor_final(ValIdx64 *part, int nparts) {
    if (threadIdx.x != 0) return;
    ValIdx64 b = part[0];
    for (int p = 1; p < nparts; ++p)
        if (vi_better(part[p], b)) b = part[p];
    part[0] = b;
}

// fallback donor: the lowest index whose cluster holds >= 2 points (kmeans.cpp:147-156)
__global__ void ex_spare_kernel(const uint32_t *__restrict__ labels, uint64_t n, const uint32_t *__restrict__ sizes,
                                unsigned long long *first) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        if (sizes[labels[i]] >= 2) {
            atomicMin(first, (unsigned long long)i);
            return;
        }
}

__global__ void ex_move_kernel(const double *__restrict__ pts, uint32_t *labels, double *cen, uint32_t *sizes,
                               unsigned long long donor, int e) {
    const uint32_t old = labels[donor];
    sizes[old] -= 1;
    sizes[e] += 1;
    labels[donor] = (uint32_t)e;
    cen[3 * e] = pts[3 * donor];
    cen[3 * e + 1] = pts[3 * donor + 1];
    cen[3 * e + 2] = pts[3 * donor + 2];
}

// weighted means, one thread per cluster, members in point order (the
// reference's sequential accumulation); points staged through shared memory
constexpr int kUpdChunk = 1024;
__global__ void __launch_bounds__(256) ex_update_kernel(const double *__restrict__ pts, const double *__restrict__ w,
                                                        uint64_t n, const uint32_t *__restrict__ labels, int K,
                                                        double *__restrict__ cen) {
    __shared__ double s_x[3 * kUpdChunk];
    __shared__ double s_w[kUpdChunk];
    __shared__ uint32_t s_l[kUpdChunk];
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    double sr = 0.0, sg = 0.0, sb = 0.0, ws = 0.0;
    for (uint64_t base = 0; base < n; base += kUpdChunk) {
        const int m = (int)(n - base < (uint64_t)kUpdChunk ? n - base : (uint64_t)kUpdChunk);
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            s_l[j] = labels[base + j];
            s_w[j] = w ? w[base + j] : 1.0;
        }
        for (int j = threadIdx.x; j < 3 * m; j += blockDim.x) s_x[j] = pts[3 * base + j];
        __syncthreads();
        if (c < K)
            for (int j = 0; j < m; ++j)
                if (s_l[j] == (uint32_t)c) {
                    const double wj = s_w[j];
                    sr = __dadd_rn(sr, __dmul_rn(wj, s_x[3 * j]));
                    sg = __dadd_rn(sg, __dmul_rn(wj, s_x[3 * j + 1]));
                    sb = __dadd_rn(sb, __dmul_rn(wj, s_x[3 * j + 2]));
                    ws = __dadd_rn(ws, wj);
                }
        __syncthreads();
    }
    if (c < K && ws > 0.0) { // an empty cluster keeps its centre (kmeans.cpp:240-243)
        cen[3 * c] = __ddiv_rn(sr, ws);
        cen[3 * c + 1] = __ddiv_rn(sg, ws);
        cen[3 * c + 2] = __ddiv_rn(sb, ws);
    }
}

// compute_sse: terms w_i * d2 (or d2) in parallel, one sequential chain in point order
constexpr int kSseChunk = 4096;
__global__ void __launch_bounds__(256) ex_sse_kernel(const double *__restrict__ pts, const double *__restrict__ w,
                                                     uint64_t n, const double *__restrict__ cen,
                                                     const uint32_t *__restrict__ labels, double *out) {
    __shared__ double s_t[kSseChunk];
    double sse = 0.0;
    for (uint64_t base = 0; base < n; base += kSseChunk) {
        const int m = (int)(n - base < (uint64_t)kSseChunk ? n - base : (uint64_t)kSseChunk);
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            const uint64_t i = base + j;
            const double d = pd2(pts + 3 * i, cen + 3 * labels[i]);
            s_t[j] = w ? __dmul_rn(w[i], d) : d;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int j = 0; j < m; ++j) sse = __dadd_rn(sse, s_t[j]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sse;
}

// min over the centres of d2(colour_p, c) (init.cpp:28-35; std::min keeps the
// current value unless the new one is strictly smaller)
__global__ void ex_mind2_kernel(const double *__restrict__ pts, uint64_t n, const double *__restrict__ cen, int k0,
                                double *__restrict__ md) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        double m = __longlong_as_double(0x7FF0000000000000ll);
        for (int j = 0; j < k0; ++j) {
            const double d = pd2(pts + 3 * i, cen + 3 * j);
            if (d < m) m = d;
        }
        md[i] = m;
    }
}

__global__ void ex_mass_kernel(const double *__restrict__ w, const double *__restrict__ md, uint64_t n,
                               double *__restrict__ mass) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        mass[i] = __dmul_rn(w[i], md[i]);
}

// maximin round: argmax of md (first maximum: strict '>' from index 0, init.cpp:42-45)
__global__ void __launch_bounds__(256) ex_argmax_kernel(const double *__restrict__ md, uint64_t n, ValIdx64 *part) {
    ValIdx64 best{-1.0, ~0ull};
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const ValIdx64 c{md[i], i};
        if (vi_better(c, best)) best = c;
    }
    __shared__ ValIdx64 s[256];
    s[threadIdx.x] = best;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if ((int)threadIdx.x < o && vi_better(s[threadIdx.x + o], s[threadIdx.x])) s[threadIdx.x] = s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

// append the chosen colour and lower every md against it
__global__ void ex_pick_kernel(const double *__restrict__ pts, uint64_t n, const ValIdx64 *best, double *cen, int slot,
                               double *__restrict__ md) {
    const uint64_t b = best->i;
    const double cr = pts[3 * b], cg = pts[3 * b + 1], cb = pts[3 * b + 2];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        cen[3 * slot] = cr;
        cen[3 * slot + 1] = cg;
        cen[3 * slot + 2] = cb;
    }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const double d = d2_exact(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], cr, cg, cb);
        if (d < md[i]) md[i] = d;
    }
}

int grid_for(const cqg_ctx *ctx, uint64_t n) {
    uint64_t g = (n + 255) / 256;
    const uint64_t gmax = (uint64_t)ctx->num_sms * 4;
    if (g > gmax) g = gmax;
    return (int)(g ? g : 1);
}

int kpow(int K) {
    int p = 1;
    while (p < K) p <<= 1;
    return p;
}

} // namespace

void exact_table_dev(cqg_ctx *ctx, const double *cen_d, int K, double *dist_d, uint32_t *order_d) {
    const int Kp = kpow(K);
    const size_t smem = (size_t)Kp * (sizeof(unsigned long long) + sizeof(int));
    if (smem > 48 * 1024) CQG_CUDA(ensure_smem((const void *)ex_table_kernel, smem));
    ex_table_kernel<<<K, 256, smem, ctx->stream>>>(cen_d, K, Kp, dist_d, order_d);
    CQG_CUDA(cudaGetLastError());
    launched(ctx);
}

double exact_sse_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, const double *cen_d,
                     const uint32_t *lab_d, double *out_d) {
    ex_sse_kernel<<<1, 256, 0, ctx->stream>>>(pts_d, w_d, n, cen_d, lab_d, out_d);
    CQG_CUDA(cudaGetLastError());
    launched(ctx);
    double *h = static_cast<double *>(ctx->pinned.ensure(4096)) + 500;
    CQG_CUDA(cudaMemcpyAsync(h, out_d, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    return *h;
}

int exact_repair_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, double *cen_d, int K,
                     uint32_t *lab_d) {
    cudaStream_t s = ctx->stream;
    uint32_t *sizes = static_cast<uint32_t *>(ctx->sizes.ensure(sizeof(uint32_t) * (size_t)K + 64));
    const int g = grid_for(ctx, n);
    ValIdx64 *part = static_cast<ValIdx64 *>(ctx->red.ensure(sizeof(ValIdx64) * (size_t)g + 64));
    unsigned long long *spare = reinterpret_cast<unsigned long long *>(part + g);
    CQG_CUDA(cudaMemsetAsync(sizes, 0, sizeof(uint32_t) * (size_t)K, s));
    ex_sizes_kernel<<<g, 256, 0, s>>>(lab_d, n, sizes);
    launched(ctx);
    std::vector<uint32_t> hs(K);
    CQG_CUDA(cudaMemcpyAsync(hs.data(), sizes, sizeof(uint32_t) * (size_t)K, cudaMemcpyDeviceToHost, s));
    CQG_CUDA(cudaStreamSynchronize(s));
    ValIdx64 *hb = reinterpret_cast<ValIdx64 *>(static_cast<char *>(ctx->pinned.ensure(4096)) + 3584);
    int repairs = 0;
    for (int e = 0; e < K;) {
        if (hs[e] != 0) {
            ++e;
            continue;
        }
        ex_donor_kernel<<<g, 256, 0, s>>>(pts_d, w_d, n, cen_d, lab_d, part);
        ex_donor_final<<<1, 32, 0, s>>>(part, g);
        launched(ctx, 2);
        CQG_CUDA(cudaMemcpyAsync(hb, part, sizeof(ValIdx64), cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaStreamSynchronize(s));
        unsigned long long donor = hb->i;
        if (!(hb->v > 0.0)) {
            CQG_CUDA(cudaMemsetAsync(spare, 0xFF, 8, s));
            ex_spare_kernel<<<g, 256, 0, s>>>(lab_d, n, sizes, spare);
            launched(ctx);
            CQG_CUDA(cudaMemcpyAsync(&hb->i, spare, 8, cudaMemcpyDeviceToHost, s));
            CQG_CUDA(cudaStreamSynchronize(s));
            donor = hb->i;
            if (donor == ~0ull) fail(CQG_E_RUNTIME, "repair_empty_clusters: more clusters than points");
        }
        uint32_t old = 0;
        CQG_CUDA(cudaMemcpy(&old, lab_d + donor, 4, cudaMemcpyDeviceToHost));
        ex_move_kernel<<<1, 1, 0, s>>>(pts_d, lab_d, cen_d, sizes, donor, e);
        launched(ctx);
        hs[old] -= 1;
        hs[e] += 1;
        ++repairs;
        e = 0; // the donor's cluster may have emptied (kmeans.cpp:164)
    }
    return repairs;
}

ExactOut exact_lloyd_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, const double *init_d,
                         int K, const cqg_term &term, bool prune_repair, uint32_t *lab_d, double *cen_d,
                         double *sse_host, uint32_t *hist_labels_user, double *hist_centers_user) {
    cudaStream_t s = ctx->stream;
    const int limit = term.fixed_iterations > 0 ? term.fixed_iterations : term.max_iterations;
    CQG_CUDA(cudaMemcpyAsync(cen_d, init_d, 24 * (size_t)K, cudaMemcpyDeviceToDevice, s));
    double *dist = static_cast<double *>(ctx->dtab.ensure(sizeof(double) * (size_t)K * K));
    uint32_t *order = static_cast<uint32_t *>(ctx->order.ensure(sizeof(uint32_t) * (size_t)K * K));
    unsigned long long *ndc = static_cast<unsigned long long *>(ctx->ndc.ensure(64));
    double *sse_d = reinterpret_cast<double *>(ndc + 2);
    CQG_CUDA(cudaMemsetAsync(ndc, 0, 8, s));
    const int g = grid_for(ctx, n);
    const size_t csm = K <= 2048 ? 24 * (size_t)K : 0;
    if (csm > 48 * 1024) CQG_CUDA(ensure_smem((const void *)ex_assign_kernel, csm));
    ExactOut out;
    std::vector<double> trace;
    for (int iter = 1;; ++iter) {
        const bool walk = prune_repair && iter > 1;
        if (walk) exact_table_dev(ctx, cen_d, K, dist, order);
        ex_assign_kernel<<<g, 256, csm, s>>>(pts_d, n, cen_d, K, dist, order, lab_d, walk ? 0 : 1, ndc);
        launched(ctx);
        if (term.record_history) { // pre-repair snapshot (kmeans.cpp:219)
            if (hist_centers_user)
                CQG_CUDA(cudaMemcpyAsync(hist_centers_user + (size_t)(iter - 1) * 3 * K, cen_d, 24 * (size_t)K,
                                         cudaMemcpyDefault, s));
            if (hist_labels_user)
                CQG_CUDA(cudaMemcpyAsync(hist_labels_user + (size_t)(iter - 1) * n, lab_d, 4 * n, cudaMemcpyDefault, s));
        }
        if (prune_repair) out.repairs += exact_repair_dev(ctx, pts_d, w_d, n, cen_d, K, lab_d);
        ex_update_kernel<<<(K + 255) / 256, 256, 0, s>>>(pts_d, w_d, n, lab_d, K, cen_d);
        launched(ctx);
        const double sse = exact_sse_dev(ctx, pts_d, w_d, n, cen_d, lab_d, sse_d);
        trace.push_back(sse);
        out.iterations = iter;
        if (term.fixed_iterations > 0) {
            if (iter >= limit) break;
        } else {
            if (sse == 0.0) break;
            if (iter >= 2 && (trace[iter - 2] - sse) / sse <= term.epsilon) break; // check_convergence (kmeans.cpp:9-12)
            if (iter >= limit) break;
        }
    }
    if (sse_host) std::memcpy(sse_host, trace.data(), 8 * trace.size());
    unsigned long long *h = reinterpret_cast<unsigned long long *>(static_cast<char *>(ctx->pinned.ensure(4096)) + 3968);
    CQG_CUDA(cudaMemcpyAsync(h, ndc, 8, cudaMemcpyDeviceToHost, s));
    CQG_CUDA(cudaStreamSynchronize(s));
    out.ndc = *h;
    return out;
}

void exact_next_masses_dev(cqg_ctx *ctx, const double *pts_d, const double *w_d, uint64_t n, const double *cen_d,
                           int k0, double *mass_d) {
    double *md = static_cast<double *>(ctx->mind2.ensure(sizeof(double) * (n + 1)));
    const int g = grid_for(ctx, n);
    ex_mind2_kernel<<<g, 256, 0, ctx->stream>>>(pts_d, n, cen_d, k0, md);
    ex_mass_kernel<<<g, 256, 0, ctx->stream>>>(w_d, md, n, mass_d);
    CQG_CUDA(cudaGetLastError());
    launched(ctx, 2);
}

void exact_maximin_pad_dev(cqg_ctx *ctx, const double *pts_d, uint64_t n, double *cen_d, int k0, int k) {
    double *md = static_cast<double *>(ctx->mind2.ensure(sizeof(double) * (n + 1)));
    const int g = grid_for(ctx, n);
    ValIdx64 *part = static_cast<ValIdx64 *>(ctx->red.ensure(sizeof(ValIdx64) * (size_t)g + 64));
    ex_mind2_kernel<<<g, 256, 0, ctx->stream>>>(pts_d, n, cen_d, k0, md);
    launched(ctx);
    for (int slot = k0; slot < k; ++slot) {
        ex_argmax_kernel<<<g, 256, 0, ctx->stream>>>(md, n, part);
        ex_donor_final<<<1, 32, 0, ctx->stream>>>(part, g);
        ex_pick_kernel<<<g, 256, 0, ctx->stream>>>(pts_d, n, part, cen_d, slot, md);
        launched(ctx, 3);
    }
    CQG_CUDA(cudaGetLastError());
}

} // namespace cqg
