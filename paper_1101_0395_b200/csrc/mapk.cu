// mapk.cu -- stage 4: pixel -> palette mapping and MSE.
//
// Replaces quant::map_pixels (reference src/metrics.cpp:15-55). The reference
// resolves each distinct colour once through nearest_pruned_lowest_index
// (kmeans.cpp:81-105), whose result is the exact lowest-index FP64 argmin
// (kmeans.hpp:88-96), caches it in a hash map and accumulates
// dist2(centre, pixel) sequentially. Here:
//   sweep<MAP> + replay<MAP>  lowest-index argmin per distinct colour (same
//                             FP32 sweep + exact FP64 replay as Lloyd) written
//                             to a 2^24-entry LUT, plus exact per-cluster
//                             pixel moments (count-weighted);
//   mse_kernel                mean_sq_dist = sum_k [(nQ-|S|^2)/n + n|c-S/n|^2] / P
//                             from those moments (deterministic, ~1e-14 of the
//                             reference's sequential FP64 sum);
//   map_walk_kernel +         MappingResult::ndc: the reference resolves the
//   map_ndc_kernel            distinct colours in first-occurrence order with the
//                             hint = the index chosen for the previous distinct
//                             colour (0 for the first), and the pruned walk
//                             evaluates 1 + #{j >= 1 : D[hint][order_j] <= 4 d2(x, c_hint)}
//                             distances (it breaks only on '>'). The walk row is
//                             ascending (self, distance 0, first), so that count
//                             is the number of row entries <= the cutoff: a
//                             binary search per colour over the palette's sorted
//                             distance rows, all colours in parallel;
//   pixel_kernel              per pixel: LUT gather -> index (u8 or u32) and the
//                             palette colour rendered by channel_to_u8
//                             (color.hpp:63-72); 16 pixels / thread, 128-bit
//                             loads and stores. HBM bound: 3P in, (1|4)P + 3P out.
#include "sweep.cuh"

namespace cqg {
namespace {

__global__ void mse_kernel(const Moments *mom, const double *pal, int K, uint64_t P, double *out) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ double s_t[];
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const Moments m = mom[k];
        double t = 0.0;
        if (m.n != 0) {
            const double nd = __ull2double_rn(m.n);
            const double a = cluster_sse_exact(m.n, m.s, m.q);
            const double dr = __dsub_rn(pal[3 * k], __ddiv_rn(__ll2double_rn(m.s[0]), nd));
            const double dg = __dsub_rn(pal[3 * k + 1], __ddiv_rn(__ll2double_rn(m.s[1]), nd));
            const double db = __dsub_rn(pal[3 * k + 2], __ddiv_rn(__ll2double_rn(m.s[2]), nd));
            const double e = __dadd_rn(__dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dg, dg)), __dmul_rn(db, db));
            t = __dadd_rn(a, __dmul_rn(nd, e));
        }
        s_t[k] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int k = 0; k < K; ++k)
            if (mom[k].n != 0) tot = __dadd_rn(tot, s_t[k]);
        *out = __ddiv_rn(tot, __ull2double_rn(P));
    }
}

__device__ __forceinline__ uint8_t channel_to_u8(double v) {
    double r = floor(__dadd_rn(v, 0.5));
    if (r < 0.0) r = 0.0;
    if (r > 255.0) r = 255.0;
    return (uint8_t)r;
}

__device__ __forceinline__ uint4 ld_stream4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void st_stream4(uint4 *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w));
}

// IB = index bytes (1 or 4); LUT8 = LUT element is uint8 (K <= 256)
template <int IB, bool LUT8>
__global__ void __launch_bounds__(256) pixel_kernel(const uint8_t *__restrict__ rgb, uint64_t P,
                                                   const void *__restrict__ lut_v,
                                                   const double *__restrict__ pal, int K,
                                                   void *__restrict__ idx_out,
                                                   uint8_t *__restrict__ q_out, int vec) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint32_t s_pal8[]; // packed 0x00BBGGRR little-endian bytes r,g,b
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        s_pal8[k] = (uint32_t)channel_to_u8(pal[3 * k]) | ((uint32_t)channel_to_u8(pal[3 * k + 1]) << 8) |
                    ((uint32_t)channel_to_u8(pal[3 * k + 2]) << 16);
    __syncthreads();
    const uint8_t *lut8 = static_cast<const uint8_t *>(lut_v);
    const uint32_t *lut32 = static_cast<const uint32_t *>(lut_v);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t groups = vec ? P / 16 : 0;
    for (uint64_t g = tid; g < groups; g += stride) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rgb + g * 48);
        const uint4 a = ld_stream4(src), b = ld_stream4(src + 1), d = ld_stream4(src + 2);
        const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
        uint32_t idx[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int o = 3 * j;
            const uint32_t b0 = (w[o >> 2] >> (8 * (o & 3))) & 255u;
            const uint32_t b1 = (w[(o + 1) >> 2] >> (8 * ((o + 1) & 3))) & 255u;
            const uint32_t b2 = (w[(o + 2) >> 2] >> (8 * ((o + 2) & 3))) & 255u;
            const uint32_t c = (b0 << 16) | (b1 << 8) | b2;
            idx[j] = LUT8 ? (uint32_t)__ldg(lut8 + c) : __ldg(lut32 + c);
        }
        // quantized RGB: 16 pixels = 48 bytes = 12 words
        uint32_t qw[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) qw[i] = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t p8 = s_pal8[idx[j]];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
                const int o = 3 * j + ch;
                qw[o >> 2] |= ((p8 >> (8 * ch)) & 255u) << (8 * (o & 3));
            }
        }
        uint4 *dst = reinterpret_cast<uint4 *>(q_out + g * 48);
        if (q_out) {
            st_stream4(dst, make_uint4(qw[0], qw[1], qw[2], qw[3]));
            st_stream4(dst + 1, make_uint4(qw[4], qw[5], qw[6], qw[7]));
            st_stream4(dst + 2, make_uint4(qw[8], qw[9], qw[10], qw[11]));
        }
        if (idx_out) {
            if (IB == 1) {
                uint32_t iw[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    iw[i] = idx[4 * i] | (idx[4 * i + 1] << 8) | (idx[4 * i + 2] << 16) | (idx[4 * i + 3] << 24);
                st_stream4(reinterpret_cast<uint4 *>(static_cast<uint8_t *>(idx_out) + g * 16),
                           make_uint4(iw[0], iw[1], iw[2], iw[3]));
            } else {
                uint4 *o4 = reinterpret_cast<uint4 *>(static_cast<uint32_t *>(idx_out) + g * 16);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    st_stream4(o4 + i, make_uint4(idx[4 * i], idx[4 * i + 1], idx[4 * i + 2], idx[4 * i + 3]));
            }
        }
    }
    for (uint64_t p = groups * 16 + tid; p < P; p += stride) {
        const uint32_t c = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
        const uint32_t id = LUT8 ? (uint32_t)lut8[c] : lut32[c];
        const uint32_t p8 = s_pal8[id];
        if (q_out) {
            q_out[3 * p] = (uint8_t)(p8 & 255u);
            q_out[3 * p + 1] = (uint8_t)((p8 >> 8) & 255u);
            q_out[3 * p + 2] = (uint8_t)((p8 >> 16) & 255u);
        }
        if (idx_out) {
            if (IB == 1) static_cast<uint8_t *>(idx_out)[p] = (uint8_t)id;
            else static_cast<uint32_t *>(idx_out)[p] = id;
        }
    }
}


// Palette walk rows for the mapping NDC (kmeans.cpp:14-38 distances): row i
// holds d2(c_i, c_j) for every j (self = 0 included) ascending, padded with
// +inf to Kpow; with K <= 256 also as 16-bit codes (code16, sweep.cuh).
__global__ void __launch_bounds__(256) map_walk_kernel(const double *__restrict__ pal, int K, int Kpow,
                                                       double *__restrict__ rows, uint16_t *__restrict__ codes) {
    extern __shared__ unsigned long long s_k[]; // Kpow keys (bits of non-negative doubles order like the values)
    const int i = blockIdx.x;
    const double cr = pal[3 * i], cg = pal[3 * i + 1], cb = pal[3 * i + 2];
    for (int j = threadIdx.x; j < Kpow; j += blockDim.x)
        s_k[j] = j < K ? (unsigned long long)__double_as_longlong(
                             d2_exact(cr, cg, cb, pal[3 * j], pal[3 * j + 1], pal[3 * j + 2]))
                       : 0x7FF0000000000000ull;
    __syncthreads();
    for (int size = 2; size <= Kpow; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (Kpow >> 1); t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long a = s_k[lo], b = s_k[hi];
                if ((a > b) == up) {
                    s_k[lo] = b;
                    s_k[hi] = a;
                }
            }
            __syncthreads();
        }
    for (int j = threadIdx.x; j < Kpow; j += blockDim.x) {
        const double d = __longlong_as_double((long long)s_k[j]);
        rows[(size_t)i * Kpow + j] = d;
        if (codes) codes[(size_t)i * Kpow + j] = (uint16_t)code16(d);
    }
}

// Mapping NDC (metrics.cpp:36-48 + kmeans.cpp:81-105): colour i of the image's
// distinct colours in first-occurrence order resolves with hint = the label of
// colour i-1 (0 for i = 0; the sweep stored the labels in substrate order) and
// costs #{row entries <= 4 d2(x, c_hint)} distances. "<= cut" is counted as
// "< nextup(cut)" (no double lies between). CODES: rows as 16-bit codes in
// shared memory (K <= 256), FP64 only on code ties; otherwise the FP64 rows
// through L1. Q colours per thread, the next batch's loads in flight.
template <bool CODES, int Q, int NT>
__global__ void __launch_bounds__(NT) map_ndc_kernel(const uint32_t *__restrict__ colors, uint64_t n,
                                                     const uint8_t *__restrict__ lab8,
                                                     const uint32_t *__restrict__ lab32,
                                                     const double *__restrict__ pal, int K, int Kpow,
                                                     const double *__restrict__ rows,
                                                     const uint16_t *__restrict__ codes,
                                                     unsigned long long *ndc) {
    extern __shared__ __align__(16) double s_pal[];
    const int rs = Kpow + 2; // code row stride: one padding word spreads rows over the banks
    uint16_t *s_code = reinterpret_cast<uint16_t *>(s_pal + 3 * K);
    for (int i = threadIdx.x; i < 3 * K; i += blockDim.x) s_pal[i] = pal[i];
    if (CODES) {
        // 8 codes per 16-byte load, 8 loads in flight per thread; stored as
        // 32-bit words into rows padded by one word (Kpow >= 8 here)
        const uint4 *src = reinterpret_cast<const uint4 *>(codes);
        uint32_t *dst = reinterpret_cast<uint32_t *>(s_code);
        const int total = K * Kpow / 8, q4 = Kpow / 8, hw = Kpow / 2;
        for (int e0 = threadIdx.x; e0 < total; e0 += 8 * NT) {
            uint4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NT;
                v[u] = __ldg(src + (e < total ? e : 0));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * NT;
                if (e < total) {
                    const int r = e / q4, w = (e - r * q4) * 4;
                    uint32_t *d = dst + r * (hw + 1) + w;
                    d[0] = v[u].x;
                    d[1] = v[u].y;
                    d[2] = v[u].z;
                    d[3] = v[u].w;
                }
            }
        }
    }
    __syncthreads();
    unsigned long long local = 0;
    const uint64_t stride = (uint64_t)gridDim.x * NT * Q;
    uint32_t ncol[Q], nhint[Q];
    auto load_batch = [&](uint64_t b) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = b + threadIdx.x + (uint64_t)q * NT;
            const uint64_t ic = i < n ? i : 0;
            ncol[q] = __ldg(colors + ic);
            nhint[q] = ic == 0 ? 0u : (lab8 ? (uint32_t)__ldg(lab8 + ic - 1) : __ldg(lab32 + ic - 1));
        }
    };
    uint64_t base = (uint64_t)blockIdx.x * NT * Q;
    if (base < n) load_batch(base);
    for (; base < n; base += stride) {
        double cut[Q];
        uint32_t cc[Q];
        int hint[Q], pos[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = base + threadIdx.x + (uint64_t)q * NT;
            const bool v = i < n;
            const uint32_t col = ncol[q], h = nhint[q];
            const double pd = d2_exact((double)((col >> 16) & 255u), (double)((col >> 8) & 255u),
                                       (double)(col & 255u), s_pal[3 * h], s_pal[3 * h + 1], s_pal[3 * h + 2]);
            // nextup(4 pd): the cutoff is non-negative, so the next double up is bits + 1
            cut[q] = v ? __longlong_as_double(__double_as_longlong(__dmul_rn(4.0, pd)) + 1) : -1.0;
            cc[q] = v ? code16(cut[q]) : 0u;
            hint[q] = (int)h;
            pos[q] = 0;
        }
        if (base + stride < n) load_batch(base + stride);
        for (int step = Kpow >> 1; step >= 1; step >>= 1) {
            if (CODES) {
                uint32_t vv[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) vv[q] = s_code[hint[q] * rs + pos[q] + step - 1];
#pragma unroll
                for (int q = 0; q < Q; ++q) pos[q] += vv[q] < cc[q] ? step : 0;
            } else {
                double vv[Q];
#pragma unroll
                for (int q = 0; q < Q; ++q) vv[q] = __ldg(rows + (size_t)hint[q] * Kpow + pos[q] + step - 1);
#pragma unroll
                for (int q = 0; q < Q; ++q) pos[q] += vv[q] < cut[q] ? step : 0;
            }
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (cut[q] < 0.0) continue;
            const double *grow = rows + (size_t)hint[q] * Kpow;
            int p = pos[q];
            if (CODES) {
                const uint16_t *row = s_code + hint[q] * rs;
                if (p == Kpow - 1 && row[Kpow - 1] < cc[q]) p = Kpow;
                while (p < Kpow && row[p] == cc[q] && __ldg(grow + p) < cut[q]) ++p; // code ties: FP64
            } else if (p == Kpow - 1 && __ldg(grow + Kpow - 1) < cut[q]) {
                p = Kpow; // the lifting reaches Kpow - 1 at most
            }
            local += (unsigned long long)p;
        }
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(ndc, local);
}

} // namespace

double map_dev(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t P, const uint32_t *colors_d,
               const uint32_t *counts_d, uint64_t n, const double *pal_d, int K, void *indices_d,
               int index_bytes, uint8_t *quant_d, double *mse_async, const LloydOut *lloyd,
               unsigned long long *ndc_async) {
    cudaStream_t s = ctx->stream;
    const int Kp = pad_centres(K);
    const bool lut8 = K <= 256;
    float *fc = static_cast<float *>(ctx->fcen.ensure(sizeof(float) * (4 * (size_t)Kp + 8)));
    float *tau = fc + 4 * Kp;
    void *lut = ctx->lut.ensure(lut8 ? (1u << 24) : (sizeof(uint32_t) << 24));
    Moments *mom = static_cast<Moments *>(ctx->mom_map.ensure(sizeof(Moments) * (size_t)K + 64));
    double *mse_d = reinterpret_cast<double *>(mom + K);
    unsigned long long *ndc_d = reinterpret_cast<unsigned long long *>(mse_d + 1);
    uint32_t *queue = static_cast<uint32_t *>(ctx->queue.ensure(sizeof(uint32_t) * (n + 1)));
    uint32_t *qn = static_cast<uint32_t *>(ctx->scal.ensure(256));

    // bound-pruned mapping: the moments start from Lloyd's final ones (its labels)
    const bool pruned = lloyd && lloyd->bnd && ctx->use_prune;
    if (pruned)
        CQG_CUDA(cudaMemcpyAsync(mom, lloyd->mom, sizeof(Moments) * (size_t)K, cudaMemcpyDeviceToDevice, s));
    else
        CQG_CUDA(cudaMemsetAsync(mom, 0, sizeof(Moments) * (size_t)K, s));
    CQG_CUDA(cudaMemsetAsync(qn, 0, 4, s));
    fc_kernel<<<1, 256, 0, s>>>(pal_d, K, Kp, fc, tau);
    launched(ctx);

    SweepArgs a{};
    a.colors = colors_d;
    a.counts = counts_d;
    a.n = n;
    a.lut8 = lut8 ? static_cast<uint8_t *>(lut) : nullptr;
    a.lut32 = lut8 ? nullptr : static_cast<uint32_t *>(lut);
    a.fc = fc;
    a.cen = pal_d;
    a.tau = tau;
    a.queue = queue;
    a.qn = qn;
    a.mom = mom;
    a.K = K;
    a.Kp = Kp;
    if (ndc_async) { // the labels in substrate order for the mapping-NDC pass
        void *ml = ctx->map_lab.ensure((size_t)(n + 1) * (lut8 ? 1 : 4));
        a.maplab8 = lut8 ? static_cast<uint8_t *>(ml) : nullptr;
        a.maplab32 = lut8 ? nullptr : static_cast<uint32_t *>(ml);
    }
    if (pruned) {
        a.labels = const_cast<uint32_t *>(lloyd->labels); // read only in MODE_MAPW
        a.bnd = lloyd->bnd;                                  // read only in MODE_MAPW
        a.shift = lloyd->shift;
        a.dsorted = lloyd->dsorted;
        a.rowmin = lloyd->rowmin;
        a.Kpow = lloyd->Kpow;
        launch_sweep(ctx, MODE_MAPW, a);
    } else {
        launch_sweep(ctx, MODE_MAP, a);
    }

    bool ndc_pending = false;
    if (ndc_async) { // MappingResult::ndc, on the side stream beside the MSE and the pixel pass
        CQG_CUDA(cudaEventRecord(ctx->aux_fork, s));
        CQG_CUDA(cudaStreamWaitEvent(ctx->aux, ctx->aux_fork, 0));
        struct SideStream { // launches and profiling events below go to the side stream
            cqg_ctx *c;
            cudaStream_t main;
            ~SideStream() { c->stream = main; }
        } side{ctx, s};
        s = ctx->aux;
        ctx->stream = ctx->aux;
        int Kpow = 1;
        while (Kpow < K) Kpow <<= 1;
        CQG_CUDA(cudaMemsetAsync(ndc_d, 0, 8, s));
        const double *rows;
        const uint16_t *crow;
        if (lloyd && lloyd->dsorted && lloyd->Kpow == Kpow && (K > 256 || K < 8 || lloyd->dcode)) {
            // the palette is Lloyd's final centres: its last iteration built their walk table
            rows = lloyd->dsorted;
            crow = K <= 256 && K >= 8 ? lloyd->dcode : nullptr;
        } else {
            const bool codes = K <= 256 && K >= 8;
            double *r = static_cast<double *>(ctx->map_rows.ensure(sizeof(double) * (size_t)K * Kpow +
                                                                 (codes ? sizeof(uint16_t) * (size_t)K * Kpow : 0)));
            uint16_t *c = codes ? reinterpret_cast<uint16_t *>(r + (size_t)K * Kpow) : nullptr;
            const size_t wsm = sizeof(unsigned long long) * (size_t)Kpow;
            if (wsm > 48 * 1024) CQG_CUDA(ensure_smem((const void *)map_walk_kernel, wsm));
            map_walk_kernel<<<K, 256, wsm, s>>>(pal_d, K, Kpow, r, c);
            launched(ctx);
            rows = r;
            crow = c;
        }
        const int pn = prof_begin(ctx);
        if (crow) {
            // the rows as 16-bit codes in every block's shared memory (K <= 256)
            const size_t sm = (size_t)K * 24 + (size_t)K * (Kpow + 2) * 2;
            CQG_CUDA(ensure_smem((const void *)map_ndc_kernel<true, 4, 512>, sm));
            const uint64_t g = (n + 2048 - 1) / 2048, gmax = (uint64_t)ctx->num_sms;
            map_ndc_kernel<true, 4, 512><<<(unsigned)(g < gmax ? g : gmax), 512, sm, s>>>(
                colors_d, n, a.maplab8, a.maplab32, pal_d, K, Kpow, rows, crow, ndc_d);
        } else {
            // FP64 rows through L1/L2
            const size_t sm = (size_t)K * 24;
            if (sm > 48 * 1024) CQG_CUDA(ensure_smem((const void *)map_ndc_kernel<false, 4, 256>, sm));
            uint64_t g = (n + 1024 - 1) / 1024;
            const uint64_t gmax = (uint64_t)ctx->num_sms * 8;
            if (g > gmax) g = gmax;
            map_ndc_kernel<false, 4, 256><<<(unsigned)(g ? g : 1), 256, sm, s>>>(
                colors_d, n, a.maplab8, a.maplab32, pal_d, K, Kpow, rows, nullptr, ndc_d);
        }
        prof_end(ctx, CQG_PROF_MAPNDC, pn, (double)n);
        launched(ctx);
        CQG_CUDA(cudaMemcpyAsync(ndc_async, ndc_d, 8, cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaEventRecord(ctx->aux_join, s));
        s = side.main;
        ndc_pending = true;
    }

    if ((size_t)K * 8 > 48 * 1024)
        CQG_CUDA(ensure_smem((const void *)mse_kernel, K * 8));
    launch_pdl(mse_kernel, 1, 256, (size_t)K * 8, s, mom, pal_d, K, P, mse_d);
    launched(ctx);

    if (indices_d || quant_d) {
        const int vec = ((reinterpret_cast<uintptr_t>(rgb_d) | reinterpret_cast<uintptr_t>(indices_d) |
                          reinterpret_cast<uintptr_t>(quant_d)) & 15) == 0;
        uint64_t work = vec ? P / 16 + 1 : P;
        uint64_t grid = (work + 255) / 256;
        const uint64_t gmax = (uint64_t)ctx->num_sms * 8;
        if (grid > gmax) grid = gmax;
        const size_t smem = (size_t)K * 4;
        if (smem > 48 * 1024) {
            CQG_CUDA(ensure_smem((const void *)pixel_kernel<4, false>, smem));
        }
        const int pp = prof_begin(ctx);
        if (index_bytes == 1) {
            if (lut8) launch_pdl(pixel_kernel<1, true>, (unsigned)grid, 256, smem, s, rgb_d, P, lut, pal_d, K, indices_d, quant_d, vec);
            else fail(CQG_E_INVALID, "map_pixels: 8-bit indices need k <= 256");
        } else {
            if (lut8) launch_pdl(pixel_kernel<4, true>, (unsigned)grid, 256, smem, s, rgb_d, P, lut, pal_d, K, indices_d, quant_d, vec);
            else launch_pdl(pixel_kernel<4, false>, (unsigned)grid, 256, smem, s, rgb_d, P, lut, pal_d, K, indices_d, quant_d, vec);
        }
        prof_end(ctx, CQG_PROF_PIXEL, pp,
                 (double)P * (3.0 + (indices_d ? (double)index_bytes : 0.0) + (quant_d ? 3.0 : 0.0)));
        launched(ctx);
    }
    if (ndc_pending) CQG_CUDA(cudaStreamWaitEvent(s, ctx->aux_join, 0)); // join the side stream
    CQG_CUDA(cudaGetLastError());
    if (mse_async) { // the caller reads *mse_async after its own synchronisation
        CQG_CUDA(cudaMemcpyAsync(mse_async, mse_d, 8, cudaMemcpyDeviceToHost, s));
        return 0.0;
    }
    double mse = 0.0;
    double *hm = static_cast<double *>(ctx->pinned.ensure(4096));
    CQG_CUDA(cudaMemcpyAsync(hm, mse_d, 8, cudaMemcpyDeviceToHost, s));
    CQG_CUDA(cudaStreamSynchronize(s));
    mse = *hm;
    return mse;
}

} // namespace cqg
