// sweep.cuh -- the FP32 nearest-centre sweep shared by the Lloyd assignment
// (iteration 1: nearest_full, iteration >= 2: assign_point_sortmeans) and the
// palette mapping (nearest_pruned_lowest_index).
//
// Per (unique colour x, centre c) the sweep evaluates the expanded form
//     d = (|c|^2 + |x|^2) - 2 x.c
// as FADD2 + 3 FFMA2 on float pairs (two centres per instruction), packs the
// centre index into the low 8 mantissa bits of d and keeps the best and the
// second-best key with 3-input integer min/max (VIMNMX3). The result is exact
// whenever the best/second gap exceeds a rigorous bound on the FP32 error
// (tau, computed per iteration from the centre magnitudes); otherwise the
// point is queued and replayed in FP64 with the reference's own walk
// (replay kernels), so labels are bit-exact with the reference.
#pragma once

#include "cqg_internal.cuh"

namespace cqg {

constexpr int kSweepThreads = 256;
constexpr int kAccPerCluster = 6; // n, s_r, s_g, s_b, q_lo16, q_hi
constexpr uint32_t kHeavyCount = 2048; // counts >= this bypass the u32 smem accumulators

enum { MODE_FULL = 0, MODE_WALK = 1, MODE_MAP = 2 };

// Shared-memory layout of the FP32 centre table (Kp = K rounded up to 4):
//   m2r[Kp], m2g[Kp], m2b[Kp], cc[Kp]  (m2* = -2 * centre, cc = |centre|^2)
// Padding centres have cc = 1e30 and never win.

struct SweepArgs {
    const uint32_t *colors;
    const uint32_t *counts;
    uint64_t n;
    uint32_t *labels;       // FULL/WALK: per-point label (WALK reads prev, writes new)
    uint8_t *lut8;          // MAP, K <= 256: 2^24 LUT colour -> label
    uint32_t *lut32;        // MAP, K > 256
    const float *fc;        // 4*Kp floats (layout above)
    const double *cen;      // K x 3 FP64 centres
    const double *dtab;     // K x K, dist2 between centres (WALK replay)
    const double *dsorted;  // K x K, row i in walk order (WALK NDC)
    const uint32_t *order;  // K x K walk order (WALK replay)
    const float *tau;       // [0] abs bound, [1] relative (truncation) bound
    uint32_t *queue;
    uint32_t *qn;
    Moments *mom;
    unsigned long long *ndc;
    int K, Kp;
};

__device__ __forceinline__ uint32_t lane_lt_mask() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void enqueue(bool flag, uint32_t idx, uint32_t *queue, uint32_t *qn) {
    // every lane of the warp reaches this call (uniform tile loops)
    const uint32_t m = __ballot_sync(0xffffffffu, flag);
    if (m == 0) return;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(qn, (uint32_t)__popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (flag) queue[base + __popc(m & lane_lt_mask())] = idx;
}

// Add sign * (count, count*x, count*|x|^2) of one point to cluster k: light
// points go to the block's u32 accumulators (flushed every tile), heavy ones
// straight to the global int64 moments.
__device__ __forceinline__ void accumulate(uint32_t *acc, Moments *mom, int k, uint32_t cnt,
                                           uint32_t r, uint32_t g, uint32_t b, int sign) {
    const uint32_t qq = r * r + g * g + b * b;
    if (cnt < kHeavyCount) {
        const uint32_t q = cnt * qq;
        uint32_t *a = acc + k * kAccPerCluster;
        const uint32_t sg = (uint32_t)sign;
        atomicAdd(a + 0, sg * cnt);
        atomicAdd(a + 1, sg * cnt * r);
        atomicAdd(a + 2, sg * cnt * g);
        atomicAdd(a + 3, sg * cnt * b);
        atomicAdd(a + 4, sg * (q & 0xFFFFu));
        atomicAdd(a + 5, sg * (q >> 16));
    } else {
        const long long sc = (long long)sign * (long long)cnt;
        atomicAdd(&mom[k].n, (unsigned long long)sc);
        atomicAdd((unsigned long long *)&mom[k].s[0], (unsigned long long)(sc * (long long)r));
        atomicAdd((unsigned long long *)&mom[k].s[1], (unsigned long long)(sc * (long long)g));
        atomicAdd((unsigned long long *)&mom[k].s[2], (unsigned long long)(sc * (long long)b));
        atomicAdd(&mom[k].q, (unsigned long long)(sc * (long long)qq));
    }
}

// global-atomic version (replay / repair paths)
__device__ __forceinline__ void accumulate_global(Moments *mom, int k, uint32_t cnt, uint32_t r,
                                                  uint32_t g, uint32_t b, int sign) {
    const long long sc = (long long)sign * (long long)cnt;
    const long long qq = (long long)(r * r + g * g + b * b);
    atomicAdd(&mom[k].n, (unsigned long long)sc);
    atomicAdd((unsigned long long *)&mom[k].s[0], (unsigned long long)(sc * (long long)r));
    atomicAdd((unsigned long long *)&mom[k].s[1], (unsigned long long)(sc * (long long)g));
    atomicAdd((unsigned long long *)&mom[k].s[2], (unsigned long long)(sc * (long long)b));
    atomicAdd(&mom[k].q, (unsigned long long)(sc * qq));
}

// Flush the block accumulators (interpreted as signed 32-bit partial sums;
// at most 2048 light points per flush keeps every partial below 2^31).
__device__ __forceinline__ void flush_acc(uint32_t *acc, Moments *mom, int K) {
    for (int e = threadIdx.x; e < K * kAccPerCluster; e += blockDim.x) {
        const int v = (int)acc[e];
        if (v != 0) {
            const int k = e / kAccPerCluster, f = e - k * kAccPerCluster;
            const long long lv = (long long)v;
            unsigned long long *dst;
            long long add = lv;
            switch (f) {
                case 0: dst = &mom[k].n; break;
                case 1: dst = (unsigned long long *)&mom[k].s[0]; break;
                case 2: dst = (unsigned long long *)&mom[k].s[1]; break;
                case 3: dst = (unsigned long long *)&mom[k].s[2]; break;
                case 4: dst = &mom[k].q; break;
                default: dst = &mom[k].q; add = lv * 65536; break;
            }
            atomicAdd(dst, (unsigned long long)add);
            acc[e] = 0;
        }
    }
}

// NDC of assign_point_sortmeans for point x with previous label prev
// (kmeans.cpp:56-79): 1 + #{walk positions j >= 1 : D[prev][order[j]] < 4*d2(x,c_prev)}.
// Rows are sorted ascending after the self-first rotation, so this is a
// lower_bound in exact FP64.
__device__ __forceinline__ uint32_t walk_ndc(double xr, double xg, double xb, int prev,
                                             const double *cen, const double *dsorted, int K) {
    const double pd = d2_exact(xr, xg, xb, cen[3 * prev], cen[3 * prev + 1], cen[3 * prev + 2]);
    const double cutoff = __dmul_rn(4.0, pd);
    const double *row = dsorted + (size_t)prev * K;
    int lo = 1, hi = K;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(row + mid) < cutoff) lo = mid + 1;
        else hi = mid;
    }
    return (uint32_t)lo; // 1 + (lo - 1)
}

// ---------------------------------------------------------------------------
// The sweep kernel. PPT points per thread amortise the shared-memory centre
// loads (one LDS.128 per 4 centres per operand array).
template <int MODE, int PPT>
__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(SweepArgs a) {
    extern __shared__ __align__(16) float smem[];
    const int K = a.K, Kp = a.Kp;
    float *s_m2r = smem, *s_m2g = smem + Kp, *s_m2b = smem + 2 * Kp, *s_cc = smem + 3 * Kp;
    uint32_t *s_acc = reinterpret_cast<uint32_t *>(smem + 4 * Kp);
    for (int i = threadIdx.x; i < 4 * Kp; i += blockDim.x) smem[i] = a.fc[i];
    for (int i = threadIdx.x; i < K * kAccPerCluster; i += blockDim.x) s_acc[i] = 0;
    __syncthreads();
    const float tau_abs = a.tau[0], tau_rel = a.tau[1];
    unsigned long long ndc_local = 0;

    const uint64_t tile = (uint64_t)kSweepThreads * PPT;
    for (uint64_t base = (uint64_t)blockIdx.x * tile; base < a.n; base += (uint64_t)gridDim.x * tile) {
        float2 xr2[PPT], xg2[PPT], xb2[PPT], xx2[PPT];
        uint32_t col[PPT];
        int b1[PPT], b2[PPT];
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const uint64_t idx = base + threadIdx.x + (uint64_t)i * kSweepThreads;
            col[i] = idx < a.n ? __ldg(a.colors + idx) : 0u;
            const float r = (float)((col[i] >> 16) & 255u), g = (float)((col[i] >> 8) & 255u),
                        b = (float)(col[i] & 255u);
            const float xx = r * r + g * g + b * b; // exact: integers < 2^18
            xr2[i] = make_float2(r, r);
            xg2[i] = make_float2(g, g);
            xb2[i] = make_float2(b, b);
            xx2[i] = make_float2(xx, xx);
            b1[i] = 0x7FFFFFFF;
            b2[i] = 0x7FFFFFFF;
        }
#pragma unroll 2
        for (int j = 0; j < Kp; j += 4) {
            const float4 r4 = *reinterpret_cast<const float4 *>(s_m2r + j);
            const float4 g4 = *reinterpret_cast<const float4 *>(s_m2g + j);
            const float4 b4 = *reinterpret_cast<const float4 *>(s_m2b + j);
            const float4 c4 = *reinterpret_cast<const float4 *>(s_cc + j);
            const float2 rlo = make_float2(r4.x, r4.y), rhi = make_float2(r4.z, r4.w);
            const float2 glo = make_float2(g4.x, g4.y), ghi = make_float2(g4.z, g4.w);
            const float2 blo = make_float2(b4.x, b4.y), bhi = make_float2(b4.z, b4.w);
            const float2 clo = make_float2(c4.x, c4.y), chi = make_float2(c4.z, c4.w);
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                float2 A = __fadd2_rn(clo, xx2[i]);
                A = __ffma2_rn(xr2[i], rlo, A);
                A = __ffma2_rn(xg2[i], glo, A);
                A = __ffma2_rn(xb2[i], blo, A);
                float2 B = __fadd2_rn(chi, xx2[i]);
                B = __ffma2_rn(xr2[i], rhi, B);
                B = __ffma2_rn(xg2[i], ghi, B);
                B = __ffma2_rn(xb2[i], bhi, B);
                const int k0 = (__float_as_int(A.x) & ~0xFF) | j;
                const int k1 = (__float_as_int(A.y) & ~0xFF) | (j + 1);
                const int k2 = (__float_as_int(B.x) & ~0xFF) | (j + 2);
                const int k3 = (__float_as_int(B.y) & ~0xFF) | (j + 3);
                int lo = min(k0, k1), hi = max(k0, k1);
                b2[i] = min(min(b2[i], hi), max(b1[i], lo));
                b1[i] = min(b1[i], lo);
                lo = min(k2, k3);
                hi = max(k2, k3);
                b2[i] = min(min(b2[i], hi), max(b1[i], lo));
                b1[i] = min(b1[i], lo);
            }
        }
        // resolve
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const uint64_t idx = base + threadIdx.x + (uint64_t)i * kSweepThreads;
            const bool valid = idx < a.n;
            const int j1 = b1[i] & 0xFF;
            const float f1 = __int_as_float(b1[i] & ~0xFF), f2 = __int_as_float(b2[i] & ~0xFF);
            const bool flag = valid && !((f2 - f1) > tau_abs + tau_rel * (fabsf(f1) + fabsf(f2)));
            const uint32_t r = (col[i] >> 16) & 255u, g = (col[i] >> 8) & 255u, b = col[i] & 255u;
            if (MODE == MODE_WALK && valid) {
                const int prev = (int)a.labels[idx];
                ndc_local += walk_ndc((double)r, (double)g, (double)b, prev, a.cen, a.dsorted, K);
                if (!flag && j1 != prev) {
                    const uint32_t cnt = __ldg(a.counts + idx);
                    a.labels[idx] = (uint32_t)j1;
                    accumulate(s_acc, a.mom, j1, cnt, r, g, b, +1);
                    accumulate(s_acc, a.mom, prev, cnt, r, g, b, -1);
                }
            } else if (valid && !flag) {
                const uint32_t cnt = __ldg(a.counts + idx);
                if (MODE == MODE_FULL) a.labels[idx] = (uint32_t)j1;
                else a.lut8[col[i]] = (uint8_t)j1;
                accumulate(s_acc, a.mom, j1, cnt, r, g, b, +1);
            }
            enqueue(flag, (uint32_t)idx, a.queue, a.qn);
        }
        __syncthreads();
        flush_acc(s_acc, a.mom, K);
        __syncthreads();
    }
    if (MODE == MODE_WALK) {
        for (int o = 16; o; o >>= 1) ndc_local += __shfl_xor_sync(0xffffffffu, ndc_local, o);
        if ((threadIdx.x & 31) == 0 && ndc_local) atomicAdd(a.ndc, ndc_local);
    }
}

// ---------------------------------------------------------------------------
// Wide variant for K > 256 (index does not fit in 8 mantissa bits): separate
// value/index tracking, one centre at a time.
template <int MODE>
__global__ void __launch_bounds__(kSweepThreads) sweep_wide_kernel(SweepArgs a) {
    extern __shared__ __align__(16) float smem[];
    const int K = a.K, Kp = a.Kp;
    float *s_m2r = smem, *s_m2g = smem + Kp, *s_m2b = smem + 2 * Kp, *s_cc = smem + 3 * Kp;
    uint32_t *s_acc = reinterpret_cast<uint32_t *>(smem + 4 * Kp);
    for (int i = threadIdx.x; i < 4 * Kp; i += blockDim.x) smem[i] = a.fc[i];
    for (int i = threadIdx.x; i < K * kAccPerCluster; i += blockDim.x) s_acc[i] = 0;
    __syncthreads();
    const float tau_abs = a.tau[0], tau_rel = a.tau[1];
    unsigned long long ndc_local = 0;
    int since_flush = 0;
    for (uint64_t base = (uint64_t)blockIdx.x * kSweepThreads; base < a.n;
         base += (uint64_t)gridDim.x * kSweepThreads) {
        const uint64_t idx = base + threadIdx.x;
        const bool valid = idx < a.n;
        const uint32_t c = valid ? __ldg(a.colors + idx) : 0u;
        const uint32_t r = (c >> 16) & 255u, g = (c >> 8) & 255u, b = c & 255u;
        const float fr = (float)r, fg = (float)g, fb = (float)b;
        const float xx = fr * fr + fg * fg + fb * fb;
        float v1 = 3.0e38f, v2 = 3.0e38f;
        int j1 = 0;
        for (int j = 0; j < K; ++j) {
            float d = s_cc[j] + xx;
            d = fmaf(fr, s_m2r[j], d);
            d = fmaf(fg, s_m2g[j], d);
            d = fmaf(fb, s_m2b[j], d);
            v2 = fminf(v2, fmaxf(v1, d));
            if (d < v1) j1 = j;
            v1 = fminf(v1, d);
        }
        const bool flag = valid && !((v2 - v1) > tau_abs + tau_rel * (fabsf(v1) + fabsf(v2)));
        if (MODE == MODE_WALK && valid) {
            const int prev = (int)a.labels[idx];
            ndc_local += walk_ndc((double)r, (double)g, (double)b, prev, a.cen, a.dsorted, K);
            if (!flag && j1 != prev) {
                const uint32_t cnt = __ldg(a.counts + idx);
                a.labels[idx] = (uint32_t)j1;
                accumulate(s_acc, a.mom, j1, cnt, r, g, b, +1);
                accumulate(s_acc, a.mom, prev, cnt, r, g, b, -1);
            }
        } else if (valid && !flag) {
            const uint32_t cnt = __ldg(a.counts + idx);
            if (MODE == MODE_FULL) a.labels[idx] = (uint32_t)j1;
            else a.lut32[c] = (uint32_t)j1;
            accumulate(s_acc, a.mom, j1, cnt, r, g, b, +1);
        }
        enqueue(flag, (uint32_t)idx, a.queue, a.qn);
        if (++since_flush == 8) { // flush every 2048 points
            since_flush = 0;
            __syncthreads();
            flush_acc(s_acc, a.mom, K);
            __syncthreads();
        }
    }
    __syncthreads();
    flush_acc(s_acc, a.mom, K);
    if (MODE == MODE_WALK) {
        for (int o = 16; o; o >>= 1) ndc_local += __shfl_xor_sync(0xffffffffu, ndc_local, o);
        if ((threadIdx.x & 31) == 0 && ndc_local) atomicAdd(a.ndc, ndc_local);
    }
}

// ---------------------------------------------------------------------------
// Exact FP64 replay of the reference's assignment for queued (near-tie) points.
//   FULL / MAP: nearest_full (kmeans.cpp:40-54): strict <, lowest index wins.
//   WALK: assign_point_sortmeans (kmeans.cpp:56-79) from the previous label.
template <int MODE>
__global__ void replay_kernel(SweepArgs a) {
    const uint32_t nq = *a.qn;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
        const uint32_t idx = a.queue[q];
        const uint32_t c = a.colors[idx], cnt = a.counts[idx];
        const uint32_t r = (c >> 16) & 255u, g = (c >> 8) & 255u, b = c & 255u;
        const double xr = (double)r, xg = (double)g, xb = (double)b;
        const int K = a.K;
        if (MODE == MODE_WALK) {
            const int prev = (int)a.labels[idx];
            const double *drow = a.dtab + (size_t)prev * K;
            const uint32_t *orow = a.order + (size_t)prev * K;
            const double pd = d2_exact(xr, xg, xb, a.cen[3 * prev], a.cen[3 * prev + 1], a.cen[3 * prev + 2]);
            const double cutoff = __dmul_rn(4.0, pd);
            double bd = pd;
            int best = prev;
            for (int j = 1; j < K; ++j) {
                const uint32_t t = orow[j];
                if (drow[t] >= cutoff) break;
                const double d = d2_exact(xr, xg, xb, a.cen[3 * t], a.cen[3 * t + 1], a.cen[3 * t + 2]);
                if (d < bd) {
                    bd = d;
                    best = (int)t;
                }
            }
            if (best != prev) {
                a.labels[idx] = (uint32_t)best;
                accumulate_global(a.mom, best, cnt, r, g, b, +1);
                accumulate_global(a.mom, prev, cnt, r, g, b, -1);
            }
        } else {
            double bd = d2_exact(xr, xg, xb, a.cen[0], a.cen[1], a.cen[2]);
            int best = 0;
            for (int j = 1; j < K; ++j) {
                const double d = d2_exact(xr, xg, xb, a.cen[3 * j], a.cen[3 * j + 1], a.cen[3 * j + 2]);
                if (d < bd) {
                    bd = d;
                    best = j;
                }
            }
            if (MODE == MODE_FULL) a.labels[idx] = (uint32_t)best;
            else if (a.lut8) a.lut8[c] = (uint8_t)best;
            else a.lut32[c] = (uint32_t)best;
            accumulate_global(a.mom, best, cnt, r, g, b, +1);
        }
    }
}

// FP32 centre table + error bound for the sweep (one block).
//   E <= u*|cc err| + u*|m2c err|*x + 4u*M  with u = 2^-24 and M the largest
//   magnitude of any partial sum (cc + xx when all coordinates are >= 0).
__global__ void fc_kernel(const double *cen, int K, int Kp, float *fc, float *tau);

// K x K centre distances, per-row walk order (sorted by (d, index), self first:
// kmeans.cpp:14-38) and the rows' distances in walk order.
__global__ void table_kernel(const double *cen, int K, double *dtab, double *dsorted, uint32_t *order);

size_t sweep_smem_bytes(int K, int Kp);
void launch_sweep(cqg_ctx *ctx, int mode, const SweepArgs &a);

} // namespace cqg
