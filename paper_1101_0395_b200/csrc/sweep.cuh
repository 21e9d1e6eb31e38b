// sweep.cuh -- the FP32 nearest-centre sweep shared by the Lloyd assignment
// (iteration 1: nearest_full, iteration >= 2: assign_point_sortmeans) and the
// palette mapping (nearest_pruned_lowest_index).
//
// Per (unique colour x, centre c) the sweep evaluates the expanded form
//     d = (|c|^2 + |x|^2) - 2 x.c
// as FADD2 + 3 FFMA2 on float pairs (two centres per instruction) and keeps
// the best and the
// second-best value with 3-input float min/max (FMNMX3). The result is exact
// whenever the best/second gap exceeds a rigorous bound on the FP32 error
// (tau, computed per iteration from the centre magnitudes); otherwise the
// point is queued and replayed in FP64 with the reference's own walk
// (replay kernels), so labels are bit-exact with the reference.
#pragma once

#include "cqg_internal.cuh"

namespace cqg {

constexpr int kSweepThreads = 256;
#ifndef CQG_GROUP
#define CQG_GROUP 8 // centres per min-chain group of the sweep (build-time experiment knob)
#endif
constexpr int kAccPerCluster = 6; // n, s_r, s_g, s_b, q_lo16, q_hi
constexpr uint32_t kHeavyCount = 2048; // counts >= this bypass the u32 smem accumulators

// MAPW: the mapping sweep of the substrate Lloyd just ran on, pruned by its
// distance bounds (palette = the final centres): labels are read, never
// written; moments start from Lloyd's final ones and take +new -old deltas.
enum { MODE_FULL = 0, MODE_WALK = 1, MODE_MAP = 2, MODE_MAPW = 3 };
// modes that keep u64 moment deltas and run the bound filter
__host__ __device__ constexpr bool mode_delta(int m) { return m == MODE_WALK || m == MODE_MAPW; }

// Shared-memory layout of the FP32 centre table (Kp = pad_centres(K)):
//   m2r[Kp], m2g[Kp], m2b[Kp], cc[Kp]  (m2* = -2 * centre, cc = |centre|^2)
// Padding centres have cc = 1e30 and never win.

// centres per FP32 table row: K rounded up to the sweep's group size
// (measured on B200, cfg3 dense sweep: 8-centre groups 40.7 TFLOP/s, 16-centre
// groups 34.6 / 33.4 with one / two groups per unrolled step)
__host__ __device__ constexpr int pad_centres(int K) { return (K + CQG_GROUP - 1) / CQG_GROUP * CQG_GROUP; }

struct SweepArgs {
    const uint32_t *colors;
    const uint32_t *counts;
    uint64_t n;
    uint32_t *labels;       // FULL/WALK: per-point label (WALK reads prev, writes new)
    uint8_t *lut8;          // MAP, K <= 256: 2^24 LUT colour -> label
    uint32_t *lut32;        // MAP, K > 256
    uint8_t *maplab8;       // MAP: the label per distinct colour, in substrate order (K <= 256), or null
    uint32_t *maplab32;     // MAP, K > 256
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
    int Kpow; // dsorted row stride: next power of two >= K
    // Distance-bound pruning (WALK/FULL; null = off): per point (ub, lb) with
    // ub >= d(x, c_label) and lb <= min_{j != label} d(x, c_j) (Euclidean,
    // directed rounding); shift = K per-centre moves since the bounds were
    // written + {max, second max, argmax bits}; swept counts the points that
    // went through the full centre loop.
    float2 *bnd;
    const float *shift;
    unsigned long long *swept;
    const uint16_t *dcode; // K x Kpow 16-bit monotone codes of dsorted (ndc_code_kernel), or null
    // persistent Lloyd kernel (no walk table inside the loop): rowmin[k] =
    // min_{j != k} D[k][j] for the stay test (else dsorted[k][1]); lab_snap
    // receives every point's label as the filter reads it (deferred NDC)
    const double *rowmin;
    uint16_t *lab_snap;
    // the caller filled the stay test's shared terms (s_aux: shift[K], 2s[K],
    // max shift, second max, argmax bits) itself
    int aux_ready;
    // the caller flushes the u32 shared accumulators once after the sweep
    // (its whole range has at most 2048 points, so no partial sum can overflow)
    int flush_at_end;
    // WALK with bounds on large substrates: survivor list (n entries + a
    // counter at n + 4) for filter_list_kernel / sweep_list_kernel, or null
    uint32_t *surv;
};

// mapping result of distinct colour idx (colour c): the LUT the pixel pass
// reads, and the label in substrate order the mapping-NDC pass reads
__device__ __forceinline__ void map_store(const SweepArgs &a, uint32_t c, uint64_t idx, uint32_t label) {
    if (a.lut8) {
        a.lut8[c] = (uint8_t)label;
        if (a.maplab8) a.maplab8[idx] = (uint8_t)label;
    } else {
        a.lut32[c] = label;
        if (a.maplab32) a.maplab32[idx] = label;
    }
}

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
    // word f of cluster k goes to Moments field min(f, 4) (n, s_r, s_g, s_b, q);
    // word 5 holds q's high part (x 65536). Branch-free addressing.
    unsigned long long *m64 = reinterpret_cast<unsigned long long *>(mom);
    for (int e = threadIdx.x; e < K * kAccPerCluster; e += blockDim.x) {
        const int v = (int)acc[e];
        if (v != 0) {
            const int k = e / kAccPerCluster, f = e - k * kAccPerCluster;
            const long long lv = (long long)v * (f == 5 ? 65536 : 1);
            atomicAdd(m64 + 5 * k + (f < 4 ? f : 4), (unsigned long long)lv);
            acc[e] = 0;
        }
    }
}

// NDC of assign_point_sortmeans for point x with previous label prev
// (kmeans.cpp:56-79): 1 + #{walk positions j >= 1 : D[prev][order[j]] < 4*d2(x,c_prev)}.
// Each row of dsorted holds the row's distances in walk order (ascending: the
// self distance 0 first), padded with +inf to Kpow = next power of two >= K.
// Binary lifting counts the entries < cutoff without branches; position 0 (the
// self entry, 0) counts iff cutoff > 0.
__device__ __forceinline__ uint32_t walk_positions(double cut, const double *row, int Kpow) {
    int pos = 0;
    for (int step = Kpow >> 1; step >= 1; step >>= 1)
        if (__ldg(row + pos + step - 1) < cut) pos += step;
    if (pos == Kpow - 1 && __ldg(row + Kpow - 1) < cut) pos = Kpow; // whole row below
    return (uint32_t)(pos - (cut > 0.0 ? 1 : 0)) + 1u; // positions visited: 0..ret-1
}

// Warp-cooperative version (all 32 lanes, same row/cutoff): a 32-ary search,
// two dependent loads for Kpow <= 1024.
__device__ __forceinline__ uint32_t walk_positions_warp(double cut, const double *row, int Kpow) {
    const int lane = threadIdx.x & 31;
    int base = 0, span = Kpow;
    while (span > 1) {
        const int S = span >= 32 ? span / 32 : 1; // stride between probes
        const int probes = span >= 32 ? 32 : span;
        const int p = base + (lane + 1) * S - 1;
        const bool lt = lane < probes && __ldg(row + p) < cut;
        const int c = __popc(__ballot_sync(0xffffffffu, lt));
        base += c * S;
        span = S;
        if (c == probes) break; // everything probed is below the cutoff
    }
    return (uint32_t)(base - (cut > 0.0 ? 1 : 0)) + 1u;
}

__device__ __forceinline__ uint32_t walk_ndc(double xr, double xg, double xb, int prev,
                                             const double *cen, const double *dsorted, int K, int Kpow) {
    const double pd = d2_exact(xr, xg, xb, cen[3 * prev], cen[3 * prev + 1], cen[3 * prev + 2]);
    return walk_positions(__dmul_rn(4.0, pd), dsorted + (size_t)prev * Kpow, Kpow);
}

// 16-bit monotone code of a non-negative double v: its round-down FP32 value
// with the exponent restricted to the window [2^-8, 2^24) (5 bits) and the top
// 11 mantissa bits (relative bucket width 2^-11). Squared colour distances and
// cutoffs lie below 2^20, so nothing real saturates at the top; values below
// 2^-8 (0 included) share code 0, +inf and padding map to 0xFFFF. Monotone,
// so code(D) < code(cut) implies D < cut and code(D) > code(cut) implies
// D >= cut; equal codes need the FP64 values. (The plain top half of the FP32
// bits, 7 mantissa bits, tied 16x more often: measured on cfg5, the NDC
// kernel spent 29% of its samples in the FP64 tie loop.)
__device__ __forceinline__ uint32_t code16(double v) {
    const uint32_t b = __float_as_uint(__double2float_rd(v));
    const int e = (int)(b >> 23) - (127 - 8);
    if (e < 0) return 0u;
    if (e > 31) return 0xFFFFu;
    return ((uint32_t)e << 11) | ((b >> 12) & 0x7FFu);
}

// NDC with the walk rows as 16-bit codes in shared memory (K <= 256): the
// branch-free lifting runs on shared memory (a few bank-conflict wavefronts
// per warp step instead of 32 L1 lines); only a code tie with the cutoff reads
// the FP64 row. One 1024-thread block per SM, 4 points per thread in flight.
constexpr int kNdcCodeMaxK = 256;
template <int Q>
static __global__ void __launch_bounds__(1024, 1) ndc_code_kernel(const uint32_t *__restrict__ colors,
                                                                   const uint32_t *__restrict__ labels, uint64_t n,
                                                                   const double *__restrict__ cen,
                                                                   const double *__restrict__ dsorted,
                                                                   const uint16_t *__restrict__ dcode, int K,
                                                                   int Kpow, unsigned long long *ndc) {
    extern __shared__ __align__(16) double s_cenc[];
    // rows padded by one 32-bit word: row r, position p lands in bank
    // (r + p / 2) mod 32, so a warp searching different rows spreads over the
    // banks (an unpadded 2^m-byte stride puts position p of every row in one bank)
    const int rs = Kpow + 2; // row stride in codes
    uint16_t *s_code = reinterpret_cast<uint16_t *>(s_cenc + 3 * K);
    for (int i = threadIdx.x; i < 3 * K; i += blockDim.x) s_cenc[i] = cen[i];
    if (Kpow >= 2) {
        const int hw = Kpow / 2; // 32-bit words per row
        const uint32_t *src = reinterpret_cast<const uint32_t *>(dcode);
        uint32_t *dst = reinterpret_cast<uint32_t *>(s_code);
        const int total = K * hw;
        // 8 loads in flight per thread (clamped source, masked store)
        for (int i0 = threadIdx.x; i0 < total; i0 += 8 * blockDim.x) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                v[u] = __ldg(src + (i < total ? i : 0));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < total) {
                    const int r = i / hw, w = i - r * hw;
                    dst[r * (hw + 1) + w] = v[u];
                }
            }
        }
    } else {
        for (int r = threadIdx.x; r < K; r += blockDim.x) s_code[r * rs] = dcode[r];
    }
    __syncthreads();
    unsigned long long local = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * Q;
    // software-pipelined: the next batch's colours and labels are loaded
    // (clamped, branch-free) while this batch runs its lifting
    uint32_t ncol[Q], nlab[Q];
    auto load_batch = [&](uint64_t b) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = b + threadIdx.x + (uint64_t)q * blockDim.x;
            const uint64_t ic = i < n ? i : 0;
            ncol[q] = __ldg(colors + ic);
            nlab[q] = __ldg(labels + ic);
        }
    };
    uint64_t base = (uint64_t)blockIdx.x * blockDim.x * Q;
    if (base < n) load_batch(base);
    for (; base < n; base += stride) {
        double cut[Q];
        uint32_t cc[Q];
        int prow[Q], pos[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = base + threadIdx.x + (uint64_t)q * blockDim.x;
            const bool v = i < n;
            const uint32_t col = ncol[q];
            const int prev = v ? (int)nlab[q] : 0;
            const double pd = d2_exact((double)((col >> 16) & 255u), (double)((col >> 8) & 255u),
                                       (double)(col & 255u), s_cenc[3 * prev], s_cenc[3 * prev + 1],
                                       s_cenc[3 * prev + 2]);
            cut[q] = v ? __dmul_rn(4.0, pd) : -1.0;
            cc[q] = v ? code16(cut[q]) : 0u; // invalid: code 0 counts nothing below
            prow[q] = prev;
            pos[q] = 0;
        }
        if (base + stride < n) load_batch(base + stride);
        for (int step = Kpow >> 1; step >= 1; step >>= 1) {
            uint32_t vv[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) vv[q] = s_code[prow[q] * rs + pos[q] + step - 1];
#pragma unroll
            for (int q = 0; q < Q; ++q) pos[q] += vv[q] < cc[q] ? step : 0;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (cut[q] < 0.0) continue;
            int p = pos[q];
            const uint16_t *row = s_code + prow[q] * rs;
            if (p == Kpow - 1 && row[Kpow - 1] < cc[q]) p = Kpow; // whole row below
            // entries whose code equals the cutoff's: decide with the FP64 values
            while (p < Kpow && row[p] == cc[q] && __ldg(dsorted + (size_t)prow[q] * Kpow + p) < cut[q]) ++p;
            local += (unsigned long long)(p - (cut[q] > 0.0 ? 1 : 0) + 1);
        }
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(ndc, local);
}

// NDC of one WALK iteration, before the sweep rewrites the labels: 4 points per
// thread with their lifting searches interleaved (independent loads in flight).
// NDC over points [lo, hi) with a thread stride of blockDim.x (per-block range
// in the persistent kernel, the whole grid range in ndc_kernel).
template <int Q>
__device__ __forceinline__ unsigned long long ndc_range(const uint32_t *__restrict__ colors,
                                                        const uint32_t *__restrict__ labels, uint64_t lo,
                                                        uint64_t hi, uint64_t first, uint64_t stride,
                                                        const double *c, const double *__restrict__ dsorted,
                                                        int Kpow) {
    unsigned long long local = 0;
    for (uint64_t base = lo + first; base < hi; base += stride) {
        double cut[Q];
        const double *row[Q];
        int pos[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = base + threadIdx.x + (uint64_t)q * blockDim.x;
            const bool v = i < hi;
            const uint32_t col = v ? __ldg(colors + i) : 0u;
            const int prev = v ? (int)labels[i] : 0;
            const double pd = d2_exact((double)((col >> 16) & 255u), (double)((col >> 8) & 255u),
                                       (double)(col & 255u), c[3 * prev], c[3 * prev + 1], c[3 * prev + 2]);
            cut[q] = v ? __dmul_rn(4.0, pd) : -1.0; // -1: counts nothing and adds 0 below
            row[q] = dsorted + (size_t)prev * Kpow;
            pos[q] = 0;
        }
        for (int step = Kpow >> 1; step >= 1; step >>= 1) {
            double vv[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) vv[q] = __ldg(row[q] + pos[q] + step - 1);
#pragma unroll
            for (int q = 0; q < Q; ++q) pos[q] += vv[q] < cut[q] ? step : 0;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            // lifting reaches at most Kpow-1: the whole row may lie below the cutoff
            if (pos[q] == Kpow - 1 && cut[q] >= 0.0 && __ldg(row[q] + Kpow - 1) < cut[q]) pos[q] = Kpow;
            if (cut[q] >= 0.0) local += (unsigned long long)(pos[q] - (cut[q] > 0.0 ? 1 : 0) + 1);
        }
    }
    return local;
}

// NDC over [lo, hi) with the first kNdcPrefix walk positions of every row as
// 16-bit codes in shared memory (s_pre: K rows, stride kNdcPrefix + 2). The
// count stays in shared memory unless kNdcPrefix or more entries lie below the
// cutoff (then the FP64 row is searched); code ties read the FP64 entries.
constexpr int kNdcPrefix = 64;
template <int Q>
__device__ __forceinline__ unsigned long long ndc_range_pre(const uint32_t *__restrict__ colors,
                                                            const uint32_t *__restrict__ labels, uint64_t lo,
                                                            uint64_t hi, uint64_t first, uint64_t stride,
                                                            const double *c, const double *__restrict__ dsorted,
                                                            int Kpow, const uint16_t *s_pre) {
    constexpr int rs = kNdcPrefix + 2;
    const int L = Kpow < kNdcPrefix ? Kpow : kNdcPrefix;
    unsigned long long local = 0;
    for (uint64_t base = lo + first; base < hi; base += stride) {
        double cut[Q];
        uint32_t cc[Q];
        int prow[Q], pos[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = base + threadIdx.x + (uint64_t)q * blockDim.x;
            const bool v = i < hi;
            const uint32_t col = v ? __ldg(colors + i) : 0u;
            const int prev = v ? (int)labels[i] : 0;
            const double pd = d2_exact((double)((col >> 16) & 255u), (double)((col >> 8) & 255u),
                                       (double)(col & 255u), c[3 * prev], c[3 * prev + 1], c[3 * prev + 2]);
            cut[q] = v ? __dmul_rn(4.0, pd) : -1.0;
            cc[q] = v ? code16(cut[q]) : 0u;
            prow[q] = prev;
            pos[q] = 0;
        }
        for (int step = L >> 1; step >= 1; step >>= 1) {
            uint32_t vv[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) vv[q] = s_pre[prow[q] * rs + pos[q] + step - 1];
#pragma unroll
            for (int q = 0; q < Q; ++q) pos[q] += vv[q] < cc[q] ? step : 0;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (cut[q] < 0.0) continue;
            const uint16_t *row = s_pre + prow[q] * rs;
            const double *grow = dsorted + (size_t)prow[q] * Kpow;
            int p = pos[q];
            if (p == L - 1 && row[L - 1] < cc[q]) p = L;
            while (p < L && row[p] == cc[q] && __ldg(grow + p) < cut[q]) ++p;
            if (p == L && L < Kpow) p = (int)walk_positions(cut[q], grow, Kpow) - 1 + (cut[q] > 0.0 ? 1 : 0);
            local += (unsigned long long)(p - (cut[q] > 0.0 ? 1 : 0) + 1);
        }
    }
    return local;
}

// NDC of a large substrate's WALK iteration with only the first kNdcPrefix walk
// positions of every row in shared memory (34 KB at K = 256 against 132 KB for
// whole rows): 4 blocks of 512 threads per SM instead of one of 1024, and a
// lifting of 6 steps instead of 8. A walk visits ~4 centres on average, so
// the FP64 row in L2 is searched for very few points.
template <int Q>
static __global__ void __launch_bounds__(512, 4) ndc_pre_kernel(const uint32_t *__restrict__ colors,
                                                                 const uint32_t *__restrict__ labels, uint64_t n,
                                                                 const double *__restrict__ cen,
                                                                 const double *__restrict__ dsorted,
                                                                 const uint16_t *__restrict__ dcode, int K, int Kpow,
                                                                 unsigned long long *ndc) {
    extern __shared__ __align__(16) double s_cenp[];
    constexpr int rs = kNdcPrefix + 2;
    uint16_t *s_pre = reinterpret_cast<uint16_t *>(s_cenp + 3 * K);
    const int L = Kpow < kNdcPrefix ? Kpow : kNdcPrefix;
    for (int i = threadIdx.x; i < 3 * K; i += blockDim.x) s_cenp[i] = cen[i];
    for (int e = threadIdx.x; e < K * L; e += blockDim.x) {
        const int r = e / L, p = e - r * L;
        s_pre[r * rs + p] = __ldg(dcode + (size_t)r * Kpow + p);
    }
    __syncthreads();
    unsigned long long local =
        ndc_range_pre<Q>(colors, labels, 0, n, (uint64_t)blockIdx.x * blockDim.x * Q,
                         (uint64_t)gridDim.x * blockDim.x * Q, s_cenp, dsorted, Kpow, s_pre);
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(ndc, local);
}

template <int Q>
static __global__ void __launch_bounds__(256, 4) ndc_kernel(const uint32_t *__restrict__ colors,
                                                  const uint32_t *__restrict__ labels, uint64_t n,
                                                  const double *__restrict__ cen,
                                                  const double *__restrict__ dsorted, int K, int Kpow,
                                                  unsigned long long *ndc) {
    extern __shared__ double s_cen[];
    const bool in_smem = K <= 2048;
    if (in_smem)
        for (int i = threadIdx.x; i < 3 * K; i += blockDim.x) s_cen[i] = cen[i];
    __syncthreads();
    const double *c = in_smem ? s_cen : cen;
    unsigned long long local =
        ndc_range<Q>(colors, labels, 0, n, (uint64_t)blockIdx.x * blockDim.x * Q,
                     (uint64_t)gridDim.x * blockDim.x * Q, c, dsorted, Kpow);
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(ndc, local);
}


// ---------------------------------------------------------------------------
// The sweep kernel. Each block owns a contiguous, equal share of the points
// (balanced across SMs); PPT points per thread amortise the shared-memory
// centre loads (one LDS.128 per 4 centres per operand array).
//
// The sweep ranks centres by e_j = |c_j|^2 - 2 c_j.x (three FMAs per distance;
// |x|^2 is the same for every centre of a point and is added back, rounded
// outward, only for the distance bounds).
// Per point, each 8-centre GROUP's minimum is formed with a 3-input float min
// chain (0.5 ALU op per distance); the group minima feed the best (b1) and the
// second-best (b2) over groups and the index of the group that last improved
// b1 (1.1 ALU ops per distance in all, against 2.5 for exact per-candidate
// top-2 tracking). The exact index and the winning group's own second value
// are recovered afterwards by recomputing that group's 8 distances with the
// identical FP operation sequence (bit-identical values): the index is the
// first that equals b1, and the true second-best is min(b2, group second).
constexpr int kGroup = CQG_GROUP;
#ifndef CQG_GROUP_UNROLL
#define CQG_GROUP_UNROLL 2
#endif
constexpr int kGroupUnroll = CQG_GROUP_UNROLL; // groups per unrolled step of the centre loop
#ifdef CQG_SWEEP_TIMING
// block 0: filter cycles, phase cycles, survivors, calls; list tiles (thread 0):
// point loads, centre loop, resolve
__device__ unsigned long long g_sweep_timing[8];
#define STIME(slot)                                                                  \
    do {                                                                             \
        if (LIST && blockIdx.x == 0 && threadIdx.x == 0) {                           \
            const unsigned long long _n = clock64();                                 \
            g_sweep_timing[slot] += _n - _tt;                                        \
            _tt = _n;                                                                \
        }                                                                            \
    } while (0)
#else
#define STIME(slot) \
    do {            \
    } while (0)
#endif
// u32 words of the sweep accumulators: u32 x kAccPerCluster (FULL/MAP) or u64 x 5 (WALK)
__host__ __device__ constexpr int sweep_acc_words(int K) {
    return K * kAccPerCluster > K * 10 ? K * kAccPerCluster : K * 10;
}
constexpr int kSmemCentres = 1024; // FP64 centres staged in shared memory up to this K

// Sweep points of this block against the FP32 centre table in shared memory
// (s_fc: m2r | m2g | m2b | cc, Kp each): slots [lo, hi), point index = the
// slot (LIST = false) or list[slot]. FULL/MAP flush the u32 shared
// accumulators after every tile (WALK / MAPW: signed deltas, +new -old).
template <int MODE, int PPT, bool LIST>
__device__ __forceinline__ void sweep_tiles(const SweepArgs &a, uint64_t lo, uint64_t hi, const uint32_t *list,
                                            float *smem, uint32_t *s_acc, float tau_abs, float tau_rel) {
    static_assert(PPT % 2 == 0, "points are processed in pairs");
    constexpr int PP = PPT / 2;
    const int K = a.K, Kp = a.Kp;
    float *s_m2r = smem, *s_m2g = smem + Kp, *s_m2b = smem + 2 * Kp, *s_cc = smem + 3 * Kp;
    // per-value error bound of the FP32 distances (tau_abs = 2E*1.0625 + 1e-3)
    const float ev = 0.5f * tau_abs;
    const uint64_t tile = (uint64_t)kSweepThreads * PPT;
    // slot of point i of this thread: contiguous per i across the block for
    // ranges (coalesced colour loads); thread-major for lists, so a partial
    // tile fills whole warps and the warps left without points skip the tile
    auto slot_of = [&](uint64_t base, int i) -> uint64_t {
        return LIST ? base + (uint64_t)threadIdx.x * PPT + i : base + threadIdx.x + (uint64_t)i * kSweepThreads;
    };
    for (uint64_t base = lo; base < hi; base += tile) {
        if (__any_sync(0xffffffffu, slot_of(base, 0) < hi)) {
#ifdef CQG_SWEEP_TIMING
        unsigned long long _tt = clock64();
#endif
        // point pairs: lane .x = point 2p, lane .y = point 2p+1 (FFMA2 with a
        // broadcast scalar centre operand evaluates one centre for both)
        float2 xr2[PP], xg2[PP], xb2[PP];
        uint32_t col[PPT];
        uint32_t pidx[PPT]; // point index (< 2^24 unique colours)
        // small tiles: the resolve's label and count issued with the colour
        // (one memory round trip per tile instead of two more per point)
        constexpr bool kPre = PPT <= 4;
        uint32_t plab[kPre ? PPT : 1], pcnt[kPre ? PPT : 1];
        float b1[PPT], b2[PPT];
        int g1[PPT];
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const uint64_t slot = slot_of(base, i);
            pidx[i] = slot < hi ? (LIST ? list[slot] : (uint32_t)slot) : 0u;
            col[i] = slot < hi ? __ldg(a.colors + pidx[i]) : 0u;
            if (kPre) {
                plab[kPre ? i : 0] = mode_delta(MODE) ? a.labels[pidx[i]] : 0u;
                pcnt[kPre ? i : 0] = __ldg(a.counts + pidx[i]);
            }
            const float r = (float)((col[i] >> 16) & 255u), g = (float)((col[i] >> 8) & 255u),
                        b = (float)(col[i] & 255u);
            // opaque copies: keep the floats resident instead of letting ptxas
            // rematerialise them from the packed colour inside the centre loop
            float rr = r, gg = g, bb = b;
            asm volatile("" : "+f"(rr), "+f"(gg), "+f"(bb));
            if (i & 1) {
                xr2[i / 2].y = rr; xg2[i / 2].y = gg; xb2[i / 2].y = bb;
            } else {
                xr2[i / 2].x = rr; xg2[i / 2].x = gg; xb2[i / 2].x = bb;
            }
            b1[i] = 3.0e38f;
            b2[i] = 3.0e38f;
            g1[i] = 0;
        }
        STIME(4);
#pragma unroll (kGroupUnroll)
        for (int j = 0; j < Kp; j += kGroup) {
            float gm[PPT]; // this group's minimum per point
#pragma unroll
            for (int i = 0; i < PPT; ++i) gm[i] = 3.0e38f;
#pragma unroll
            for (int q = 0; q < kGroup; q += 4) {
                const float4 r4 = *reinterpret_cast<const float4 *>(s_m2r + j + q);
                const float4 g4 = *reinterpret_cast<const float4 *>(s_m2g + j + q);
                const float4 b4 = *reinterpret_cast<const float4 *>(s_m2b + j + q);
                const float4 c4 = *reinterpret_cast<const float4 *>(s_cc + j + q);
#pragma unroll
                for (int p = 0; p < PP; ++p) {
                    float2 A0 = __ffma2_rn(xr2[p], make_float2(r4.x, r4.x), make_float2(c4.x, c4.x));
                    A0 = __ffma2_rn(xg2[p], make_float2(g4.x, g4.x), A0);
                    A0 = __ffma2_rn(xb2[p], make_float2(b4.x, b4.x), A0);
                    float2 A1 = __ffma2_rn(xr2[p], make_float2(r4.y, r4.y), make_float2(c4.y, c4.y));
                    A1 = __ffma2_rn(xg2[p], make_float2(g4.y, g4.y), A1);
                    A1 = __ffma2_rn(xb2[p], make_float2(b4.y, b4.y), A1);
                    float2 A2 = __ffma2_rn(xr2[p], make_float2(r4.z, r4.z), make_float2(c4.z, c4.z));
                    A2 = __ffma2_rn(xg2[p], make_float2(g4.z, g4.z), A2);
                    A2 = __ffma2_rn(xb2[p], make_float2(b4.z, b4.z), A2);
                    float2 A3 = __ffma2_rn(xr2[p], make_float2(r4.w, r4.w), make_float2(c4.w, c4.w));
                    A3 = __ffma2_rn(xg2[p], make_float2(g4.w, g4.w), A3);
                    A3 = __ffma2_rn(xb2[p], make_float2(b4.w, b4.w), A3);
                    gm[2 * p] = fminf(fminf(fminf(gm[2 * p], A0.x), A1.x), fminf(A2.x, A3.x));
                    gm[2 * p + 1] = fminf(fminf(fminf(gm[2 * p + 1], A0.y), A1.y), fminf(A2.y, A3.y));
                }
            }
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                const float lo = gm[i];
                g1[i] = lo < b1[i] ? j : g1[i]; // the first group reaching the final minimum
                b2[i] = fminf(b2[i], fmaxf(b1[i], lo));
                b1[i] = fminf(b1[i], lo);
            }
        }
        STIME(5);
        // resolve: larger tiles load every point's label and count here, all
        // in flight together (small tiles issued them with the colours)
        uint32_t rlab[kPre ? 1 : PPT], rcnt[kPre ? 1 : PPT];
        if (!kPre) {
#pragma unroll
            for (int i = 0; i < PPT; ++i) {
                rlab[kPre ? 0 : i] = mode_delta(MODE) ? a.labels[pidx[i]] : 0u;
                rcnt[kPre ? 0 : i] = __ldg(a.counts + pidx[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const uint32_t idx = pidx[i];
            const bool valid = slot_of(base, i) < hi;
            const float f1 = b1[i];
            // exact index: first centre of group g1 whose (bit-identical) value
            // is b1; the group's second value completes the second-best
            int j1;
            float f2;
            {
                const int g0 = g1[i];
                const float xr = (i & 1) ? xr2[i / 2].y : xr2[i / 2].x;
                const float xg = (i & 1) ? xg2[i / 2].y : xg2[i / 2].x;
                const float xb = (i & 1) ? xb2[i / 2].y : xb2[i / 2].x;
                // the group's 8 values, two centres per FFMA2 (per lane the same
                // operations as the sweep: bit-identical), 128-bit loads
                float dv[kGroup];
#pragma unroll
                for (int q = 0; q < kGroup; q += 4) {
                    const float4 c4 = *reinterpret_cast<const float4 *>(s_cc + g0 + q);
                    const float4 r4 = *reinterpret_cast<const float4 *>(s_m2r + g0 + q);
                    const float4 gq = *reinterpret_cast<const float4 *>(s_m2g + g0 + q);
                    const float4 bq = *reinterpret_cast<const float4 *>(s_m2b + g0 + q);
                    float2 A = __ffma2_rn(make_float2(xr, xr), make_float2(r4.x, r4.y), make_float2(c4.x, c4.y));
                    A = __ffma2_rn(make_float2(xg, xg), make_float2(gq.x, gq.y), A);
                    A = __ffma2_rn(make_float2(xb, xb), make_float2(bq.x, bq.y), A);
                    float2 B = __ffma2_rn(make_float2(xr, xr), make_float2(r4.z, r4.w), make_float2(c4.z, c4.w));
                    B = __ffma2_rn(make_float2(xg, xg), make_float2(gq.z, gq.w), B);
                    B = __ffma2_rn(make_float2(xb, xb), make_float2(bq.z, bq.w), B);
                    dv[q] = A.x;
                    dv[q + 1] = A.y;
                    dv[q + 2] = B.x;
                    dv[q + 3] = B.y;
                }
                int found = kGroup;
                float w1 = 3.0e38f, w2 = 3.0e38f;
#pragma unroll
                for (int q = kGroup - 1; q >= 0; --q) found = dv[q] == f1 ? q : found; // first match
#pragma unroll
                for (int q = 0; q < kGroup; ++q) {
                    w2 = fminf(w2, fmaxf(w1, dv[q]));
                    w1 = fminf(w1, dv[q]);
                }
                j1 = g0 + (found < kGroup ? found : 0);
                f2 = fminf(b2[i], w2);
            }
            const bool flag = valid && !((f2 - f1) > tau_abs + tau_rel * (fabsf(f1) + fabsf(f2)));
            if (MODE != MODE_MAP && MODE != MODE_MAPW && a.bnd && valid) {
                // new bounds for label j1 (flagged points: replayed, bounds void)
                // back from the xx-free values to squared distances, outward
                const float cr = (float)((col[i] >> 16) & 255u), cg = (float)((col[i] >> 8) & 255u),
                            cb = (float)(col[i] & 255u);
                const float xx = cr * cr + cg * cg + cb * cb; // exact
                const float d1 = __fadd_ru(f1, xx), d2 = __fadd_rd(f2, xx);
                const float ub = __fsqrt_ru(__fadd_ru(d1 > 0.f ? d1 : 0.f, ev));
                const float l2 = __fadd_rd(d2, -ev);
                const float lb = __fsqrt_rd(l2 > 0.f ? l2 : 0.f);
                a.bnd[idx] = flag ? make_float2(__int_as_float(0x7f800000), 0.f) : make_float2(ub, lb);
            }
            const uint32_t r = (col[i] >> 16) & 255u, g = (col[i] >> 8) & 255u, b = col[i] & 255u;
            if (mode_delta(MODE) && valid) {
                const int prev = kPre ? (int)plab[kPre ? i : 0] : (int)rlab[kPre ? 0 : i];
                if (MODE == MODE_MAPW && !flag) map_store(a, col[i], idx, (uint32_t)j1);
                if (!flag && j1 != prev) {
                    const uint32_t cnt = kPre ? pcnt[kPre ? i : 0] : rcnt[kPre ? 0 : i];
                    if (MODE == MODE_WALK) a.labels[idx] = (uint32_t)j1;
                    accumulate(s_acc, a.mom, j1, cnt, r, g, b, +1);
                    accumulate(s_acc, a.mom, prev, cnt, r, g, b, -1);
                }
            } else if (valid && !flag) {
                const uint32_t cnt = kPre ? pcnt[kPre ? i : 0] : rcnt[kPre ? 0 : i];
                if (MODE == MODE_FULL) a.labels[idx] = (uint32_t)j1;
                else map_store(a, col[i], idx, (uint32_t)j1);
                accumulate(s_acc, a.mom, j1, cnt, r, g, b, +1);
            }
            enqueue(flag, (uint32_t)idx, a.queue, a.qn);
        }
        STIME(6);
        } // warp has points
        // u32 shared partial sums, flushed every tile (the 64-bit shared
        // atomics they replace compile to CAS loops: 29% of the cfg5 WALK
        // sweep's stall samples)
        if (!a.flush_at_end) {
            __syncthreads();
            flush_acc(s_acc, a.mom, K);
            __syncthreads();
        }
    }
}

// Points per block-local chunk of the pruned WALK sweep (shared-memory list).
#ifndef CQG_PRUNE_CHUNK
#define CQG_PRUNE_CHUNK 4096
#endif
constexpr int kPruneChunk = CQG_PRUNE_CHUNK;
constexpr float kBoundMargin = 1.0e-3f; // Euclidean gap that keeps the FP64 reference order

// Stay test (exact): after the centres moved by shift[], the label is provably
// unchanged when ub' + margin < lb* with (directed rounding throughout)
//   ub' = ub + shift[label], or the own-centre distance recomputed here,
//   lb* = max(lb - max_{j != label} shift[j],          (Hamerly)
//             2 s(label) - ub')                        (Elkan: s = half the distance
//                                                       from c_label to its nearest centre,
//                                                       dsorted[label][1]).
// The reference picks the incumbent whenever it is the unique nearest centre
// (nearest_full and assign_point_sortmeans alike), so skipped points keep
// their labels and moments. s_aux = {shift[K], 2s[K]} in shared memory.
// Returns true when the point needs the full sweep.
__device__ __forceinline__ bool prune_needs_sweep(const SweepArgs &a, uint64_t i, uint32_t lab, float2 bd,
                                                  uint32_t c, const float *s_fc, const float *s_aux, int Kp,
                                                  float ev, float smax1, float smax2, int sarg,
                                                  bool keep_bounds = true) {
    const float sl = s_aux[lab];
    const float two_s = s_aux[a.K + lab];
    const float so = (int)lab == sarg ? smax2 : smax1;
    float ub = __fadd_ru(bd.x, sl);
    const float lbh = __fadd_rd(bd.y, -so);
    float lb = fmaxf(lbh, __fadd_rd(two_s, -ub));
    bool stay = __fadd_ru(ub, kBoundMargin) < lb;
    if (!stay) {
        // tighten ub with the own-centre FP32 distance (sweep operation order)
        const float r = (float)((c >> 16) & 255u), g = (float)((c >> 8) & 255u), b = (float)(c & 255u);
        const float xx = r * r + g * g + b * b;
        float e = __fmaf_rn(r, s_fc[lab], s_fc[3 * Kp + lab]);
        e = __fmaf_rn(g, s_fc[Kp + lab], e);
        e = __fmaf_rn(b, s_fc[2 * Kp + lab], e);
        const float d = __fadd_ru(e, xx);
        ub = __fsqrt_ru(__fadd_ru(d > 0.f ? d : 0.f, ev));
        lb = fmaxf(lbh, __fadd_rd(two_s, -ub));
        stay = __fadd_ru(ub, kBoundMargin) < lb;
    }
    if (stay && keep_bounds) a.bnd[i] = make_float2(ub, lb);
    return !stay;
}

// Shared words the pruned WALK sweep needs besides the list: shift[K], 2s[K].
__host__ __device__ constexpr int prune_aux_words(int K) { return 2 * K + 4; }
#ifndef CQG_FILTER_PPT
#define CQG_FILTER_PPT 8
#endif
constexpr int kFilterPPT = CQG_FILTER_PPT; // points per thread per filter step (loads in flight)

// Sweep points [lo, hi) of this block. WALK with bounds: per chunk, the stay
// test appends the points that may change label to a shared-memory list
// (s_list: list_cap + one big tile of entries); full PPT-point tiles are swept
// as soon as they fill, the remainder carries over to the next chunk, and the
// final remainder is swept in 2-point tiles. s_aux: prune_aux_words(K) floats.
template <int MODE, int PPT>
__device__ __forceinline__ void sweep_range(const SweepArgs &a, uint64_t lo, uint64_t hi, float *smem,
                                            uint32_t *s_acc, float tau_abs, float tau_rel,
                                            uint32_t *s_list = nullptr, uint32_t list_cap = kPruneChunk,
                                            float *s_aux = nullptr) {
    if (!mode_delta(MODE) || a.bnd == nullptr || s_list == nullptr) {
        sweep_tiles<MODE, PPT, false>(a, lo, hi, nullptr, smem, s_acc, tau_abs, tau_rel);
        return;
    }
    __shared__ uint32_t s_m;
    const int Kp = a.Kp, K = a.K;
    const float ev = 0.5f * tau_abs;
    if (!a.aux_ready) {
        // per-centre terms of the stay test: shift and 2 s (nearest other centre, walk position 1)
        for (int k = threadIdx.x; k < K; k += blockDim.x) {
            s_aux[k] = __ldg(a.shift + k);
            const double nearest = a.rowmin ? a.rowmin[k] : __ldg(a.dsorted + (size_t)k * a.Kpow + 1);
            s_aux[K + k] = K > 1 ? __fsqrt_rd(__double2float_rd(__dmul_rd(nearest, 1.0 - 0x1.0p-40)))
                                 : __int_as_float(0x7f800000);
        }
        if (threadIdx.x < 3) s_aux[2 * K + threadIdx.x] = __ldg(a.shift + K + threadIdx.x);
        __syncthreads();
    }
    const float smax1 = s_aux[2 * K], smax2 = s_aux[2 * K + 1];
    const int sarg = __float_as_int(s_aux[2 * K + 2]);
    constexpr uint32_t big = kSweepThreads * PPT;
    unsigned long long swept = 0;
    if (threadIdx.x == 0) s_m = 0;
    __syncthreads();
#ifdef CQG_SWEEP_TIMING
    unsigned long long _st0 = clock64(), _sf = 0;
#endif
    for (uint64_t cb = lo; cb < hi; cb += list_cap) {
        const uint64_t ce = cb + list_cap < hi ? cb + list_cap : hi;
        for (uint64_t i0 = cb; i0 < ce; i0 += (uint64_t)blockDim.x * kFilterPPT) {
            uint32_t lab[kFilterPPT], col[kFilterPPT];
            float2 bd[kFilterPPT];
#pragma unroll
            for (int f = 0; f < kFilterPPT; ++f) {
                const uint64_t i = i0 + threadIdx.x + (uint64_t)f * blockDim.x;
                const bool v = i < ce;
                lab[f] = v ? a.labels[i] : 0u;
                bd[f] = v ? a.bnd[i] : make_float2(0.f, 0.f);
                col[f] = v ? __ldg(a.colors + i) : 0u;
            }
            if (a.lab_snap) {
#pragma unroll
                for (int f = 0; f < kFilterPPT; ++f) {
                    const uint64_t i = i0 + threadIdx.x + (uint64_t)f * blockDim.x;
                    if (i < ce) a.lab_snap[i] = (uint16_t)lab[f];
                }
            }
#pragma unroll
            for (int f = 0; f < kFilterPPT; ++f) {
                const uint64_t i = i0 + threadIdx.x + (uint64_t)f * blockDim.x;
                const bool need = i < ce && prune_needs_sweep(a, i, lab[f], bd[f], col[f], smem, s_aux, Kp, ev, smax1,
                                                              smax2, sarg, MODE == MODE_WALK);
                if (MODE == MODE_MAPW && i < ce && !need) // provably keeps its label under the palette
                    map_store(a, col[f], i, lab[f]);
                const uint32_t m = __ballot_sync(0xffffffffu, need);
                if (m) {
                    const int leader = __ffs(m) - 1;
                    uint32_t pos = 0;
                    if ((int)(threadIdx.x & 31) == leader) pos = atomicAdd(&s_m, (uint32_t)__popc(m));
                    pos = __shfl_sync(0xffffffffu, pos, leader);
                    if (need) s_list[pos + __popc(m & lane_lt_mask())] = (uint32_t)i;
                }
            }
        }
        __syncthreads();
#ifdef CQG_SWEEP_TIMING
        _sf += clock64() - _st0;
#endif
        const uint32_t m = s_m;
        const uint32_t mb = m / big * big;
        if (mb) {
            sweep_tiles<MODE, PPT, true>(a, 0, mb, s_list, smem, s_acc, tau_abs, tau_rel);
            swept += mb;
            __syncthreads();
            // carry the remainder (< big entries) to the front: [mb, m) -> [0, m - mb), disjoint
            for (uint32_t t = threadIdx.x; t < m - mb; t += blockDim.x) s_list[t] = s_list[mb + t];
            __syncthreads();
            if (threadIdx.x == 0) s_m = m - mb;
        }
        __syncthreads();
    }
    const uint32_t rest = s_m;
    if (rest) sweep_tiles<MODE, 2, true>(a, 0, rest, s_list, smem, s_acc, tau_abs, tau_rel);
    swept += rest;
    __syncthreads();
#ifdef CQG_SWEEP_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        g_sweep_timing[0] += _sf;
        g_sweep_timing[1] += clock64() - _st0;
        g_sweep_timing[2] += swept;
        g_sweep_timing[3] += 1;
    }
#endif
    if (threadIdx.x == 0 && a.swept && swept) atomicAdd(a.swept, swept);
}

// Large substrates, WALK iterations with bounds: one light pass runs the stay
// test over every point (bounds of stayers rewritten) and appends the points
// that may change label to a global survivor list; sweep_list_kernel then
// sweeps only the list in full 8-point tiles, with no filter or list
// bookkeeping in the 128-register sweep. (The NDC stays in its own kernel:
// fused into this pass it made a 1-block-per-SM latency-bound kernel, 216 us
// against 109 + ~70 us separately on cfg5.) List order is irrelevant: every
// per-point result is deterministic and moments are integer sums.
constexpr int kFilterThreads = 256;
constexpr int kFilterQ = 8;
__host__ __device__ constexpr size_t filter_list_smem(int K, int Kp) {
    return (size_t)4 * Kp * 4 + (size_t)prune_aux_words(K) * 4;
}
static __global__ void __launch_bounds__(kFilterThreads) filter_list_kernel(SweepArgs a, uint32_t *list,
                                                                          uint32_t *listn) {
    extern __shared__ __align__(16) float s_ff[];
    __shared__ uint32_t s_wcnt[64]; // per-warp survivor counts, then each warp's first list slot
    const int K = a.K, Kp = a.Kp, Kpow = a.Kpow;
    float *s_fc = s_ff;              // 4 Kp
    float *s_aux = s_fc + 4 * Kp;    // 2K + 4
    for (int i = threadIdx.x; i < 4 * Kp; i += blockDim.x) s_fc[i] = a.fc[i];
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        s_aux[k] = __ldg(a.shift + k);
        s_aux[K + k] = K > 1 ? __fsqrt_rd(__double2float_rd(__dmul_rd(__ldg(a.dsorted + (size_t)k * Kpow + 1),
                                                                        1.0 - 0x1.0p-40)))
                             : __int_as_float(0x7f800000);
    }
    if (threadIdx.x < 3) s_aux[2 * K + threadIdx.x] = __ldg(a.shift + K + threadIdx.x);
    __syncthreads();
    const float ev = 0.5f * __ldg(a.tau);
    const float smax1 = s_aux[2 * K], smax2 = s_aux[2 * K + 1];
    const int sarg = __float_as_int(s_aux[2 * K + 2]);
    constexpr int Q = kFilterQ;
    const uint64_t n = a.n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * Q;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * Q; base < n; base += stride) {
        uint32_t col[Q], lab[Q];
        float2 bd[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = base + threadIdx.x + (uint64_t)q * blockDim.x;
            const uint64_t ic = i < n ? i : 0;
            col[q] = __ldg(a.colors + ic);
            lab[q] = a.labels[ic];
            bd[q] = a.bnd[ic];
        }
        // stay test; the batch's survivors are appended with ONE global atomic
        // per block (a per-warp atomic on the single counter serialised)
        uint32_t need = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = base + threadIdx.x + (uint64_t)q * blockDim.x;
            if (i < n && prune_needs_sweep(a, i, lab[q], bd[q], col[q], s_fc, s_aux, Kp, ev, smax1, smax2, sarg, true))
                need |= 1u << q;
        }
        uint32_t wm[Q], wc = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            wm[q] = __ballot_sync(0xffffffffu, (need >> q) & 1u);
            wc += __popc(wm[q]);
        }
        if (lane == 0) s_wcnt[warp] = wc;
        __syncthreads();
        if (warp == 0) {
            const uint32_t c = lane < (int)(blockDim.x >> 5) ? s_wcnt[lane] : 0u;
            uint32_t incl = c;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
            uint32_t b0 = 0;
            if (lane == 0 && tot) b0 = atomicAdd(listn, tot);
            b0 = __shfl_sync(0xffffffffu, b0, 0);
            s_wcnt[32 + lane] = b0 + incl - c; // each warp's first slot
        }
        __syncthreads();
        uint32_t slot = s_wcnt[32 + warp];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint64_t i = base + threadIdx.x + (uint64_t)q * blockDim.x;
            if ((need >> q) & 1u) list[slot + __popc(wm[q] & lane_lt_mask())] = (uint32_t)i;
            slot += __popc(wm[q]);
        }
        __syncthreads(); // s_wcnt is rewritten by the next batch
    }
}

// The survivor list of filter_list_kernel, swept in full PPT-point tiles
// (blocks stride over the tiles; the count is read on the device).
template <int PPT>
static __global__ void __launch_bounds__(kSweepThreads, 2) sweep_list_kernel(SweepArgs a, const uint32_t *list,
                                                                             const uint32_t *listn) {
    extern __shared__ __align__(16) float smem[];
    const int K = a.K, Kp = a.Kp;
    uint32_t *s_acc = reinterpret_cast<uint32_t *>(smem + 4 * Kp);
    for (int i = threadIdx.x; i < 4 * Kp; i += blockDim.x) smem[i] = a.fc[i];
    for (int i = threadIdx.x; i < K * kAccPerCluster; i += blockDim.x) s_acc[i] = 0;
    __syncthreads();
    const uint64_t m = *listn;
    constexpr uint64_t tile = (uint64_t)kSweepThreads * PPT;
    for (uint64_t lo = (uint64_t)blockIdx.x * tile; lo < m; lo += (uint64_t)gridDim.x * tile) {
        const uint64_t hi = lo + tile < m ? lo + tile : m;
        sweep_tiles<MODE_WALK, PPT, true>(a, lo, hi, list, smem, s_acc, __ldg(a.tau), __ldg(a.tau + 1));
    }
    if (threadIdx.x == 0 && a.swept && m && blockIdx.x == 0) atomicAdd(a.swept, m);
}

template <int MODE, int PPT>
__global__ void __launch_bounds__(kSweepThreads, 2) sweep_kernel(SweepArgs a) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) float smem[];
    const int K = a.K, Kp = a.Kp;
    uint32_t *s_acc = reinterpret_cast<uint32_t *>(smem + 4 * Kp);
    for (int i = threadIdx.x; i < 4 * Kp; i += blockDim.x) smem[i] = a.fc[i];
    for (int i = threadIdx.x; i < K * kAccPerCluster; i += blockDim.x) s_acc[i] = 0;
    __syncthreads();
    const uint64_t chunk = (a.n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    const uint64_t hi = lo + chunk < a.n ? lo + chunk : a.n;
    uint32_t *s_list = reinterpret_cast<uint32_t *>(s_acc) + sweep_acc_words(K);
    float *s_aux = reinterpret_cast<float *>(s_list + kPruneChunk + kSweepThreads * 8);
    sweep_range<MODE, PPT>(a, lo, hi, smem, s_acc, a.tau[0], a.tau[1], s_list, kPruneChunk, s_aux);
}

// ---------------------------------------------------------------------------
// Exact FP64 replay of the reference's assignment for queued (near-tie) points,
// one warp per point (lanes split the candidates, lexicographic warp min).
//   FULL / MAP: nearest_full (kmeans.cpp:40-54): min d, lowest index on ties.
//   WALK: assign_point_sortmeans (kmeans.cpp:56-79): candidates are walk
//         positions 0..cnt (0 = the previous label) with cnt from the exact
//         cutoff; the walk keeps the FIRST minimum in walk order, i.e. the
//         minimum of (d, position).
__device__ __forceinline__ void warp_min_dp(double &d, int &p) {
    for (int o = 16; o; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, d, o);
        const int op = __shfl_xor_sync(0xffffffffu, p, o);
        if (od < d || (od == d && op < p)) {
            d = od;
            p = op;
        }
    }
}

template <int MODE>
__device__ __forceinline__ void replay_range(const SweepArgs &a, uint32_t gwarp, uint32_t warps) {
    const uint32_t nq = *a.qn;
    const int lane = threadIdx.x & 31;
    for (uint32_t q = gwarp; q < nq; q += warps) {
        const uint32_t idx = a.queue[q];
        const uint32_t c = a.colors[idx], cnt = a.counts[idx];
        const uint32_t r = (c >> 16) & 255u, g = (c >> 8) & 255u, b = c & 255u;
        const double xr = (double)r, xg = (double)g, xb = (double)b;
        const int K = a.K;
        double bd = 1.0e300;
        int bp = 0x7FFFFFFF;
        int best;
        if (MODE == MODE_WALK) {
            const int prev = (int)a.labels[idx];
            const double pd = d2_exact(xr, xg, xb, a.cen[3 * prev], a.cen[3 * prev + 1], a.cen[3 * prev + 2]);
            const uint32_t npos = walk_positions_warp(__dmul_rn(4.0, pd), a.dsorted + (size_t)prev * a.Kpow,
                                                      a.Kpow); // positions 0..npos-1
            const uint32_t *orow = a.order + (size_t)prev * K;
            for (uint32_t p = lane; p < npos; p += 32) {
                const uint32_t t = orow[p];
                const double d = d2_exact(xr, xg, xb, a.cen[3 * t], a.cen[3 * t + 1], a.cen[3 * t + 2]);
                if (d < bd) {
                    bd = d;
                    bp = (int)p;
                }
            }
            warp_min_dp(bd, bp);
            best = (int)orow[bp];
            if (lane == 0 && best != prev) {
                a.labels[idx] = (uint32_t)best;
                accumulate_global(a.mom, best, cnt, r, g, b, +1);
                accumulate_global(a.mom, prev, cnt, r, g, b, -1);
            }
        } else {
            for (int j = lane; j < K; j += 32) {
                const double d = d2_exact(xr, xg, xb, a.cen[3 * j], a.cen[3 * j + 1], a.cen[3 * j + 2]);
                if (d < bd) {
                    bd = d;
                    bp = j;
                }
            }
            warp_min_dp(bd, bp);
            best = bp;
            if (lane == 0) {
                if (MODE == MODE_FULL) a.labels[idx] = (uint32_t)best;
                else map_store(a, c, idx, (uint32_t)best);
                if (MODE == MODE_MAPW) { // moments hold Lloyd's final labels: move the point
                    const int prev = (int)a.labels[idx];
                    if (best != prev) {
                        accumulate_global(a.mom, best, cnt, r, g, b, +1);
                        accumulate_global(a.mom, prev, cnt, r, g, b, -1);
                    }
                } else {
                    accumulate_global(a.mom, best, cnt, r, g, b, +1);
                }
            }
        }
    }
}

// WALK replay without the sorted walk table (persistent Lloyd kernel): the
// walk of assign_point_sortmeans visits prev first, then every j with
// D[prev][j] < cutoff in (D[prev][j], j) order, and keeps the first strict
// minimum; so the winner is the lexicographic minimum of (d(x, c_j), walk
// key) with walk key (-1) for prev and (D[prev][j], j) otherwise. Lanes split
// the centres; D is recomputed as the reference's table holds it (dist2).
__device__ __forceinline__ void replay_walk_tableless(const SweepArgs &a, uint32_t gwarp, uint32_t warps) {
    const uint32_t nq = *a.qn;
    const int lane = threadIdx.x & 31;
    const double *cen = a.cen;
    const int K = a.K;
    for (uint32_t q = gwarp; q < nq; q += warps) {
        const uint32_t idx = a.queue[q];
        const uint32_t c = a.colors[idx], cnt = a.counts[idx];
        const uint32_t r = (c >> 16) & 255u, g = (c >> 8) & 255u, b = c & 255u;
        const double xr = (double)r, xg = (double)g, xb = (double)b;
        const int prev = (int)a.labels[idx];
        const double pr = cen[3 * prev], pg = cen[3 * prev + 1], pb = cen[3 * prev + 2];
        const double pd = d2_exact(xr, xg, xb, pr, pg, pb);
        const double cut = __dmul_rn(4.0, pd);
        double bd = lane == 0 ? pd : 1.0e300, bD = -1.0;
        int bj = lane == 0 ? prev : 0x7FFFFFFF;
        for (int j = lane; j < K; j += 32) {
            if (j == prev) continue;
            const double D = d2_exact(pr, pg, pb, cen[3 * j], cen[3 * j + 1], cen[3 * j + 2]);
            if (!(D < cut)) continue;
            const double d = d2_exact(xr, xg, xb, cen[3 * j], cen[3 * j + 1], cen[3 * j + 2]);
            if (d < bd || (d == bd && (D < bD || (D == bD && j < bj)))) {
                bd = d;
                bD = D;
                bj = j;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const double oD = __shfl_xor_sync(0xffffffffu, bD, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (od < bd || (od == bd && (oD < bD || (oD == bD && oj < bj)))) {
                bd = od;
                bD = oD;
                bj = oj;
            }
        }
        if (lane == 0 && bj != prev) {
            a.labels[idx] = (uint32_t)bj;
            accumulate_global(a.mom, bj, cnt, r, g, b, +1);
            accumulate_global(a.mom, prev, cnt, r, g, b, -1);
        }
    }
}

template <int MODE>
__global__ void replay_kernel(SweepArgs a) {
    pdl_wait();
    pdl_trigger();
    replay_range<MODE>(a, (blockIdx.x * blockDim.x + threadIdx.x) >> 5, (gridDim.x * blockDim.x) >> 5);
}

// FP32 centre table + error bound for the sweep (one block).
//   E <= u*|cc err| + u*|m2c err|*x + 3u*M  with u = 2^-24 and M the largest
//   magnitude of any partial sum (cc + xx when all coordinates are >= 0).
__device__ void fc_block(const double *cen, int K, int Kp, float *fc, float *tau);
__global__ void fc_kernel(const double *cen, int K, int Kp, float *fc, float *tau);


size_t sweep_smem_bytes(int K, int Kp, int mode);
void launch_sweep(cqg_ctx *ctx, int mode, const SweepArgs &a);

} // namespace cqg
