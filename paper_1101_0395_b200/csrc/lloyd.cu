// lloyd.cu -- stages 2+3: weighted sort-means on the device.
//
// Replaces quant::wsm / run_lloyd (reference src/kmeans.cpp:173-277) for
// count-weighted substrates. Per iteration (all on the context stream):
//   sweep<FULL|WALK>   FP32 argmin + near-tie queue + NDC + moment deltas
//   replay<FULL|WALK>  exact FP64 reference assignment for queued points
//   iter_end           (K blocks) centres = S/n in FP64, SSE from the int128
//                      moment numerators, termination test (kmeans.cpp:249-257),
//                      FP32 centre table + error bound, and the K x K walk
//                      table for the next iteration (kmeans.cpp:14-38)
// Iteration 1 runs eagerly; iterations >= 2 run as ONE CUDA graph whose
// conditional WHILE node is driven by iter_end (cudaGraphSetConditional), so
// there is no host round trip per iteration. Empty clusters (rare) stop the
// loop; the host then runs a device-kernel replay of repair_empty_clusters
// (kmeans.cpp:124-169) and resumes.
#include <algorithm>
#include <cstring>

#include <cooperative_groups.h>

#include "sweep.cuh"

namespace cg = cooperative_groups;

namespace cqg {

// FP32 centre table and sweep error bound from FP64 centres (device helper,
// block-cooperative). E <= u|cc err| + u|m2c err| x + 3 u M, u = 2^-24, M the
// largest |partial sum| of the FMA chain (<= 3C^2 + 6XC).
__device__ void fc_block(const double *cen, int K, int Kp, float *fc, float *tau) {
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
        // e = fma(b, m2b, fma(g, m2g, fma(r, m2r, cc))): the FP32 table's own
        // rounding (cc, m2) plus one rounding per FMA of a partial sum bounded
        // by |cc| + sum |x m2| <= 3C^2 + 6XC
        (void)anyneg;
        const double u = 0x1.0p-24, X = 255.0;
        const double cc_err = u * 3.0 * C * C;
        const double m2c_err = u * 2.0 * X * 3.0 * C;
        const double M = 3.0 * C * C + 6.0 * X * C;
        const double E = cc_err + m2c_err + 3.0 * u * M;
        tau[0] = (float)(2.0 * E * 1.0625 + 1.0e-3);
        tau[1] = 0x1.0p-20f; // rounding of the FP32 gap test itself
    }
    __syncthreads();
}

__global__ void fc_kernel(const double *cen, int K, int Kp, float *fc, float *tau) {
    pdl_trigger();
    fc_block(cen, K, Kp, fc, tau);
}

namespace {

struct IterArgs {
    Moments *mom;
    double *cen;
    int K, Kp;
    uint64_t P;
    uint64_t n_points;
    double eps;
    int limit, fixed;
    double *sse_arr;
    IterStatus *st;
    int *iter_dev;       // last completed iteration
    const uint32_t *qn;
    unsigned long long *ndc;
    unsigned long long *flagged;
    float *fc, *tau;
    double *dtab, *dsorted;
    uint32_t *order;
    int Kpow;
    cudaGraphConditionalHandle cond;
    int use_cond;
    int reset_qn; // persistent kernel: clear the replay queue counter
    uint16_t *dcode;  // K x Kpow codes of dsorted for ndc_code_kernel, or null
    float *shift;     // K centre moves (FP64 -> float, rounded up) + {max, 2nd max, argmax}; null = off
    int *shift_inval; // set by a repair: the next shifts are +inf (all bounds void)
    // persistent kernel: no walk rows in the loop (no_walk_rows), only each
    // centre's nearest-other distance rowmin[K] for the stay test; snapshots of
    // the labels (snap_lab, n per iteration) and centres (snap_cen, 3K) each
    // WALK iteration starts from, for the deferred NDC (ndc_post_kernel), in
    // win slots
    int no_walk_rows;
    double *rowmin;
    double *snap_cen;
    uint16_t *snap_lab;
    int win;
    Moments *dmom; // persistent kernel: 3 x K moment deltas (iteration t into slot t % 3)
};

__device__ __forceinline__ void top2_merge(float &m1, int &i1, float &m2, float n1, int j1, float n2) {
    if (n1 > m1) {
        m2 = fmaxf(m1, n2);
        m1 = n1;
        i1 = j1;
    } else {
        m2 = fmaxf(m2, n1);
    }
}

// Finalise one iteration and build the next walk table. Called by every block
// of a grid (iter_end_kernel, or the persistent kernel's phase C): block 0
// writes centres / SSE / termination status; every block computes the centres
// in shared memory; rows of the walk table are distributed over the blocks.
// fc_dst/tau_dst receive the FP32 sweep table: global (block 0 only) or this
// block's shared memory (fc_every_block). Returns false when a cluster is empty
// (status 2 written, nothing else changed).
#ifdef CQG_INIT_TIMING
__device__ unsigned long long g_lloyd_timing[8];
__device__ unsigned long long g_block_timing[1024 * 3]; // per block: ndc, sweep, replay cycles
#define BTIME(slot)                                                                  \
    do {                                                                             \
        if (threadIdx.x == 0) {                                                      \
            const unsigned long long _n = clock64();                                 \
            g_block_timing[blockIdx.x * 3 + (slot)] += _n - _bprev;                  \
            _bprev = _n;                                                             \
        }                                                                            \
    } while (0)
#else
#define BTIME(slot) \
    do {            \
    } while (0)
#endif

// Bitonic sort of KP (key, index) pairs held one per thread (threads >= KP
// idle in the exchanges): strides < 32 by warp shuffles, larger strides
// through shared memory (s_key / s_idx, KP entries). All stages unrolled.
template <int KP>
__device__ __forceinline__ void bitonic_reg(unsigned long long &key, int &r, int t, unsigned long long *s_key,
                                            int *s_idx) {
    const bool in = t < KP;
#pragma unroll
    for (int size = 2; size <= KP; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            unsigned long long ok;
            int orr;
            if (stride >= 32) {
                __syncthreads();
                if (in) {
                    s_key[t] = key;
                    s_idx[t] = r;
                }
                __syncthreads();
                ok = in ? s_key[t ^ stride] : ~0ull;
                orr = in ? s_idx[t ^ stride] : 0x7FFFFFFF;
            } else {
                ok = __shfl_xor_sync(0xffffffffu, key, stride);
                orr = __shfl_xor_sync(0xffffffffu, r, stride);
            }
            const bool up = (t & size) == 0;
            const bool low = (t & stride) == 0;
            const bool other_less = ok < key || (ok == key && orr < r);
            if (other_less == (low == up)) { // the low slot keeps the smaller key when ascending
                key = ok;
                r = orr;
            }
        }
    }
}

// Nearest other centre per row, min_{j != i} dist2(c_i, c_j) (the stay
// test's Elkan term), rows spread over the blocks of the grid.
__device__ void rowmin_rows(const double *c, int K, double *out) {
    __shared__ double s_rm[32];
    const double kInf = __longlong_as_double(0x7FF0000000000000ll);
    for (int i = blockIdx.x; i < K; i += gridDim.x) {
        const double cr = c[3 * i], cg = c[3 * i + 1], cb = c[3 * i + 2];
        double m = kInf;
        for (int j = threadIdx.x; j < K; j += blockDim.x)
            if (j != i) m = fmin(m, d2_exact(cr, cg, cb, c[3 * j], c[3 * j + 1], c[3 * j + 2]));
        for (int o = 16; o; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0) s_rm[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmin(m, s_rm[w]);
            out[i] = m;
        }
        __syncthreads();
    }
}

// The exact-moment SSE's summation order (shared with the oracle's
// tree_sum): pairwise on a complete binary tree over the next power of two
// >= K, left + right at every node, in place in shared memory, one level per
// step. Every thread of the block calls it; the sum is a[0].
__device__ double tree_sum_block(double *a, int K) {
    for (int st = 1; st < K; st <<= 1) {
        __syncthreads();
        for (int i = 2 * st * (int)threadIdx.x; i + st < K; i += 2 * st * (int)blockDim.x)
            a[i] = __dadd_rn(a[i], a[i + st]);
    }
    __syncthreads();
    return a[0];
}

// The same tree with every thread of a block (blockDim a power of two, K <=
// 4 blockDim): thread t sums its aligned segment of L = N / blockDim entries
// (the tree's lowest levels) in registers, the next five levels run inside the
// warp by shuffles, the last ones across the warp sums in warp 0. No shared
// memory bank conflicts (a single lane walking a segment would hit one bank).
// The sum is returned to thread 0; s_w: one double per warp.
__device__ double tree_sum_threads(const double *a, int K, double *s_w) {
    const int nt = blockDim.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    int N = nt;
    while (N < K) N <<= 1;
    const int L = N / nt, base = t * L; // L <= 4
    double v0 = base < K ? a[base] : 0.0;
    if (L >= 2) {
        const double v1 = base + 1 < K ? a[base + 1] : 0.0;
        double u = __dadd_rn(v0, v1);
        if (L == 4) {
            const double v2 = base + 2 < K ? a[base + 2] : 0.0, v3 = base + 3 < K ? a[base + 3] : 0.0;
            u = __dadd_rn(u, __dadd_rn(v2, v3));
        }
        v0 = u;
    }
    for (int o = 1; o < 32; o <<= 1) {
        const double w = __shfl_down_sync(0xffffffffu, v0, o);
        if ((lane & (2 * o - 1)) == 0) v0 = __dadd_rn(v0, w);
    }
    if (lane == 0) s_w[warp] = v0;
    __syncthreads();
    double r = 0.0;
    if (warp == 0) {
        const int nw = nt >> 5;
        r = lane < nw ? s_w[lane] : 0.0;
        for (int o = 1; o < nw; o <<= 1) {
            const double w = __shfl_down_sync(0xffffffffu, r, o);
            if ((lane & (2 * o - 1)) == 0) r = __dadd_rn(r, w);
        }
    }
    return r;
}

__device__ bool iter_end_body(const IterArgs &a, double *sm, float *fc_dst, float *tau_dst, bool fc_every_block) {
#ifdef CQG_INIT_TIMING
    const unsigned long long _ie0 = clock64();
#endif
    // the bookkeeping block (SSE, status, shifts, global centres / FP32 table):
    // the last one, which owns no walk row when the grid exceeds K
    const bool boss = blockIdx.x == gridDim.x - 1;
    const int K = a.K;
    double *s_c = sm;               // 3K centres
    double *s_a = sm + 3 * K;       // K per-cluster SSE terms (block 0)
    double *s_d = sm + 4 * K;       // Kpow row distances (sort keys)
    int *s_rank = reinterpret_cast<int *>(sm + 4 * K + a.Kpow); // Kpow payload indices
    __shared__ int s_empty;
    if (threadIdx.x == 0) s_empty = 0;
    __syncthreads();
    int empty = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const Moments m = a.mom[k];
        if (m.n == 0) {
            empty = 1;
            continue;
        }
        const double nd = __ull2double_rn(m.n);
        s_c[3 * k] = __ddiv_rn(__ll2double_rn(m.s[0]), nd);
        s_c[3 * k + 1] = __ddiv_rn(__ll2double_rn(m.s[1]), nd);
        s_c[3 * k + 2] = __ddiv_rn(__ll2double_rn(m.s[2]), nd);
        if (boss) s_a[k] = cluster_sse_exact(m.n, m.s, m.q);
    }
    if (empty) atomicOr(&s_empty, 1);
    __syncthreads();
    const int iter = *a.iter_dev + 1;
    if (s_empty) {
        if (boss && threadIdx.x == 0) {
            a.st->state = 2;
            a.st->iteration = iter;
            a.st->n_flagged = *a.qn;
            if (a.use_cond) cudaGraphSetConditional(a.cond, 0);
        }
        return false;
    }
    if (boss) {
        // centre moves for the distance bounds, then publish the new centres
        float m1 = -1.f, m2 = -1.f;
        int i1 = -1;
        for (int k = threadIdx.x; k < K; k += blockDim.x) {
            if (a.shift) {
                const double dr = __dsub_rn(s_c[3 * k], a.cen[3 * k]);
                const double dg = __dsub_rn(s_c[3 * k + 1], a.cen[3 * k + 1]);
                const double db = __dsub_rn(s_c[3 * k + 2], a.cen[3 * k + 2]);
                const double d = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dg, dg)), __dmul_rn(db, db)));
                const float f = __double2float_ru(__dmul_ru(d, 1.0 + 0x1.0p-40)); // covers FP64 rounding
                a.shift[k] = f;
                top2_merge(m1, i1, m2, f, k, -1.f);
            }
            a.cen[3 * k] = s_c[3 * k];
            a.cen[3 * k + 1] = s_c[3 * k + 1];
            a.cen[3 * k + 2] = s_c[3 * k + 2];
        }
        if (a.shift) {
            __shared__ float s_m1[32], s_m2[32];
            __shared__ int s_i1[32];
            for (int o = 16; o; o >>= 1) {
                const float n1 = __shfl_xor_sync(0xffffffffu, m1, o), n2 = __shfl_xor_sync(0xffffffffu, m2, o);
                const int j1 = __shfl_xor_sync(0xffffffffu, i1, o);
                top2_merge(m1, i1, m2, n1, j1, n2);
            }
            if ((threadIdx.x & 31) == 0) {
                s_m1[threadIdx.x >> 5] = m1;
                s_m2[threadIdx.x >> 5] = m2;
                s_i1[threadIdx.x >> 5] = i1;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                for (int w = 1; w < (int)(blockDim.x >> 5); ++w) top2_merge(m1, i1, m2, s_m1[w], s_i1[w], s_m2[w]);
                const bool inval = *a.shift_inval != 0;
                const float inf = __int_as_float(0x7f800000);
                a.shift[K] = inval ? inf : fmaxf(m1, 0.f);
                a.shift[K + 1] = inval ? inf : fmaxf(m2, 0.f);
                a.shift[K + 2] = __int_as_float(i1);
                *a.shift_inval = 0;
            }
        }
        const double tot = tree_sum_block(s_a, K);
        if (threadIdx.x == 0) {
            const double sse = __ddiv_rn(tot, __ull2double_rn(a.P));
            a.sse_arr[iter - 1] = sse;
            int done;
            if (a.fixed > 0) {
                done = iter >= a.limit;
            } else {
                done = (sse == 0.0);
                if (!done && iter >= 2) {
                    const double prev = a.sse_arr[iter - 2];
                    done = __ddiv_rn(__dsub_rn(prev, sse), sse) <= a.eps;
                }
                if (!done && iter >= a.limit) done = 1;
            }
            if (iter == 1) *a.ndc += (unsigned long long)a.n_points * (unsigned long long)K;
            const uint32_t nq = *a.qn;
            *a.flagged += nq;
            if (a.reset_qn) *const_cast<uint32_t *>(a.qn) = 0;
            a.st->state = done ? 1 : 0;
            a.st->iteration = iter;
            a.st->n_flagged = nq;
            a.st->sse = sse;
            *a.iter_dev = iter;
            if (a.use_cond) cudaGraphSetConditional(a.cond, done ? 0 : 1);
        }
    }
    if (boss || fc_every_block) fc_block(s_c, K, a.Kp, fc_dst, tau_dst);
#ifdef CQG_INIT_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) g_lloyd_timing[6] += clock64() - _ie0;
#endif
    const double kInf = __longlong_as_double(0x7FF0000000000000ll);
    if (a.rowmin) rowmin_rows(s_c, K, a.rowmin);
    if (a.no_walk_rows) return true;
    // walk table row i (kmeans.cpp:14-38): sort by (d, index), then rotate self
    // to the front. Block bitonic sort over Kpow keys (padding = +inf).
    for (int i = blockIdx.x; i < K; i += gridDim.x) {
        const double cr = s_c[3 * i], cg = s_c[3 * i + 1], cb = s_c[3 * i + 2];
        for (int j = threadIdx.x; j < a.Kpow; j += blockDim.x) {
            double d = kInf;
            if (j < K) {
                d = d2_exact(cr, cg, cb, s_c[3 * j], s_c[3 * j + 1], s_c[3 * j + 2]);
                a.dtab[(size_t)i * K + j] = d;
            }
            s_d[j] = d;
            s_rank[j] = j; // index payload
        }
        __syncthreads();
        if (a.Kpow <= (int)blockDim.x) {
            // one element per thread, in registers, the stage loops unrolled
            // for the padded row length; keys compare as (u64 bits of d >= 0, index)
            const int t = threadIdx.x;
            unsigned long long key = t < a.Kpow ? (unsigned long long)__double_as_longlong(s_d[t]) : ~0ull;
            int r = t < a.Kpow ? s_rank[t] : 0x7FFFFFFF;
            unsigned long long *s_key = reinterpret_cast<unsigned long long *>(s_d);
            switch (a.Kpow) {
                case 512: bitonic_reg<512>(key, r, t, s_key, s_rank); break;
                case 256: bitonic_reg<256>(key, r, t, s_key, s_rank); break;
                case 128: bitonic_reg<128>(key, r, t, s_key, s_rank); break;
                case 64: bitonic_reg<64>(key, r, t, s_key, s_rank); break;
                default: bitonic_reg<32>(key, r, t, s_key, s_rank); break; // Kpow <= 32: padding lanes sort last
            }
            __syncthreads();
            if (t < a.Kpow) {
                s_d[t] = __longlong_as_double((long long)key);
                s_rank[t] = r;
            }
            __syncthreads();
        } else {
        for (int size = 2; size <= a.Kpow; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < (a.Kpow >> 1); t += blockDim.x) {
                    const int lo_i = 2 * t - (t & (stride - 1));
                    const int hi_i = lo_i + stride;
                    const bool up = (lo_i & size) == 0;
                    const double d0 = s_d[lo_i], d1 = s_d[hi_i];
                    const int i0 = s_rank[lo_i], i1 = s_rank[hi_i];
                    const bool gt = d0 > d1 || (d0 == d1 && i0 > i1);
                    if (gt == up) {
                        s_d[lo_i] = d1;
                        s_d[hi_i] = d0;
                        s_rank[lo_i] = i1;
                        s_rank[hi_i] = i0;
                    }
                }
                __syncthreads();
            }
        }
        }
        // position of self, then rotate it to the front
        __shared__ int s_self;
        for (int p = threadIdx.x; p < K; p += blockDim.x)
            if (s_rank[p] == i) s_self = p;
        __syncthreads();
        const int ps = s_self;
        for (int p = threadIdx.x; p < a.Kpow; p += blockDim.x) {
            const int np = p < ps ? p + 1 : (p == ps ? 0 : p);
            if (p < K) a.order[(size_t)i * K + np] = (uint32_t)s_rank[p];
            a.dsorted[(size_t)i * a.Kpow + np] = s_d[p];
            if (a.dcode) a.dcode[(size_t)i * a.Kpow + np] = (uint16_t)code16(s_d[p]);
        }
        __syncthreads();
    }
#ifdef CQG_INIT_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) g_lloyd_timing[7] += clock64() - _ie0;
#endif
    return true;
}

__global__ void __launch_bounds__(1024) iter_end_kernel(IterArgs a) {
    extern __shared__ double sm[];
    iter_end_body(a, sm, a.fc, a.tau, false);
}

// phase timing of the persistent kernel (timing builds, tools/init_timing.py)
#ifdef CQG_INIT_TIMING
#define PTIME(slot)                                                                  \
    do {                                                                             \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                   \
            const unsigned long long _n = clock64();                                 \
            g_lloyd_timing[slot] += _n - _tprev;                                     \
            _tprev = _n;                                                             \
        }                                                                            \
    } while (0)
#else
#define PTIME(slot) \
    do {            \
    } while (0)
#endif

// Persistent cooperative Lloyd loop for small substrates: one launch runs all
// iterations with ONE grid barrier per iteration. Per iteration t:
//   sweep t (centres C_t) + block-local exact replay; moment deltas into
//   dmom[t % 3]; block 0 clears dmom[(t + 1) % 3]
//   | grid barrier |
//   every block finalises redundantly: absolute moments M_t (shared copy) +=
//   dmom[t % 3], centres C_{t+1} = S / n, centre shifts, per-cluster SSE, the
//   SSE in the oracle's tree order and the termination test
//   (kmeans.cpp:249-257), the FP32 table, and the stay test's Hamerly terms.
// Deltas are read one barrier after they are written and cleared one barrier
// before they are reused (three slots). The walk table and the NDC leave the
// loop (label / centre snapshots + ndc_post_kernel). On exit (done, window
// full, empty cluster) block 0 publishes the state the host, the mapping and
// a relaunch start from: centres, absolute moments, shifts, status; every
// block computes its rows of the exact row minima (the mapping's Elkan term).
template <int PPT>
__global__ void __launch_bounds__(kSweepThreads, 2) lloyd_persistent_kernel(SweepArgs a, IterArgs ia, int first_full,
                                                                            uint32_t list_cap) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double psm[];
    const int K = a.K, Kp = a.Kp;
    const int tid = threadIdx.x;
    Moments *s_M = reinterpret_cast<Moments *>(psm);          // K absolute moments
    double *s_cen = reinterpret_cast<double *>(s_M + K);      // 2 x 3K centres (current / next)
    double *s_sse = s_cen + 6 * K;                            // K per-cluster SSE terms
    float *s_fc = reinterpret_cast<float *>(s_sse + K);       // 4 Kp
    float *s_tau = s_fc + 4 * Kp;                             // 2 (+2 pad)
    uint32_t *s_acc = reinterpret_cast<uint32_t *>(s_tau + 4); // 10 K u32 (= 5 K u64)
    uint32_t *s_list = s_acc + 10 * K;                        // prune list + carried tile
    float *s_aux = reinterpret_cast<float *>(s_list + list_cap + kSweepThreads * 4); // 2K + 4
    __shared__ float s_rmax[8], s_rm1[8], s_rm2[8];
    __shared__ int s_ri1[8], s_rempty[8];
    __shared__ int s_state;
    __shared__ double s_ssev, s_wsum[32];
    __shared__ uint32_t s_qn;

    const uint64_t chunk = (a.n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    const uint64_t hi = lo + chunk < a.n ? lo + chunk : a.n;
    const uint32_t warp = tid >> 5, nw = blockDim.x >> 5;
    SweepArgs la = a; // block-local near-tie queue
    la.queue = a.queue + lo;
    la.qn = &s_qn;
    la.aux_ready = 1;
    // one flush per sweep when the block owns at most 2048 points (no u32
    // partial sum can overflow: SM-budgeted contexts give blocks more points)
    la.flush_at_end = chunk <= 2048 ? 1 : 0;

    // entry state: centres C_t, moments M_{t-1} (zero before iteration 1)
    bool full = first_full != 0;
    int t = *ia.iter_dev + 1; // the iteration about to run
    const int t0 = full ? t + 1 : t; // first WALK iteration: snapshot slot 0
    double *cen = s_cen, *cnx = s_cen + 3 * K;
    for (int i = tid; i < 3 * K; i += blockDim.x) cen[i] = a.cen[i];
    {
        unsigned long long *m = reinterpret_cast<unsigned long long *>(s_M);
        const unsigned long long *g = reinterpret_cast<const unsigned long long *>(ia.mom);
        for (int i = tid; i < 5 * K; i += blockDim.x) m[i] = full ? 0ull : g[i];
    }
    double sse_prev = (!full && t >= 2) ? ia.sse_arr[t - 2] : 0.0;
    for (int k = tid; k < K; k += blockDim.x) s_aux[K + k] = 0.f; // no Elkan term in this loop
    if (!full && a.bnd) { // a relaunch: the host-side finalise left the shifts
        for (int k = tid; k < K; k += blockDim.x) {
            s_aux[k] = a.shift[k];
            s_aux[K + k] = 0.f; // Hamerly only (see the finalise below)
        }
        if (tid < 3) s_aux[2 * K + tid] = a.shift[K + tid];
    }
    __syncthreads();                   // cen[] is read across threads below
    fc_block(cen, K, Kp, s_fc, s_tau); // ends with a block barrier
#ifdef CQG_INIT_TIMING
    unsigned long long _tprev = clock64();
    unsigned long long _bprev = _tprev;
#endif
    for (;;) {
        Moments *dst = ia.dmom + (size_t)(t % 3) * K;
        SweepArgs wa = la;
        wa.cen = cen;
        wa.mom = dst;
        if (tid == 0) s_qn = 0;
        if (full) {
            for (int i = tid; i < K * kAccPerCluster; i += blockDim.x) s_acc[i] = 0;
            __syncthreads();
            sweep_range<MODE_FULL, PPT>(wa, lo, hi, s_fc, s_acc, s_tau[0], s_tau[1]);
            __syncthreads();
            if (la.flush_at_end) flush_acc(s_acc, dst, K);
            replay_range<MODE_FULL>(wa, warp, nw);
        } else {
            // the NDC of this iteration is counted after the loop (ndc_post_kernel)
            // from the labels and centres it starts from
            const int slot = t - t0;
            if (blockIdx.x == 0)
                for (int i = tid; i < 3 * K; i += blockDim.x) ia.snap_cen[(size_t)slot * 3 * K + i] = cen[i];
            wa.lab_snap = ia.snap_lab + (size_t)slot * a.n;
            if (a.bnd == nullptr) // no filter pass: copy the labels here
                for (uint64_t i = lo + tid; i < hi; i += blockDim.x) wa.lab_snap[i] = (uint16_t)a.labels[i];
            for (int i = tid; i < K * kAccPerCluster; i += blockDim.x) s_acc[i] = 0;
            __syncthreads();
            PTIME(0);
            BTIME(0);
            sweep_range<MODE_WALK, PPT>(wa, lo, hi, s_fc, s_acc, s_tau[0], s_tau[1], s_list, list_cap, s_aux);
            __syncthreads();
            PTIME(1);
            BTIME(1);
            if (la.flush_at_end) flush_acc(s_acc, dst, K);
            replay_walk_tableless(wa, warp, nw);
            PTIME(2);
            BTIME(2);
        }
        __syncthreads();
        if (tid == 0 && s_qn) atomicAdd(ia.flagged, (unsigned long long)s_qn);
        if (blockIdx.x == 0) {
            unsigned long long *z = reinterpret_cast<unsigned long long *>(ia.dmom + (size_t)((t + 1) % 3) * K);
            for (int i = tid; i < 5 * K; i += blockDim.x) z[i] = 0ull;
        }
        grid.sync();
        PTIME(3);
#ifdef CQG_INIT_TIMING
        _bprev = clock64();
#endif
        // ---- finalise iteration t (every block, identical results) ----
        // pass 1, per cluster: moments += deltas, centre, shift, SSE term, FP32
        // table row, and the neighbour terms of C_t (two nearest, rounded down)
        {
            // absolute moments += this iteration's deltas: coalesced L2 reads of
            // the 5K words (other blocks' atomics), all issued before the adds
            const unsigned long long *dq = reinterpret_cast<const unsigned long long *>(dst);
            unsigned long long *mq = reinterpret_cast<unsigned long long *>(s_M);
            const int nwd = 5 * K;
            for (int e0 = tid; e0 < nwd; e0 += 8 * blockDim.x) {
                unsigned long long v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int e = e0 + u * blockDim.x;
                    v[u] = e < nwd ? __ldcg(dq + e) : 0ull;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int e = e0 + u * blockDim.x;
                    if (e < nwd) mq[e] += v[u];
                }
            }
        }
        __syncthreads();
        float cm = 0.f, m1 = -1.f, m2 = -1.f;
        int i1 = -1, empty = 0;
        for (int k = tid; k < K; k += blockDim.x) {
            const Moments &m = s_M[k];
            s_sse[k] = 0.0;
            if (m.n == 0) {
                empty = 1;
                continue;
            }
            const double nd = __ull2double_rn(m.n);
            const double r = __ddiv_rn(__ll2double_rn(m.s[0]), nd);
            const double g = __ddiv_rn(__ll2double_rn(m.s[1]), nd);
            const double b = __ddiv_rn(__ll2double_rn(m.s[2]), nd);
            cnx[3 * k] = r;
            cnx[3 * k + 1] = g;
            cnx[3 * k + 2] = b;
            s_sse[k] = cluster_sse_exact(m.n, m.s, m.q);
            const double dr = __dsub_rn(r, cen[3 * k]), dg = __dsub_rn(g, cen[3 * k + 1]),
                         db = __dsub_rn(b, cen[3 * k + 2]);
            const double dd = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dg, dg)), __dmul_rn(db, db)));
            const float f = __double2float_ru(__dmul_ru(dd, 1.0 + 0x1.0p-40)); // covers FP64 rounding
            s_aux[k] = f;
            top2_merge(m1, i1, m2, f, k, -1.f);
            // FP32 sweep table of the new centre (fc_block's arithmetic)
            s_fc[k] = __double2float_rn(__dmul_rn(-2.0, r));
            s_fc[Kp + k] = __double2float_rn(__dmul_rn(-2.0, g));
            s_fc[2 * Kp + k] = __double2float_rn(__dmul_rn(-2.0, b));
            s_fc[3 * Kp + k] =
                __double2float_rn(__dadd_rn(__dadd_rn(__dmul_rn(r, r), __dmul_rn(g, g)), __dmul_rn(b, b)));
            cm = fmaxf(cm, __double2float_ru(fmax(fabs(r), fmax(fabs(g), fabs(b)))));
        }
        for (int o = 16; o; o >>= 1) {
            cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
            empty |= __shfl_xor_sync(0xffffffffu, empty, o);
            const float n1 = __shfl_xor_sync(0xffffffffu, m1, o), n2 = __shfl_xor_sync(0xffffffffu, m2, o);
            const int j1 = __shfl_xor_sync(0xffffffffu, i1, o);
            top2_merge(m1, i1, m2, n1, j1, n2);
        }
        if ((tid & 31) == 0) {
            s_rmax[warp] = cm;
            s_rempty[warp] = empty;
            s_rm1[warp] = m1;
            s_rm2[warp] = m2;
            s_ri1[warp] = i1;
        }
        __syncthreads();
#ifdef CQG_INIT_TIMING
        if (blockIdx.x == 0 && tid == 0) g_lloyd_timing[6] += clock64() - _bprev;
#endif
        // the SSE in the oracle's tree order (all threads), then thread 0: the
        // status; thread 32: the sweep's error bound and the largest shifts
        const double tot = tree_sum_threads(s_sse, K, s_wsum);
        if (warp == 0) {
            if (tid == 0) {
                for (int w = 1; w < (int)nw; ++w) empty |= s_rempty[w];
                int state = 0;
                if (empty) {
                    state = 2;
                } else {
                    const double sse = __ddiv_rn(tot, __ull2double_rn(ia.P));
                    int done;
                    if (ia.fixed > 0) {
                        done = t >= ia.limit;
                    } else {
                        done = (sse == 0.0);
                        if (!done && t >= 2) done = __ddiv_rn(__dsub_rn(sse_prev, sse), sse) <= ia.eps;
                        if (!done && t >= ia.limit) done = 1;
                    }
                    state = done ? 1 : (t + 1 - t0 >= ia.win ? 3 : 0);
                    s_ssev = sse;
                    if (blockIdx.x == 0) {
                        ia.sse_arr[t - 1] = sse;
                        if (t == 1) *ia.ndc += (unsigned long long)ia.n_points * (unsigned long long)K;
                    }
                }
                s_state = state;
            }
        } else {
            // the other warps: the two largest shifts for the stay test's
            // Hamerly term (the Elkan term is off inside this loop: measured on
            // cfg2, its per-iteration row minima cost more than the pruning
            // they add -- survivor tiles are latency-bound, not count-bound)
            if (tid == 32) {
                m1 = s_rm1[0];
                m2 = s_rm2[0];
                i1 = s_ri1[0];
                cm = s_rmax[0];
                for (int w = 1; w < (int)nw; ++w) {
                    top2_merge(m1, i1, m2, s_rm1[w], s_ri1[w], s_rm2[w]);
                    cm = fmaxf(cm, s_rmax[w]);
                }
                s_aux[2 * K] = fmaxf(m1, 0.f);
                s_aux[2 * K + 1] = fmaxf(m2, 0.f);
                s_aux[2 * K + 2] = __int_as_float(i1);
                const double u = 0x1.0p-24, X = 255.0, C = (double)cm;
                const double E = u * 3.0 * C * C + u * 2.0 * X * 3.0 * C + 3.0 * u * (3.0 * C * C + 6.0 * X * C);
                s_tau[0] = (float)(2.0 * E * 1.0625 + 1.0e-3);
                s_tau[1] = 0x1.0p-20f;
            }
        }
        __syncthreads();
#ifdef CQG_INIT_TIMING
        if (blockIdx.x == 0 && tid == 0) g_lloyd_timing[7] += clock64() - _bprev;
#endif
        const int state = s_state;
        if (state == 2) {
            // an empty cluster: the host repairs from the centres of this
            // iteration's assignment and the absolute moments
            if (blockIdx.x == 0) {
                for (int i = tid; i < 3 * K; i += blockDim.x) ia.cen[i] = cen[i];
                unsigned long long *g = reinterpret_cast<unsigned long long *>(ia.mom);
                const unsigned long long *m = reinterpret_cast<const unsigned long long *>(s_M);
                for (int i = tid; i < 5 * K; i += blockDim.x) g[i] = m[i];
                if (tid == 0) {
                    ia.st->state = 2;
                    ia.st->iteration = t;
                    ia.st->n_flagged = 0;
                }
            }
            break;
        }
        PTIME(4);
        if (state != 0) {
            // done or window full: publish C_{t+1}, shifts, moments, exact row minima
            if (blockIdx.x == 0) {
                for (int i = tid; i < 3 * K; i += blockDim.x) ia.cen[i] = cnx[i];
                unsigned long long *g = reinterpret_cast<unsigned long long *>(ia.mom);
                const unsigned long long *m = reinterpret_cast<const unsigned long long *>(s_M);
                for (int i = tid; i < 5 * K; i += blockDim.x) g[i] = m[i];
                if (ia.shift) {
                    const bool inval = *ia.shift_inval != 0;
                    const float inf = __int_as_float(0x7f800000);
                    for (int k = tid; k < K; k += blockDim.x) ia.shift[k] = s_aux[k];
                    if (tid == 0) {
                        ia.shift[K] = inval ? inf : s_aux[2 * K];
                        ia.shift[K + 1] = inval ? inf : s_aux[2 * K + 1];
                        ia.shift[K + 2] = s_aux[2 * K + 2];
                    }
                }
                if (tid == 0) {
                    ia.st->state = state;
                    ia.st->iteration = t;
                    ia.st->n_flagged = 0;
                    ia.st->sse = s_ssev;
                    *ia.iter_dev = t;
                }
            }
            if (ia.rowmin) rowmin_rows(cnx, K, ia.rowmin);
            break;
        }
        sse_prev = s_ssev;
        double *tmp = cen;
        cen = cnx;
        cnx = tmp;
        ++t;
        full = false;
        __syncthreads();
        PTIME(5);
    }
}

// ---- deferred NDC of the persistent loop ----------------------------------
// The reference counts, for iteration t >= 2, 1 + #{j != prev : D_t[prev][j] <
// 4 d2(x, c_t,prev)} distances per point (assign_point_sortmeans). The
// persistent kernel keeps only the labels and centres each WALK iteration
// started from; after the loop, walk_keys_kernel sorts every iteration's
// rows as 32-bit keys (code16(D) << 16 | j) and ndc_post_kernel counts by
// binary lifting over the codes (FP64 only for entries whose code equals the
// cutoff's), all iterations at once.
template <int KS>
__device__ __forceinline__ void bitonic_u32(uint32_t &key, int t, uint32_t *s_key) {
#pragma unroll
    for (int size = 2; size <= KS; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            uint32_t ok;
            if (stride >= 32) {
                __syncthreads();
                s_key[t] = key;
                __syncthreads();
                ok = s_key[t ^ stride];
            } else {
                ok = __shfl_xor_sync(0xffffffffu, key, stride);
            }
            const bool up = (t & size) == 0;
            const bool low = (t & stride) == 0;
            if ((ok < key) == (low == up)) key = ok;
        }
    }
}

// rows of every snapshot table: KS (>= 32, >= K, power of two) keys per row,
// 1024 / KS rows per block, padding keys 0xFFFFFFFF
template <int KS>
__global__ void __launch_bounds__(1024) walk_keys_kernel(const double *__restrict__ snap_cen, int K,
                                                         const IterStatus *st, int t0, uint32_t *__restrict__ keys) {
    constexpr int RPB = 1024 / KS;
    __shared__ uint32_t s_key[1024];
    extern __shared__ double s_c[]; // 3 K
    const int nt = st->iteration - t0 + 1;
    if (nt <= 0) return;
    const int groups = (K + RPB - 1) / RPB;
    const int t = threadIdx.x & (KS - 1), rr = threadIdx.x / KS;
    for (int it = blockIdx.x; it < nt * groups; it += gridDim.x) {
        const int tab = it / groups, row = (it - tab * groups) * RPB + rr;
        const double *cen = snap_cen + (size_t)tab * 3 * K;
        __syncthreads();
        for (int i = threadIdx.x; i < 3 * K; i += blockDim.x) s_c[i] = cen[i];
        __syncthreads();
        uint32_t key = 0xFFFFFFFFu;
        if (row < K && t < K)
            key = (code16(d2_exact(s_c[3 * row], s_c[3 * row + 1], s_c[3 * row + 2], s_c[3 * t], s_c[3 * t + 1],
                                   s_c[3 * t + 2]))
                   << 16) |
                  (uint32_t)t;
        bitonic_u32<KS>(key, t, s_key + rr * KS);
        if (row < K) keys[((size_t)tab * K + row) * KS + t] = key;
    }
}

constexpr int kNdcPostThreads = 512;
constexpr int kNdcPostChunk = 4096;
// Per block a contiguous range of (table, point chunk) items; the table's
// centres and the first L codes of each of its rows live in shared memory.
template <int Q>
__global__ void __launch_bounds__(kNdcPostThreads) ndc_post_kernel(const uint32_t *__restrict__ colors, uint64_t n,
                                                                  const uint16_t *__restrict__ snap_lab,
                                                                  const double *__restrict__ snap_cen,
                                                                  const uint32_t *__restrict__ keys, int K, int KS,
                                                                  int L, const IterStatus *st, int t0,
                                                                  unsigned long long *ndc) {
    extern __shared__ __align__(16) double s_c2[]; // 3 K centres, then K rows of L + 2 codes
    uint16_t *s_pre = reinterpret_cast<uint16_t *>(s_c2 + 3 * K);
    const int rs = L + 2;
    const int nt = st->iteration - t0 + 1;
    if (nt <= 0) return;
    // chunks sized so that (table, chunk) items roughly fill the grid once:
    // a multiple of one batch (Q x threads), at least kNdcPostChunk / 4
    constexpr uint64_t batch = (uint64_t)Q * kNdcPostThreads;
    uint64_t csz = ((uint64_t)nt * n + gridDim.x - 1) / gridDim.x;
    csz = (csz + batch - 1) / batch * batch;
    if (csz < kNdcPostChunk / 4) csz = kNdcPostChunk / 4;
    const uint64_t nch = (n + csz - 1) / csz;
    const uint64_t items = (uint64_t)nt * nch;
    const uint64_t per = (items + gridDim.x - 1) / gridDim.x;
    const uint64_t i0 = (uint64_t)blockIdx.x * per, i1 = i0 + per < items ? i0 + per : items;
    unsigned long long local = 0;
    int cur = -1;
    for (uint64_t it = i0; it < i1; ++it) {
        const int tab = (int)(it / nch);
        const uint64_t p0 = (it - (uint64_t)tab * nch) * csz;
        const uint64_t p1 = p0 + csz < n ? p0 + csz : n;
        const uint32_t *tkeys = keys + (size_t)tab * K * KS;
        if (tab != cur) {
            __syncthreads();
            for (int i = threadIdx.x; i < 3 * K; i += blockDim.x) s_c2[i] = snap_cen[(size_t)tab * 3 * K + i];
            for (int e = threadIdx.x; e < K * L; e += blockDim.x) {
                const int r = e / L, p = e - r * L;
                s_pre[r * rs + p] = (uint16_t)(__ldg(tkeys + (size_t)r * KS + p) >> 16);
            }
            __syncthreads();
            cur = tab;
        }
        const uint16_t *lab = snap_lab + (size_t)tab * n;
        for (uint64_t base = p0; base < p1; base += (uint64_t)Q * kNdcPostThreads) {
            double cut[Q];
            uint32_t cc[Q];
            int prow[Q], pos[Q];
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const uint64_t i = base + threadIdx.x + (uint64_t)q * kNdcPostThreads;
                const bool v = i < p1;
                const uint32_t col = v ? __ldg(colors + i) : 0u;
                const int prev = v ? (int)__ldg(lab + i) : 0;
                const double pd = d2_exact((double)((col >> 16) & 255u), (double)((col >> 8) & 255u),
                                           (double)(col & 255u), s_c2[3 * prev], s_c2[3 * prev + 1],
                                           s_c2[3 * prev + 2]);
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
                const uint32_t *grow = tkeys + (size_t)prow[q] * KS;
                int p = pos[q];
                if (p == L - 1 && row[L - 1] < cc[q]) p = L;
                if (p == L && L < KS) {
                    // beyond the prefix: the entries with a smaller code, by lifting over the keys
                    const uint32_t kc = cc[q] << 16;
                    int b = 0;
                    for (int step = KS >> 1; step >= 1; step >>= 1)
                        if (__ldg(grow + b + step - 1) < kc) b += step;
                    if (b == KS - 1 && __ldg(grow + KS - 1) < kc) b = KS;
                    p = b;
                }
                int cnt = p;
                // entries whose code equals the cutoff's (sorted by index): decide in FP64
                if (p < KS && (p < L ? (uint32_t)row[p] : (__ldg(grow + p) >> 16)) == cc[q]) {
                    const double cr = s_c2[3 * prow[q]], cg = s_c2[3 * prow[q] + 1], cb = s_c2[3 * prow[q] + 2];
                    for (; p < KS; ++p) {
                        const uint32_t key = __ldg(grow + p);
                        if ((key >> 16) != cc[q]) break;
                        const int j = (int)(key & 0xFFFFu);
                        cnt += d2_exact(cr, cg, cb, s_c2[3 * j], s_c2[3 * j + 1], s_c2[3 * j + 2]) < cut[q];
                    }
                }
                local += (unsigned long long)(cnt - (cut[q] > 0.0 ? 1 : 0) + 1);
            }
        }
    }
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(ndc, local);
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
                                  double *cen, Moments *mom, uint32_t *sizes, uint64_t donor, int e,
                                  int *shift_inval) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (shift_inval) *shift_inval = 1; // labels/centres changed outside the bounds' bookkeeping
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

size_t sweep_smem_bytes(int K, int Kp, int mode) {
    // FP32 table, u32 accumulators (FULL/MAP) or u64 (WALK): reserve the larger,
    // and the WALK prune list
    return (size_t)4 * Kp * sizeof(float) + (size_t)sweep_acc_words(K) * sizeof(uint32_t) +
           (mode_delta(mode) ? ((size_t)kPruneChunk + kSweepThreads * 8 + prune_aux_words(K)) * sizeof(uint32_t)
                              : 0);
}

template <int MODE, int PPT>
static int sweep_bps(const cqg_ctx *ctx, size_t smem) {
    // occupancy per (device, kernel, smem): cached so launches do no host-side queries
    static thread_local size_t c_smem = (size_t)-1;
    static thread_local int c_dev = -1;
    static thread_local int c_bps = 1;
    if (c_smem == smem && c_dev == ctx->device) return c_bps;
    int bps = 0;
    CQG_CUDA(ensure_smem((const void *)sweep_kernel<MODE, PPT>, smem));
    CQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, sweep_kernel<MODE, PPT>, kSweepThreads, smem));
    c_bps = bps < 1 ? 1 : bps;
    c_smem = smem;
    c_dev = ctx->device;
    return c_bps;
}

template <int MODE, int PPT>
static void launch_ppt(cqg_ctx *ctx, const SweepArgs &a, size_t smem, int bps) {
    // one balanced wave: every SM gets bps blocks with equal point ranges
    uint64_t grid = (uint64_t)ctx->num_sms * (uint64_t)bps;
    const uint64_t cap = (a.n + 63) / 64; // at least 64 points per block
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    // chained to the previous kernel by programmatic dependent launch, except
    // in the captured Lloyd loop (WALK), whose graph keeps plain edges
    if (MODE == MODE_WALK) sweep_kernel<MODE, PPT><<<(unsigned)grid, kSweepThreads, smem, ctx->stream>>>(a);
    else launch_pdl(sweep_kernel<MODE, PPT>, (unsigned)grid, kSweepThreads, smem, ctx->stream, a);
}

#ifndef CQG_LIST_PPT
#define CQG_LIST_PPT 4
#endif
constexpr int kListPPT = CQG_LIST_PPT; // points per thread of the survivor-list sweep (build-time knob)
#ifndef CQG_DENSE_PPT
#define CQG_DENSE_PPT 8
#endif
constexpr int kDensePPT = CQG_DENSE_PPT; // largest points per thread of the range sweeps (build-time knob)
// Shared-memory attributes of the list sweep and its blocks per SM (cached
// per device and size; called once before any graph capture).
static int sweep_list_setup(cqg_ctx *ctx, int K, int Kp) {
    const size_t lsm = (size_t)4 * Kp * sizeof(float) + (size_t)sweep_acc_words(K) * sizeof(uint32_t);
    static thread_local size_t c_lsm = (size_t)-1;
    static thread_local int c_dev = -1, c_bps = 1;
    if (c_lsm != lsm || c_dev != ctx->device) {
        CQG_CUDA(ensure_smem((const void *)sweep_list_kernel<kListPPT>, lsm));
        int bps = 0;
        CQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, sweep_list_kernel<kListPPT>, kSweepThreads, lsm));
        c_bps = bps < 1 ? 1 : bps;
        c_lsm = lsm;
        c_dev = ctx->device;
    }
    return c_bps;
}

template <int MODE>
static void launch_sweep_mode(cqg_ctx *ctx, const SweepArgs &a) {
    const size_t smem = sweep_smem_bytes(a.K, a.Kp, MODE);
    const uint64_t n = a.n;
    const uint64_t sms = (uint64_t)ctx->num_sms;
    if (MODE == MODE_WALK && a.surv) {
        // the NDC, then one stay-test pass writing a survivor list, then the
        // list sweep (buffers and kernel attributes set up before any graph
        // capture: sweep_list_setup)
        uint32_t *list = a.surv;
        uint32_t *listn = list + n + 4;
        // the NDC (reads the labels before the sweep changes them) runs on the
        // second side stream beside the stay-test pass, joined before the sweep
        CQG_CUDA(cudaEventRecord(ctx->walk_fork, ctx->stream));
        CQG_CUDA(cudaStreamWaitEvent(ctx->aux2, ctx->walk_fork, 0));
        {
            // prefix codes in shared memory, 2 blocks of 512 threads per SM: half of each SM's threads
            // stay free for the stay-test pass running beside it (measured: 1 / 2 / 3 / 4 blocks per SM
            // -> cfg5 Lloyd 11.52 / 10.44 / 10.52 / 10.59 ms; whole rows in one 1024-thread block 10.57)
            const size_t cs = (size_t)a.K * 24 + (size_t)a.K * (kNdcPrefix + 2) * 2;
            const int gc = pick_grid(ctx, n, 512 * 4, 2);
            ndc_pre_kernel<4><<<gc, 512, cs, ctx->aux2>>>(a.colors, a.labels, n, a.cen, a.dsorted, a.dcode, a.K,
                                                         a.Kpow, a.ndc);
        }
        CQG_CUDA(cudaEventRecord(ctx->walk_join, ctx->aux2));
        CQG_CUDA(cudaMemsetAsync(listn, 0, 4, ctx->stream));
        const size_t fsm = filter_list_smem(a.K, a.Kp);
        const int gf = pick_grid(ctx, n, kFilterThreads * kFilterQ, 8);
        const int pb = prof_begin(ctx);
        filter_list_kernel<<<(unsigned)gf, kFilterThreads, fsm, ctx->stream>>>(a, list, listn);
        CQG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->walk_join, 0));
        const size_t lsm = (size_t)4 * a.Kp * sizeof(float) + (size_t)sweep_acc_words(a.K) * sizeof(uint32_t);
        const int bps = sweep_list_setup(ctx, a.K, a.Kp);
        sweep_list_kernel<kListPPT><<<(unsigned)(sms * bps), kSweepThreads, lsm, ctx->stream>>>(a, list, listn);
        prof_end(ctx, CQG_PROF_SWEEP, pb, (double)n * (double)a.K);
        const int rg = pick_grid(ctx, n * 32 / 256 + 1, 256, 2);
        const int pr = prof_begin(ctx);
        replay_kernel<MODE><<<rg, 256, 0, ctx->stream>>>(a);
        prof_end(ctx, CQG_PROF_REPLAY, pr, 0.0);
        CQG_CUDA(cudaGetLastError());
        launched(ctx, 4);
        std::memcpy(ctx->last_sweep, &a, sizeof(SweepArgs));
        ctx->have_last_sweep = true;
        return;
    }
    if (MODE == MODE_WALK) {
        const size_t csm = a.K <= 2048 ? (size_t)a.K * 24 : 0;
        if (csm > 48 * 1024) { // ensure_smem caches per (device, kernel)
            CQG_CUDA(ensure_smem((const void *)ndc_kernel<8>, 2048 * 24));
            CQG_CUDA(ensure_smem((const void *)ndc_kernel<2>, 2048 * 24));
        }
        const bool big = n >= (uint64_t)ctx->num_sms * 4 * 256 * 8;
        const int g = big ? pick_grid(ctx, n, 2048, 4) : pick_grid(ctx, n, 512, 8);
        const int pn = prof_begin(ctx);
        if (a.dcode && a.K <= kNdcCodeMaxK) {
            const size_t cs = (size_t)a.K * 24 + (size_t)a.K * (a.Kpow + 2) * 2;
            CQG_CUDA(ensure_smem((const void *)ndc_code_kernel<4>, kNdcCodeMaxK * 24 + kNdcCodeMaxK * (kNdcCodeMaxK + 2) * 2));
            const int gc = pick_grid(ctx, n, 1024 * 4, 1);
            ndc_code_kernel<4><<<gc, 1024, cs, ctx->stream>>>(a.colors, a.labels, n, a.cen, a.dsorted, a.dcode,
                                                             a.K, a.Kpow, a.ndc);
        } else if (big)
            ndc_kernel<8><<<g, 256, csm, ctx->stream>>>(a.colors, a.labels, n, a.cen, a.dsorted, a.K, a.Kpow, a.ndc);
        else
            ndc_kernel<2><<<g, 256, csm, ctx->stream>>>(a.colors, a.labels, n, a.cen, a.dsorted, a.K, a.Kpow, a.ndc);
        prof_end(ctx, CQG_PROF_NDC, pn, (double)n);
        launched(ctx);
    }
    // smallest points-per-thread whose single wave covers all points (fewest
    // idle lanes, most blocks); large inputs loop over 8-point tiles
    const int b2 = sweep_bps<MODE, 2>(ctx, smem), b4 = sweep_bps<MODE, 4>(ctx, smem), b8 = sweep_bps<MODE, 8>(ctx, smem);
    int ppt, bps;
    if (n <= sms * b2 * kSweepThreads * 2) ppt = 2, bps = b2;
    else if (n <= sms * b4 * kSweepThreads * 4 || kDensePPT == 4) ppt = 4, bps = b4;
    else ppt = 8, bps = b8;
    uint64_t grid = sms * (uint64_t)bps;
    const uint64_t cap = (n + 63) / 64; // at least 64 points per block
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    const int rg = pick_grid(ctx, n * 32 / 256 + 1, 256, 2);
    const int pb = prof_begin(ctx);
    if (ppt == 2) sweep_kernel<MODE, 2><<<(unsigned)grid, kSweepThreads, smem, ctx->stream>>>(a);
    else if (ppt == 4) sweep_kernel<MODE, 4><<<(unsigned)grid, kSweepThreads, smem, ctx->stream>>>(a);
    else sweep_kernel<MODE, 8><<<(unsigned)grid, kSweepThreads, smem, ctx->stream>>>(a);
    prof_end(ctx, MODE == MODE_MAP || MODE == MODE_MAPW ? CQG_PROF_MAPSWEEP : CQG_PROF_SWEEP, pb,
             (double)n * (double)a.K);
    const int pr = prof_begin(ctx);
    if (MODE == MODE_WALK) replay_kernel<MODE><<<rg, 256, 0, ctx->stream>>>(a);
    else launch_pdl(replay_kernel<MODE>, rg, 256, 0, ctx->stream, a);
    prof_end(ctx, CQG_PROF_REPLAY, pr, 0.0);
    CQG_CUDA(cudaGetLastError());
    launched(ctx, 2);
    if (MODE == MODE_WALK) {
        static_assert(sizeof(SweepArgs) <= sizeof(ctx->last_sweep), "scratch too small");
        std::memcpy(ctx->last_sweep, &a, sizeof(SweepArgs));
        ctx->have_last_sweep = true;
    }
}

// Isolated sweep timing (cqg_bench_sweep): reps back-to-back WALK sweeps.
void bench_sweep_dev(cqg_ctx *ctx, int reps, double *ms, double *units) {
    SweepArgs a;
    std::memcpy(&a, ctx->last_sweep, sizeof(SweepArgs));
    a.bnd = nullptr; // the dense sweep (every point against every centre)
    // the global FP32 table of the final centres (the persistent kernel kept its own)
    fc_kernel<<<1, 256, 0, ctx->stream>>>(a.cen, a.K, a.Kp, const_cast<float *>(a.fc), const_cast<float *>(a.tau));
    launched(ctx);
    const size_t smem = sweep_smem_bytes(a.K, a.Kp, MODE_WALK);
    const uint64_t sms = (uint64_t)ctx->num_sms, n = a.n;
    const int b2 = sweep_bps<MODE_WALK, 2>(ctx, smem), b4 = sweep_bps<MODE_WALK, 4>(ctx, smem),
              b8 = sweep_bps<MODE_WALK, 8>(ctx, smem);
    int ppt, bps;
    if (n <= sms * b2 * kSweepThreads * 2) ppt = 2, bps = b2;
    else if (n <= sms * b4 * kSweepThreads * 4 || kDensePPT == 4) ppt = 4, bps = b4;
    else ppt = 8, bps = b8;
    uint64_t grid = sms * (uint64_t)bps;
    const uint64_t cap = (n + 63) / 64;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    cudaEvent_t e0, e1;
    CQG_CUDA(cudaEventCreate(&e0));
    CQG_CUDA(cudaEventCreate(&e1));
    auto one = [&]() {
        if (ppt == 2) sweep_kernel<MODE_WALK, 2><<<(unsigned)grid, kSweepThreads, smem, ctx->stream>>>(a);
        else if (ppt == 4) sweep_kernel<MODE_WALK, 4><<<(unsigned)grid, kSweepThreads, smem, ctx->stream>>>(a);
        else sweep_kernel<MODE_WALK, 8><<<(unsigned)grid, kSweepThreads, smem, ctx->stream>>>(a);
    };
    one(); // warm
    CQG_CUDA(cudaEventRecord(e0, ctx->stream));
    for (int r = 0; r < reps; ++r) one();
    CQG_CUDA(cudaEventRecord(e1, ctx->stream));
    CQG_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    CQG_CUDA(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    launched(ctx, reps + 1);
    *ms = (double)t / reps;
    *units = (double)n * (double)a.K;
}

void launch_sweep(cqg_ctx *ctx, int mode, const SweepArgs &a) {
    if (mode == MODE_FULL) launch_sweep_mode<MODE_FULL>(ctx, a);
    else if (mode == MODE_WALK) launch_sweep_mode<MODE_WALK>(ctx, a);
    else if (mode == MODE_MAPW) launch_sweep_mode<MODE_MAPW>(ctx, a);
    else launch_sweep_mode<MODE_MAP>(ctx, a);
}

// ---------------------------------------------------------------------------

static int repair_loop(cqg_ctx *ctx, const uint32_t *colors, const uint32_t *counts, uint64_t n,
                       uint64_t P, int K, uint32_t *labels, double *cen, Moments *mom, int *shift_inval) {
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
        apply_move_kernel<<<1, 32, 0, s>>>(colors, counts, labels, cen, mom, sizes, best.i, e, shift_inval);
        launched(ctx);
        hsz[old] -= 1;
        hsz[e] += 1;
        ++repairs;
    }
    return repairs;
}

static int kpow_of(int K) {
    int p = 1;
    while (p < K) p <<= 1;
    return p;
}
static size_t iter_end_smem(int K) {
    return (size_t)K * 4 * sizeof(double) + (size_t)kpow_of(K) * (sizeof(double) + sizeof(int));
}

static void launch_iter_end(cqg_ctx *ctx, const IterArgs &ia) {
    const size_t smem = iter_end_smem(ia.K);
    if (smem > 48 * 1024)
        CQG_CUDA(ensure_smem((const void *)iter_end_kernel, (int)smem));
    iter_end_kernel<<<ia.K, 256, smem, ctx->stream>>>(ia);
    launched(ctx);
}

// Cached CUDA graph: WHILE(cond) { memset(qn); sweep<WALK>; replay<WALK>; iter_end }
static cudaGraphExec_t loop_graph(cqg_ctx *ctx, const SweepArgs &a, IterArgs ia, uint32_t *qn) {
    std::vector<uint64_t> key = {(uint64_t)a.colors, (uint64_t)a.counts, a.n, (uint64_t)a.labels,
                                 (uint64_t)a.cen, (uint64_t)a.K, (uint64_t)ia.limit, (uint64_t)ia.fixed,
                                 ia.P, __builtin_bit_cast(uint64_t, ia.eps), (uint64_t)a.mom,
                                 (uint64_t)a.queue, (uint64_t)ia.sse_arr, (uint64_t)ia.st,
                                 (uint64_t)ctx->stream};
    if (ctx->loop_exec && ctx->loop_key == key) return ctx->loop_exec;
    release_graphs(ctx);
    cudaGraph_t graph;
    CQG_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle h;
    CQG_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CQG_CUDA(cudaGraphAddNode(&cn, graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    ia.cond = h;
    ia.use_cond = 1;
    const bool prof = ctx->prof_on;
    ctx->prof_on = false; // no event records inside the captured body
    CQG_CUDA(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    CQG_CUDA(cudaMemsetAsync(qn, 0, 4, ctx->stream));
    launch_sweep(ctx, MODE_WALK, a);
    launch_iter_end(ctx, ia);
    cudaGraph_t captured;
    CQG_CUDA(cudaStreamEndCapture(ctx->stream, &captured));
    ctx->prof_on = prof;
    CQG_CUDA(cudaGraphInstantiate(&ctx->loop_exec, graph, 0));
    ctx->loop_graph = graph;
    ctx->loop_key = key;
    return ctx->loop_exec;
}

void release_graphs(cqg_ctx *ctx) {
    if (ctx->loop_exec) cudaGraphExecDestroy(ctx->loop_exec);
    if (ctx->loop_graph) cudaGraphDestroy(ctx->loop_graph);
    ctx->loop_exec = nullptr;
    ctx->loop_graph = nullptr;
    ctx->loop_key.clear();
}


static size_t persist_smem(int K, int Kp, size_t list_cap) {
    // moments, 2 x centres, SSE terms, FP32 table + tau, accumulators, prune
    // list + carried tile + stay-test terms (lloyd_persistent_kernel's layout)
    return (size_t)K * sizeof(Moments) + (size_t)7 * K * sizeof(double) + (size_t)4 * Kp * sizeof(float) +
           4 * sizeof(float) + (size_t)10 * K * sizeof(uint32_t) +
           (list_cap + kSweepThreads * 4 + prune_aux_words(K)) * sizeof(uint32_t);
}

// prune-list capacity of the persistent kernel: a block's whole point range
static size_t persist_list_words(const cqg_ctx *ctx, uint64_t n) {
    // grid = min(num_sms * bps, ceil(n / 64)): a block owns <= max(ceil(n / num_sms), 64) points
    uint64_t r = (n + ctx->num_sms - 1) / ctx->num_sms;
    if (r < 128) r = 128;
    return (size_t)(r < (uint64_t)kPruneChunk ? r : (uint64_t)kPruneChunk);
}

// Launch the persistent loop if it fits co-resident; returns false otherwise.
static bool launch_persistent(cqg_ctx *ctx, const SweepArgs &a, IterArgs ia, bool first_full) {
    const uint32_t list_cap = a.bnd ? (uint32_t)persist_list_words(ctx, a.n) : 0u;
    const size_t smem = persist_smem(a.K, a.Kp, list_cap);
    // 2-point tiles up to 4 points per thread of the grid (survivor tiles are
    // latency-bound; measured cfg1 0.216 -> 0.212 ms, cfg2 0.591 -> 0.584 ms vs 4-point)
    const int ppt = a.n <= (uint64_t)ctx->num_sms * 2 * kSweepThreads * 4 ? 2 : 4;
    const void *kern = ppt == 2 ? (const void *)lloyd_persistent_kernel<2> : (const void *)lloyd_persistent_kernel<4>;
    static thread_local const void *c_kern = nullptr;
    static thread_local size_t c_smem = 0;
    static thread_local int c_dev = -1;
    static thread_local int c_bps = 0;
    int bps = c_bps;
    if (c_kern != kern || c_smem != smem || c_dev != ctx->device) {
        CQG_CUDA(ensure_smem((const void *)kern, (int)smem));
        CQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern, kSweepThreads, smem));
        c_kern = kern;
        c_smem = smem;
        c_dev = ctx->device;
        c_bps = bps;
    }
    if (bps < 1) return false;
    uint64_t grid = (uint64_t)ctx->num_sms * (uint64_t)bps;
    const uint64_t cap = (a.n + 63) / 64;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    ia.use_cond = 0;
    ia.reset_qn = 1;
    CQG_CUDA(cudaMemsetAsync(ia.dmom, 0, 3 * sizeof(Moments) * (size_t)a.K, ctx->stream));
    SweepArgs aa = a;
    int ff = first_full ? 1 : 0;
    uint32_t lc = list_cap;
    void *args[] = {&aa, &ia, &ff, &lc};
    CQG_CUDA(launch_cooperative(ctx, kern, dim3((unsigned)grid), dim3(kSweepThreads), args, smem));
    launched(ctx);
    return true;
}

// key-row stride of the deferred NDC tables: a power of two >= max(K, 32)
static int ndc_key_stride(int K) {
    const int p = kpow_of(K);
    return p < 32 ? 32 : p;
}
// prefix codes per row kept in shared memory by ndc_post_kernel
static int ndc_post_prefix(int K, int KS) {
    const int L = K <= 256 ? 64 : 32;
    return L < KS ? L : KS;
}

// The NDC of the WALK iterations t0 .. st->iteration of one persistent launch
// (the count of iterations is read on the device: nothing waits on the host).
static void launch_ndc_post(cqg_ctx *ctx, const SweepArgs &a, const IterArgs &ia, uint32_t *keys, int t0) {
    cudaStream_t s = ctx->stream;
    const int K = a.K, KS = ndc_key_stride(K);
    const size_t ksm = 24 * (size_t)K;
    const unsigned gk = (unsigned)ctx->num_sms * 2;
    switch (KS) {
#define CQG_WALK_KEYS(V)                                                                        \
    case V:                                                                                     \
        if (ksm > 48 * 1024) CQG_CUDA(ensure_smem((const void *)walk_keys_kernel<V>, ksm));     \
        walk_keys_kernel<V><<<gk, 1024, ksm, s>>>(ia.snap_cen, K, ia.st, t0, keys);            \
        break;
        CQG_WALK_KEYS(32)
        CQG_WALK_KEYS(64)
        CQG_WALK_KEYS(128)
        CQG_WALK_KEYS(256)
        CQG_WALK_KEYS(512)
        CQG_WALK_KEYS(1024)
#undef CQG_WALK_KEYS
        default: fail(CQG_E_INVALID, "persistent Lloyd: K above 1024");
    }
    const int L = ndc_post_prefix(K, KS);
    const size_t sm = 24 * (size_t)K + (size_t)K * (L + 2) * sizeof(uint16_t);
    static thread_local size_t c_sm = 0;
    static thread_local int c_dev = -1, c_bps = 1;
    if (c_sm != sm || c_dev != ctx->device) {
        CQG_CUDA(ensure_smem((const void *)ndc_post_kernel<4>, sm));
        int bps = 0;
        CQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, ndc_post_kernel<4>, kNdcPostThreads, sm));
        c_bps = bps < 1 ? 1 : bps;
        c_sm = sm;
        c_dev = ctx->device;
    }
    ndc_post_kernel<4><<<(unsigned)ctx->num_sms * c_bps, kNdcPostThreads, sm, s>>>(
        a.colors, a.n, ia.snap_lab, ia.snap_cen, keys, K, KS, L, ia.st, t0, a.ndc);
    CQG_CUDA(cudaGetLastError());
    launched(ctx, 2);
}

int lloyd_finish(cqg_ctx *ctx, LloydOut &out, uint64_t n, int K) {
    const unsigned char *hsc = static_cast<const unsigned char *>(ctx->pinned.p);
    const IterStatus *hst = reinterpret_cast<const IterStatus *>(hsc + 32);
    const unsigned long long *hcnt = reinterpret_cast<const unsigned long long *>(hsc); // ndc, flagged
    out.pending = false;
    out.iterations = hst->iteration;
    prof_add_units(ctx, out.prof_rec, (double)n * (double)K * (double)out.iterations);
    out.ndc = hcnt[0];
    out.flagged = hcnt[1];
    out.swept = ctx->lloyd_prune_pending ? hcnt[12] + n : n * (unsigned long long)out.iterations;
    return hst->state;
}

LloydOut lloyd_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n,
                   uint64_t P, const double *init_d, int K, const cqg_term &term, uint32_t *labels_d,
                   double *centers_d, double *sse_host, uint32_t *hist_labels_user,
                   double *hist_centers_user, bool allow_defer) {
    cudaStream_t s = ctx->stream;
    const int Kp = pad_centres(K);
    const int limit = term.fixed_iterations > 0 ? term.fixed_iterations : term.max_iterations;
    double *cen = centers_d;
    CQG_CUDA(cudaMemcpyAsync(cen, init_d, sizeof(double) * 3 * K, cudaMemcpyDeviceToDevice, s));
    float *fc = static_cast<float *>(ctx->fcen.ensure(sizeof(float) * (4 * (size_t)Kp + 8)));
    float *tau = fc + 4 * Kp;
    double *dtab = static_cast<double *>(ctx->dtab.ensure(sizeof(double) * (size_t)K * K));
    int Kpow = 1;
    while (Kpow < K) Kpow <<= 1;
    double *dsorted = static_cast<double *>(ctx->dsorted.ensure(sizeof(double) * (size_t)K * Kpow));
    uint16_t *dcode = K <= kNdcCodeMaxK && ctx->use_ndc_code
                          ? static_cast<uint16_t *>(ctx->dcode.ensure(sizeof(uint16_t) * (size_t)K * Kpow + 16))
                          : nullptr;
    uint32_t *order = static_cast<uint32_t *>(ctx->order.ensure(sizeof(uint32_t) * (size_t)K * K));
    Moments *mom = static_cast<Moments *>(ctx->mom.ensure(sizeof(Moments) * (size_t)K));
    uint32_t *queue = static_cast<uint32_t *>(ctx->queue.ensure(sizeof(uint32_t) * (n + 1)));
    uint32_t *qn = static_cast<uint32_t *>(ctx->scal.ensure(256));
    unsigned long long *ndc = reinterpret_cast<unsigned long long *>(qn + 8);
    unsigned long long *flagged = reinterpret_cast<unsigned long long *>(qn + 10);
    int *iter_dev = reinterpret_cast<int *>(qn + 12);
    IterStatus *st = reinterpret_cast<IterStatus *>(qn + 16);
    unsigned long long *swept = reinterpret_cast<unsigned long long *>(qn + 32);
    int *shift_inval = reinterpret_cast<int *>(qn + 36);
    const bool prune = ctx->use_prune;
    float2 *bnd = prune ? static_cast<float2 *>(ctx->bnd.ensure(sizeof(float2) * (n + 1))) : nullptr;
    float *shift = prune ? static_cast<float *>(ctx->shift.ensure(sizeof(float) * ((size_t)K + 4))) : nullptr;
    double *sse_d = static_cast<double *>(ctx->sse.ensure(sizeof(double) * (size_t)(limit + 1)));
    // pinned read-back of scalar bytes 32..136: ndc, flagged, iter_dev, IterStatus (byte 64), swept (byte 128)
    unsigned char *hsc = static_cast<unsigned char *>(ctx->pinned.ensure(4096));
    IterStatus *hst = reinterpret_cast<IterStatus *>(hsc + 32);
    const bool hist = term.record_history && (hist_labels_user || hist_centers_user);
    uint32_t *hl_d = nullptr;
    double *hc_d = nullptr;
    if (hist) {
        hl_d = static_cast<uint32_t *>(ctx->hist_labels.ensure(sizeof(uint32_t) * n * (size_t)limit));
        hc_d = static_cast<double *>(ctx->hist_centers.ensure(sizeof(double) * 3 * (size_t)K * limit));
    }

    const bool use_graph = !hist && ctx->use_graphs;
    // small substrates: the whole loop as one persistent cooperative kernel
    // (every block builds its own FP32 table: no fc_kernel launch)
    const bool persistent = use_graph && K <= 1024 &&
                            n <= (uint64_t)ctx->dev_sms * 2 * kSweepThreads * 4 * 2;
    // persistent loop: the walk tables and the NDC leave the loop (deferred
    // NDC over per-iteration snapshots, win iterations per launch)
    double *rowmin = nullptr, *snap_cen = nullptr;
    uint16_t *snap_lab = nullptr;
    uint32_t *ndc_keys = nullptr;
    Moments *dmom = nullptr;
    int win = 0;
    if (persistent) {
        const int KS = ndc_key_stride(K);
        uint64_t w = (uint64_t)limit;
        const uint64_t wl = (128ull << 20) / (2 * n + 2), wk = (64ull << 20) / (4ull * K * KS);
        if (w > wl) w = wl;
        if (w > wk) w = wk;
        if (ctx->dbg_ndc_win > 0 && w > (uint64_t)ctx->dbg_ndc_win) w = (uint64_t)ctx->dbg_ndc_win;
        win = w < 1 ? 1 : (int)w;
        rowmin = static_cast<double *>(ctx->rowmin.ensure(sizeof(double) * (size_t)K));
        snap_cen = static_cast<double *>(ctx->snap_cen.ensure(24 * (size_t)K * win));
        snap_lab = static_cast<uint16_t *>(ctx->snap_lab.ensure(2 * n * (size_t)win + 16));
        ndc_keys = static_cast<uint32_t *>(ctx->ndc_keys.ensure(4 * (size_t)K * KS * win));
        dmom = static_cast<Moments *>(ctx->dmom.ensure(3 * sizeof(Moments) * (size_t)K));
        dcode = nullptr; // no walk rows inside the loop
    }
    CQG_CUDA(cudaMemsetAsync(mom, 0, sizeof(Moments) * (size_t)K, s));
    // one memset for the scalars: queue counter, ndc, flagged, iter_dev, status, swept, shift_inval
    CQG_CUDA(cudaMemsetAsync(qn, 0, 160, s));
    if (!persistent) {
        fc_kernel<<<1, 256, 0, s>>>(cen, K, Kp, fc, tau);
        launched(ctx);
    }

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
    a.Kpow = Kpow;
    a.bnd = bnd;
    a.shift = shift;
    a.dcode = dcode;
    a.swept = swept;
    std::memcpy(ctx->last_sweep, &a, sizeof(SweepArgs)); // for cqg_bench_sweep
    ctx->have_last_sweep = true;

    IterArgs ia{};
    ia.mom = mom;
    ia.cen = cen;
    ia.K = K;
    ia.Kp = Kp;
    ia.P = P;
    ia.n_points = n;
    ia.eps = term.epsilon;
    ia.limit = limit;
    ia.fixed = term.fixed_iterations;
    ia.sse_arr = sse_d;
    ia.st = st;
    ia.iter_dev = iter_dev;
    ia.qn = qn;
    ia.ndc = ndc;
    ia.flagged = flagged;
    ia.fc = fc;
    ia.tau = tau;
    ia.dtab = dtab;
    ia.dsorted = dsorted;
    ia.order = order;
    ia.Kpow = Kpow;
    ia.use_cond = 0;
    ia.shift = shift;
    ia.shift_inval = shift_inval;
    ia.dcode = dcode;
    a.rowmin = rowmin;
    ia.rowmin = rowmin;
    if (!persistent && prune && dcode && K <= kNdcCodeMaxK && Kpow >= 8 && ctx->use_filter_list) {
        a.surv = static_cast<uint32_t *>(ctx->survivors.ensure(4 * (n + 8)));
        CQG_CUDA(ensure_smem((const void *)ndc_code_kernel<4>,
                             kNdcCodeMaxK * 24 + kNdcCodeMaxK * (kNdcCodeMaxK + 2) * 2));
        sweep_list_setup(ctx, K, Kp);
    }
    ia.no_walk_rows = persistent ? 1 : 0;
    ia.snap_cen = snap_cen;
    ia.snap_lab = snap_lab;
    ia.win = win;
    ia.dmom = dmom;

    // The graph path needs no per-iteration host work: used unless history is
    // recorded (per-iteration copies) or kernel profiling is on (per-launch events).
    LloydOut out;
    int iter = 0;
    bool done = false;
    while (!done) {
        const bool first = (iter == 0);
        int rec = -1;
        const int before = iter;
        if (persistent) {
            // a launch rewrites the snapshots an earlier launch's NDC pass reads
            CQG_CUDA(cudaStreamWaitEvent(s, ctx->lloyd_join, 0));
            const int pb = prof_begin(ctx);
            if (!launch_persistent(ctx, a, ia, first)) fail(CQG_E_CUDA, "persistent Lloyd kernel does not fit");
            rec = prof_end(ctx, CQG_PROF_LLOYD, pb, 0.0);
            // the deferred NDC on the side stream, beside what follows on this
            // one (the mapping); its counter is read back from there
            CQG_CUDA(cudaEventRecord(ctx->lloyd_fork, s));
            CQG_CUDA(cudaStreamWaitEvent(ctx->aux2, ctx->lloyd_fork, 0));
            {
                struct SideStream { // launches and profiling events below go to the side stream
                    cqg_ctx *c;
                    cudaStream_t main;
                    ~SideStream() { c->stream = main; }
                } side{ctx, s};
                ctx->stream = ctx->aux2;
                const int pn = prof_begin(ctx);
                launch_ndc_post(ctx, a, ia, ndc_keys, first ? 2 : iter + 1);
                prof_end(ctx, CQG_PROF_NDC, pn, 0.0);
                CQG_CUDA(cudaMemcpyAsync(hsc, reinterpret_cast<unsigned char *>(qn) + 32, 8, cudaMemcpyDeviceToHost,
                                         ctx->aux2));
                CQG_CUDA(cudaEventRecord(ctx->lloyd_join, ctx->aux2));
            }
        } else if (!first && use_graph) {
            cudaGraphExec_t ge = loop_graph(ctx, a, ia, qn);
            const int pb = prof_begin(ctx);
            CQG_CUDA(cudaGraphLaunch(ge, s));
            rec = prof_end(ctx, CQG_PROF_LLOYD, pb, 0.0);
            launched(ctx, 4);
        } else {
            CQG_CUDA(cudaMemsetAsync(qn, 0, 4, s));
            launch_sweep(ctx, first ? MODE_FULL : MODE_WALK, a);
            if (hist) {
                if (hist_labels_user)
                    CQG_CUDA(cudaMemcpyAsync(hl_d + (size_t)iter * n, labels_d, 4 * n, cudaMemcpyDeviceToDevice, s));
                if (hist_centers_user)
                    CQG_CUDA(cudaMemcpyAsync(hc_d + (size_t)iter * 3 * K, cen, 24 * (size_t)K,
                                             cudaMemcpyDeviceToDevice, s));
            }
            launch_iter_end(ctx, ia);
        }
        // one read-back per launch: counters, status (scalars bytes 32..136) and
        // the SSE trace (the persistent path reads the NDC, bytes 32..40, on the side stream)
        if (persistent)
            CQG_CUDA(cudaMemcpyAsync(hsc + 8, reinterpret_cast<unsigned char *>(qn) + 40, 96, cudaMemcpyDeviceToHost, s));
        else
            CQG_CUDA(cudaMemcpyAsync(hsc, reinterpret_cast<unsigned char *>(qn) + 32, 104, cudaMemcpyDeviceToHost, s));
        if (sse_host) CQG_CUDA(cudaMemcpyAsync(sse_host, sse_d, sizeof(double) * (size_t)limit, cudaMemcpyDefault, s));
        if (persistent && first && allow_defer) {
            // the persistent kernel ends done (state 1) or on an empty cluster
            // (state 2): let the caller enqueue the mapping behind it and check
            // after its own synchronisation (lloyd_finish)
            out.pending = true;
            out.prof_rec = rec;
            if (prune) {
                out.labels = labels_d;
                out.bnd = bnd;
                out.shift = shift;
                out.rowmin = rowmin; // the persistent loop built no walk table
                out.mom = mom;
                out.Kpow = Kpow;
            }
            ctx->lloyd_prune_pending = prune;
            return out;
        }
        CQG_CUDA(cudaStreamSynchronize(s));
        iter = hst->iteration;
        prof_add_units(ctx, rec, (double)n * (double)K * (double)(iter - before));
        if (hst->state == 2) {
            out.repairs += repair_loop(ctx, colors_d, counts_d, n, P, K, labels_d, cen, mom, shift_inval);
            IterArgs ib = ia;
            ib.reset_qn = persistent ? 1 : 0;
            launch_iter_end(ctx, ib);
            // (the persistent path's NDC counter may still be growing on the side stream)
            CQG_CUDA(cudaMemcpyAsync(hsc + 8, reinterpret_cast<unsigned char *>(qn) + 40, 96, cudaMemcpyDeviceToHost, s));
            if (sse_host) CQG_CUDA(cudaMemcpyAsync(sse_host, sse_d, sizeof(double) * (size_t)limit, cudaMemcpyDefault, s));
            CQG_CUDA(cudaStreamSynchronize(s));
            if (hst->state == 2) fail(CQG_E_RUNTIME, "repair left an empty cluster");
            iter = hst->iteration;
        }
        done = hst->state == 1;
    }
    out.iterations = iter;
    if (hist) {
        if (hist_labels_user) copy_out(ctx, hist_labels_user, hl_d, sizeof(uint32_t) * n * (size_t)iter);
        if (hist_centers_user) copy_out(ctx, hist_centers_user, hc_d, 24 * (size_t)K * iter);
        CQG_CUDA(cudaStreamSynchronize(s));
    }
    if (persistent) {
        // the NDC counter after the side stream's last pass (and any repair's
        // finalise on this stream; the repair also reuses the pinned buffer)
        CQG_CUDA(cudaStreamWaitEvent(s, ctx->lloyd_join, 0));
        CQG_CUDA(cudaMemcpyAsync(hsc, reinterpret_cast<unsigned char *>(qn) + 32, 8, cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaStreamSynchronize(s));
    }
    const unsigned long long *hcnt = reinterpret_cast<const unsigned long long *>(hsc); // ndc, flagged
    out.ndc = hcnt[0];
    out.flagged = hcnt[1];
    // FULL first iteration sweeps every point; WALK iterations count the survivors
    out.swept = prune ? hcnt[12] + n : n * (unsigned long long)iter; // swept: scalar byte 128
    if (prune) { // bounds of the last assignment, shifts to the final centres, their walk table
        out.labels = labels_d;
        out.bnd = bnd;
        out.shift = shift;
        if (persistent) {
            out.rowmin = rowmin;
        } else {
            out.dsorted = dsorted;
            out.dcode = dcode;
        }
        out.mom = mom;
        out.Kpow = Kpow;
    }
    return out;
}


// ---------------------------------------------------------------------------
// Sharded Lloyd (one huge image over ranks): the caller allreduces the packed
// partials between cqg_shard_assign and cqg_shard_finalize.

struct ShardState {
    SweepArgs a;
    IterArgs ia;
    uint64_t n = 0, P = 0;
    int K = 0, iter = 0, limit = 0;
    int pending = 0;        // iterations finalised without a host read (cqg_shard_finalize_async)
    int32_t *slog = nullptr; // device log: the state of each pending iteration
};

namespace {
__global__ void pack_partial_kernel(const Moments *mom, int K, const unsigned long long *ndc, const uint32_t *qn,
                                    long long extra_ndc, int with_counts, long long *out) {
    const long long *m = reinterpret_cast<const long long *>(mom);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 5 * K; i += gridDim.x * blockDim.x) out[i] = m[i];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[5 * K] = with_counts ? (long long)(*ndc) + extra_ndc : 0;
        out[5 * K + 1] = with_counts ? (long long)(*qn) : 0;
    }
}

__global__ void set_centre_kernel(double *cen, int e, uint32_t c) {
    if (threadIdx.x == 0) {
        cen[3 * e] = (double)((c >> 16) & 255u);
        cen[3 * e + 1] = (double)((c >> 8) & 255u);
        cen[3 * e + 2] = (double)(c & 255u);
    }
}
} // namespace

static ShardState &shard_state(cqg_ctx *ctx) {
    if (!ctx->shard) fail(CQG_E_INVALID, "cqg_shard: call cqg_shard_begin first");
    return *static_cast<ShardState *>(ctx->shard);
}

void shard_release(cqg_ctx *ctx) {
    delete static_cast<ShardState *>(ctx->shard);
    ctx->shard = nullptr;
}
int shard_k(cqg_ctx *ctx) { return shard_state(ctx).K; }
uint64_t shard_n(cqg_ctx *ctx) { return shard_state(ctx).n; }

void shard_begin_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n, uint64_t P,
                     const double *init_d, int K, const cqg_term &term) {
    cudaStream_t s = ctx->stream;
    if (!ctx->shard) ctx->shard = new ShardState();
    ShardState &S = *static_cast<ShardState *>(ctx->shard);
    const int Kp = pad_centres(K);
    int Kpow = 1;
    while (Kpow < K) Kpow <<= 1;
    S = ShardState();
    S.n = n;
    S.P = P;
    S.K = K;
    S.limit = term.fixed_iterations > 0 ? term.fixed_iterations : term.max_iterations;
    double *cen = static_cast<double *>(ctx->cen.ensure(24 * (size_t)K));
    CQG_CUDA(cudaMemcpyAsync(cen, init_d, 24 * (size_t)K, cudaMemcpyDeviceToDevice, s));
    float *fc = static_cast<float *>(ctx->fcen.ensure(sizeof(float) * (4 * (size_t)Kp + 8)));
    double *dtab = static_cast<double *>(ctx->dtab.ensure(sizeof(double) * (size_t)K * K));
    double *dsorted = static_cast<double *>(ctx->dsorted.ensure(sizeof(double) * (size_t)K * Kpow));
    uint32_t *order = static_cast<uint32_t *>(ctx->order.ensure(sizeof(uint32_t) * (size_t)K * K));
    Moments *mom = static_cast<Moments *>(ctx->mom.ensure(sizeof(Moments) * (size_t)K));
    Moments *mom_g = static_cast<Moments *>(ctx->mom_g.ensure(sizeof(Moments) * (size_t)K));
    uint32_t *queue = static_cast<uint32_t *>(ctx->queue.ensure(sizeof(uint32_t) * (n + 1)));
    uint32_t *labels = static_cast<uint32_t *>(ctx->labels.ensure(sizeof(uint32_t) * (n + 1)));
    uint32_t *qn = static_cast<uint32_t *>(ctx->scal.ensure(256));
    unsigned long long *ndc = reinterpret_cast<unsigned long long *>(qn + 8);
    unsigned long long *flagged = reinterpret_cast<unsigned long long *>(qn + 10);
    int *iter_dev = reinterpret_cast<int *>(qn + 12);
    IterStatus *st = reinterpret_cast<IterStatus *>(qn + 16);
    unsigned long long *ndc_unused = reinterpret_cast<unsigned long long *>(qn + 24);
    unsigned long long *swept = reinterpret_cast<unsigned long long *>(qn + 32);
    int *shift_inval = reinterpret_cast<int *>(qn + 36);
    // distance-bound pruning and the NDC code table, as in lloyd_dev: every rank
    // finalises identically, so every rank computes the same centre shifts
    const bool prune = ctx->use_prune;
    float2 *bnd = prune && n ? static_cast<float2 *>(ctx->bnd.ensure(sizeof(float2) * (n + 1))) : nullptr;
    float *shift = prune ? static_cast<float *>(ctx->shift.ensure(sizeof(float) * ((size_t)K + 4))) : nullptr;
    uint16_t *dcode = K <= kNdcCodeMaxK && ctx->use_ndc_code
                          ? static_cast<uint16_t *>(ctx->dcode.ensure(sizeof(uint16_t) * (size_t)K * Kpow + 16))
                          : nullptr;
    double *sse_d = static_cast<double *>(ctx->sse.ensure(sizeof(double) * (size_t)(S.limit + 1)));
    CQG_CUDA(cudaMemsetAsync(mom, 0, sizeof(Moments) * (size_t)K, s));
    CQG_CUDA(cudaMemsetAsync(qn, 0, 160, s));
    fc_kernel<<<1, 256, 0, s>>>(cen, K, Kp, fc, fc + 4 * Kp);
    launched(ctx);
    SweepArgs &a = S.a;
    a = SweepArgs{};
    a.colors = colors_d;
    a.counts = counts_d;
    a.n = n;
    a.labels = labels;
    a.fc = fc;
    a.cen = cen;
    a.dtab = dtab;
    a.dsorted = dsorted;
    a.order = order;
    a.tau = fc + 4 * Kp;
    a.queue = queue;
    a.qn = qn;
    a.mom = mom;
    a.ndc = ndc;
    a.K = K;
    a.Kp = Kp;
    a.Kpow = Kpow;
    a.bnd = bnd;
    a.shift = shift;
    a.swept = swept;
    a.dcode = dcode;
    IterArgs &ia = S.ia;
    ia = IterArgs{};
    ia.shift = shift;
    ia.shift_inval = shift_inval;
    ia.dcode = dcode;
    ia.mom = mom_g;
    ia.cen = cen;
    ia.K = K;
    ia.Kp = Kp;
    ia.P = P;
    ia.n_points = 0; // NDC is summed from the ranks' partials
    ia.eps = term.epsilon;
    ia.limit = S.limit;
    ia.fixed = term.fixed_iterations;
    ia.sse_arr = sse_d;
    ia.st = st;
    ia.iter_dev = iter_dev;
    ia.qn = qn;
    ia.ndc = ndc_unused;
    ia.flagged = flagged;
    ia.fc = fc;
    ia.tau = fc + 4 * Kp;
    ia.dtab = dtab;
    ia.dsorted = dsorted;
    ia.order = order;
    ia.Kpow = Kpow;
    ia.use_cond = 0;
    ia.reset_qn = 1;
}

void shard_assign_dev(cqg_ctx *ctx, long long *partial_d, bool run) {
    ShardState &S = shard_state(ctx);
    cudaStream_t s = ctx->stream;
    long long extra = 0;
    if (run) {
        CQG_CUDA(cudaMemsetAsync(S.a.qn, 0, 4, s));
        CQG_CUDA(cudaMemsetAsync(S.a.ndc, 0, 8, s));
        if (S.n > 0) {
            if (S.iter == 0) {
                launch_sweep(ctx, MODE_FULL, S.a);
                extra = (long long)S.n * (long long)S.K; // nearest_full: K per point
            } else {
                launch_sweep(ctx, MODE_WALK, S.a);
            }
        }
    }
    pack_partial_kernel<<<1, 256, 0, s>>>(S.a.mom, S.K, S.a.ndc, S.a.qn, extra, run ? 1 : 0, partial_d);
    launched(ctx);
    CQG_CUDA(cudaGetLastError());
}


// Finalise without a host synchronisation: the iteration's state is appended
// to a device log and the host assumes "continue" (iter + 1). shard_status_dev
// reads the log once: a fixed-iteration run needs no per-iteration round trip.
void shard_finalize_async_dev(cqg_ctx *ctx, const long long *global_d) {
    ShardState &S = shard_state(ctx);
    cudaStream_t s = ctx->stream;
    if (!S.slog) S.slog = static_cast<int32_t *>(ctx->shard_log.ensure(sizeof(int32_t) * 4096));
    if (S.pending >= 4096) fail(CQG_E_INVALID, "cqg_shard_finalize_async: more than 4096 pending iterations");
    CQG_CUDA(cudaMemcpyAsync(S.ia.mom, global_d, sizeof(Moments) * (size_t)S.K, cudaMemcpyDeviceToDevice, s));
    launch_iter_end(ctx, S.ia);
    CQG_CUDA(cudaMemcpyAsync(S.slog + S.pending, &S.ia.st->state, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
    ++S.pending;
    ++S.iter; // the next assignment walks (WALK mode) unless the log says otherwise
}

// 0: every pending iteration continued, 1: the last one finished and none
// before it stopped, 2: some iteration hit an empty cluster or stopped early
// (the run must be redone with the synchronous protocol)
int shard_status_dev(cqg_ctx *ctx, int *iterations) {
    ShardState &S = shard_state(ctx);
    int result = 0;
    if (S.pending) {
        std::vector<int32_t> h(S.pending);
        CQG_CUDA(cudaMemcpyAsync(h.data(), S.slog, sizeof(int32_t) * S.pending, cudaMemcpyDeviceToHost, ctx->stream));
        CQG_CUDA(cudaStreamSynchronize(ctx->stream));
        for (int i = 0; i < S.pending; ++i) {
            if (h[i] == 2 || (h[i] == 1 && i + 1 < S.pending)) result = 2;
            else if (h[i] == 1 && result == 0) result = 1;
        }
        S.pending = 0;
    }
    if (iterations) *iterations = S.iter;
    return result;
}

int shard_finalize_dev(cqg_ctx *ctx, const long long *global_d, double *sse) {
    ShardState &S = shard_state(ctx);
    cudaStream_t s = ctx->stream;
    CQG_CUDA(cudaMemcpyAsync(S.ia.mom, global_d, sizeof(Moments) * (size_t)S.K, cudaMemcpyDeviceToDevice, s));
    launch_iter_end(ctx, S.ia);
    IterStatus *hst = static_cast<IterStatus *>(ctx->pinned.ensure(4096));
    CQG_CUDA(cudaMemcpyAsync(hst, S.ia.st, sizeof(IterStatus), cudaMemcpyDeviceToHost, s));
    CQG_CUDA(cudaStreamSynchronize(s));
    if (hst->state != 2) S.iter = hst->iteration;
    if (sse) *sse = hst->sse;
    return hst->state;
}

void shard_sizes_dev(cqg_ctx *ctx, uint32_t *sizes_d) {
    ShardState &S = shard_state(ctx);
    CQG_CUDA(cudaMemsetAsync(sizes_d, 0, 4 * (size_t)S.K, ctx->stream));
    if (S.n > 0) sizes_kernel<<<pick_grid(ctx, S.n, 256, 2), 256, 0, ctx->stream>>>(S.a.labels, S.n, sizes_d);
    launched(ctx);
}

void shard_donor_dev(cqg_ctx *ctx, const uint32_t *gsizes_d, int fallback, double *value, uint64_t *index,
                     uint32_t *colour, uint32_t *label) {
    ShardState &S = shard_state(ctx);
    cudaStream_t s = ctx->stream;
    *value = -2.0;
    *index = ~0ull;
    *colour = 0;
    *label = 0;
    if (S.n == 0) return;
    const int nparts = pick_grid(ctx, S.n, 256, 2);
    ValIdx *part = static_cast<ValIdx *>(ctx->red.ensure(sizeof(ValIdx) * (size_t)nparts));
    argmax_kernel<<<nparts, 256, 0, s>>>(S.a.colors, S.a.counts, S.a.labels, S.n, S.a.cen, 1.0 / (double)S.P,
                                         gsizes_d, fallback, part);
    argmax_final<<<1, 32, 0, s>>>(part, nparts);
    launched(ctx, 2);
    ValIdx *h = static_cast<ValIdx *>(ctx->pinned.ensure(4096));
    CQG_CUDA(cudaMemcpyAsync(h, part, sizeof(ValIdx), cudaMemcpyDeviceToHost, s));
    CQG_CUDA(cudaStreamSynchronize(s));
    const ValIdx best = *h;
    *value = best.v;
    *index = best.i;
    if (best.i < S.n) {
        uint32_t *h32 = reinterpret_cast<uint32_t *>(h + 1);
        CQG_CUDA(cudaMemcpyAsync(h32, S.a.colors + best.i, 4, cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaMemcpyAsync(h32 + 1, S.a.labels + best.i, 4, cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaStreamSynchronize(s));
        *colour = h32[0];
        *label = h32[1];
    }
}

void shard_move_dev(cqg_ctx *ctx, uint64_t index, int e, uint32_t colour) {
    ShardState &S = shard_state(ctx);
    cudaStream_t s = ctx->stream;
    if (index < S.n) {
        uint32_t *sizes = static_cast<uint32_t *>(ctx->sizes.ensure((size_t)S.K * 4));
        apply_move_kernel<<<1, 32, 0, s>>>(S.a.colors, S.a.counts, S.a.labels, S.ia.cen, S.a.mom, sizes, index, e,
                                            S.ia.shift_inval);
    } else {
        set_centre_kernel<<<1, 32, 0, s>>>(S.ia.cen, e, colour);
        // the centres moved outside the bounds' bookkeeping on this rank too
        if (S.ia.shift_inval) CQG_CUDA(cudaMemsetAsync(S.ia.shift_inval, 0x01, 1, s));
    }
    launched(ctx);
    CQG_CUDA(cudaGetLastError());
}

int shard_end_dev(cqg_ctx *ctx, double *centers_user, uint32_t *labels_user, double *sse_user) {
    ShardState &S = shard_state(ctx);
    copy_out(ctx, centers_user, S.a.cen, 24 * (size_t)S.K);
    copy_out(ctx, labels_user, S.a.labels, 4 * S.n);
    copy_out(ctx, sse_user, S.ia.sse_arr, 8 * (size_t)S.iter);
    CQG_CUDA(cudaStreamSynchronize(ctx->stream));
    return S.iter;
}

} // namespace cqg

#ifdef CQG_INIT_TIMING
extern "C" int cqg_dbg_lloyd_timing(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_lloyd_timing, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(cqg::g_lloyd_timing, z, sizeof(z));
    }
    return 0;
}
#endif

#ifdef CQG_INIT_TIMING
extern "C" int cqg_dbg_block_timing(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_block_timing, 1024 * 3 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    if (reset) {
        static unsigned long long z[1024 * 3] = {};
        cudaMemcpyToSymbol(cqg::g_block_timing, z, sizeof(z));
    }
    return 0;
}
#endif

#ifdef CQG_SWEEP_TIMING
extern "C" int cqg_dbg_sweep_timing(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_sweep_timing, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(cqg::g_sweep_timing, z, sizeof(z));
    }
    return 0;
}
#endif
