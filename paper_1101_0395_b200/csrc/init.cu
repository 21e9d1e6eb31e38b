// init.cu -- maximin and k-means++ initialisers on the device, bit-exact with
// the reference (src/init.cpp:37-52, 127-138, 295-314; rng.hpp:43-54).
//
// Centres are histogram colours, so every distance is an exact integer; the
// running min-distances are uint32. One persistent cooperative kernel runs all
// K rounds with ONE grid barrier per round:
//
//   update   block b owns a contiguous index range (segments of 1024 points);
//            mind2 = min(mind2, d2(x, c_last)) into a ping-pong buffer, plus
//            either the packed (mind2, ~index) maximum (maximin) or the exact
//            mass sums per segment and per block (k-means++).
//   barrier  grid.sync()
//   select   every block redundantly finds the same winner:
//            maximin  warp max over block partials (lowest index on ties,
//                     init.cpp:43-46);
//            draw     masses m_i = fl(fl(count_i * (1/P)) * mind2_i), formed as
//                     the reference forms them, summed EXACTLY in 128-bit fixed
//                     point (2^-88 units). u = fl(unit * total) is located by
//                     warp scans over block sums, then segment sums, then a
//                     block scan inside the 1024-point segment.
//            When P is a power of two every mass is an integer multiple of 1/P
//            and all prefix sums stay below 2^53/P, so the reference's
//            sequential FP64 sums are exact and the located index IS the
//            reference's. Otherwise the decision is accepted only when u is
//            farther than a rigorous bound on the sequential rounding from
//            both neighbouring prefix sums, and one thread replays the
//            reference's sequential weighted_draw when it is not (counted).
#include <cooperative_groups.h>

#include <random>

#include "cqg_internal.cuh"

#include <cstring>

namespace cg = cooperative_groups;

namespace cqg {
namespace {

typedef unsigned __int128 u128;
constexpr int kFix = 88;        // fixed-point fraction bits
constexpr int kInitThreads = 256;
constexpr int kSeg = 1024;      // points per segment (4 per thread)
constexpr uint32_t kWeightsOnly = 0xFFFFFFFFu;
constexpr int kLocateMax = 448; // block sums / segments one warp_locate scans (registers): 3 x 148 blocks

struct InitArgs {
    const uint32_t *colors;
    const uint32_t *counts;
    uint64_t n;
    double inv;
    int K;
    int kind;            // 0 maximin, 1 k-means++
    int weighted_first;  // maximin only
    int exact_sums;      // P is a power of two: sequential FP64 sums are exact
    uint64_t first_index;
    uint64_t chunk;      // points per block (multiple of kSeg)
    const double *nu;    // unit draws, in consumption order
    uint32_t *md;        // 2 x n ping-pong min distances (init_kernel) or n x {colour, md} (init_kernel_rec)
    int mds;             // stride of md values in `md` seen by the locate (1, or 2 for records)
    u128 *parts;         // 2 x gridDim block mass sums
    u128 *segs;          // 2 x nseg segment mass sums
    unsigned long long *mparts; // 2 x gridDim maximin keys
    unsigned long long *result; // [2] fallback result slots
    unsigned long long *fallbacks;
    double *cen;
    int force_seq;       // tests only (CQG_DBG_INIT_FORCE_SEQ): 1 every draw ambiguous, 2 every draw "beyond every prefix"
    // colour-space tiles (init_kernel_tile): points in Morton order of their
    // colour, kTile per tile; md values are read through hpos (histogram
    // index -> tile position) by the locate
    const uint32_t *hpos; // null: md is indexed by histogram position
    const uint32_t *tcol; // colour of each tile-order point
    uint32_t *tmd;        // md of each tile-order point
    const uint32_t *tidx; // histogram index of each tile-order point
    const uint32_t *tcnt; // count of each tile-order point (k-means++)
    const uint2 *tbox;    // per tile: packed min / max colour channels
    uint32_t *tmax;       // per tile: largest md
    unsigned long long *tkey; // per tile (maximin): largest (md, ~index)
    uint64_t ntiles;
    unsigned long long *tflags; // per block release words (kFlagStride apart), zero at launch
};

// md of histogram point i (direct, or through the tile layout)
__device__ __forceinline__ uint32_t md_at(const InitArgs &a, const uint32_t *md, uint64_t i) {
    return md[(a.hpos ? (uint64_t)a.hpos[i] : i) * (uint64_t)a.mds];
}

__device__ __forceinline__ u128 to_fixed(double m) {
    if (m == 0.0) return 0;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(m);
    const int e = (int)((bits >> 52) & 0x7FF);
    const unsigned long long mant = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    const int s = e - 1075 + kFix; // >= 0 for m >= 2^-36, i.e. P < 2^32
    return s >= 0 ? ((u128)mant) << s : (u128)(mant >> (-s > 63 ? 63 : -s));
}

__device__ __forceinline__ u128 floor_fixed(double u) {
    if (u <= 0.0) return 0;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(u);
    const int e = (int)((bits >> 52) & 0x7FF);
    const unsigned long long mant = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    const int s = e - 1075 + kFix;
    if (s >= 0) return ((u128)mant) << s;
    if (-s >= 64) return 0;
    return (u128)(mant >> (-s));
}

__device__ __forceinline__ double fixed_to_double(u128 x) { return scalbn(u128_to_double(x), -kFix); }

// exact squared distance of two packed 0x00RRGGBB colours with byte dot
// products: |a-b|^2 = a.a + b.b - 2 a.b (IDP4A x2 + IMAD, all < 2^18)
__device__ __forceinline__ uint32_t d2_int(uint32_t a, uint32_t b) {
    return __dp4a(a, a, __dp4a(b, b, 0u)) - 2u * __dp4a(a, b, 0u);
}
// same with the centre's b.b precomputed
__device__ __forceinline__ uint32_t d2_int_bb(uint32_t a, uint32_t b, uint32_t bb) {
    return __dp4a(a, a, bb) - 2u * __dp4a(a, b, 0u);
}

// the reference's mass: weights[i] (* mind2[i])
__device__ __forceinline__ double mass_c(uint32_t cnt, double inv, uint32_t md) {
    const double w = __dmul_rn((double)cnt, inv);
    return md == kWeightsOnly ? w : __dmul_rn(w, (double)md);
}
__device__ __forceinline__ double mass_of(const InitArgs &a, uint64_t i, uint32_t md) {
    return mass_c(a.counts[i], a.inv, md);
}

__device__ __forceinline__ u128 shfl_u128(u128 v, int src) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    lo = __shfl_sync(0xffffffffu, lo, src);
    hi = __shfl_sync(0xffffffffu, hi, src);
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ u128 shfl_up_u128(u128 v, int d) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)(v >> 64);
    lo = __shfl_up_sync(0xffffffffu, lo, d);
    hi = __shfl_up_sync(0xffffffffu, hi, d);
    return ((u128)hi << 64) | lo;
}

// ---- mass arithmetic -----------------------------------------------------
// Exact: P is a power of two, masses are the integers count*mind2 (the
//        reference's FP64 masses times P, all partial sums < 2^53), u*P is
//        fl(unit * T) exactly; no rounding ambiguity exists.
// Fixed: masses are the reference's FP64 masses in 2^-88 fixed point (u128);
//        decisions closer than a rigorous bound to a prefix boundary replay the
//        reference sequentially.
struct ExactMass {
    typedef unsigned long long T;
    static __device__ __forceinline__ T mass(const InitArgs &a, uint64_t i, uint32_t md) {
        return mass_c(a, a.counts[i], md);
    }
    static __device__ __forceinline__ T mass_c(const InitArgs &, uint32_t cnt, uint32_t md) {
        return md == kWeightsOnly ? (T)cnt : (T)cnt * (T)md;
    }
    static __device__ __forceinline__ T target(double nu, T total) {
        return (T)floor(__dmul_rn(nu, (double)total)); // u * P, exact scaling
    }
    static __device__ __forceinline__ T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
    static __device__ __forceinline__ T shfl_up(T v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
    static __device__ __forceinline__ T bound(uint64_t, T) { return 0; }
    static constexpr bool exact = true;
};

struct FixedMass {
    typedef u128 T;
    static __device__ __forceinline__ T mass(const InitArgs &a, uint64_t i, uint32_t md) {
        return to_fixed(mass_of(a, i, md));
    }
    static __device__ __forceinline__ T mass_c(const InitArgs &a, uint32_t cnt, uint32_t md) {
        return to_fixed(cqg::mass_c(cnt, a.inv, md));
    }
    static __device__ __forceinline__ T target(double nu, T total) {
        return floor_fixed(__dmul_rn(nu, fixed_to_double(total)));
    }
    static __device__ __forceinline__ T shfl(T v, int src) { return shfl_u128(v, src); }
    static __device__ __forceinline__ T shfl_up(T v, int d) { return shfl_up_u128(v, d); }
    // |reference prefix (or u) - exact| <= (n+4) * 2^-52 * T, doubled
    static __device__ __forceinline__ T bound(uint64_t n, T total) {
        return (u128)2 * (u128)(n + 4) * ((total >> 52) + 1) + 2;
    }
    static constexpr bool exact = false;
};

template <class M>
__device__ __forceinline__ typename M::T warp_incl(typename M::T v) {
    const int lane = threadIdx.x & 31;
    for (int o = 1; o < 32; o <<= 1) {
        const typename M::T t = M::shfl_up(v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Warp-cooperative: arr[0..cnt) held in registers (lane l owns the contiguous
// run [l*R, l*R+R)). Returns the first j whose inclusive prefix exceeds U
// (cnt if none), the exclusive prefix before it, and the total. When
// want_total_first, U is computed from the total by `target` first.
template <class M>
__device__ int warp_locate(const typename M::T *arr, int cnt, bool from_total, double nu,
                           typename M::T &U, typename M::T *before, typename M::T *total) {
    typedef typename M::T T;
    constexpr int RMAX = kLocateMax / 32; // cnt <= kLocateMax (the host caps grids and segments)
    const int lane = threadIdx.x & 31;
    const int R = (cnt + 31) / 32;
    T v[RMAX];
    T loc = 0;
#pragma unroll
    for (int r = 0; r < RMAX; ++r) {
        const int j = lane * R + r;
        v[r] = (r < R && j < cnt) ? arr[j] : (T)0;
        loc += v[r];
    }
    const T incl = warp_incl<M>(loc);
    const T tot = M::shfl(incl, 31);
    if (from_total) U = M::target(nu, tot);
    const T excl = incl - loc;
    const unsigned m = __ballot_sync(0xffffffffu, incl > U);
    int found = cnt;
    T fb = 0;
    if (m) {
        const int l = __ffs(m) - 1;
        if (lane == l) {
            T run = excl;
#pragma unroll
            for (int r = 0; r < RMAX; ++r) {
                if (r < R && found == cnt && run + v[r] > U) {
                    found = lane * R + r;
                    fb = run;
                }
                run += v[r];
            }
        }
        found = __shfl_sync(0xffffffffu, found, l);
        fb = M::shfl(fb, l);
    }
    *before = fb;
    *total = tot;
    return found;
}


template <class M>
__device__ typename M::T block_excl(typename M::T v, typename M::T *s_w, typename M::T *total) {
    typedef typename M::T T;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const T incl = warp_incl<M>(v);
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    T off = 0, tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
        if (i < wid) off += s_w[i];
        tot += s_w[i];
    }
    __syncthreads();
    *total = tot;
    return off + incl - v;
}

// Reference rng.hpp:43-54 replayed sequentially in FP64 (one thread).
__device__ uint64_t sequential_draw(const InitArgs &a, const uint32_t *md, double nu, int weights_only) {
    double total = 0.0;
    for (uint64_t i = 0; i < a.n; ++i)
        total = __dadd_rn(total, mass_of(a, i, weights_only ? kWeightsOnly : md_at(a, md, i)));
    const double u = __dmul_rn(nu, total);
    double acc = 0.0;
    for (uint64_t i = 0; i + 1 < a.n; ++i) {
        acc = __dadd_rn(acc, mass_of(a, i, weights_only ? kWeightsOnly : md_at(a, md, i)));
        if (u < acc) return i;
    }
    return a.n - 1;
}

// Update pass over this block's range: new min distances (unless weights_only)
// and mass sums per segment and per block. One warp per 1024-point segment,
// 8 points per lane loaded before use (memory-level parallelism), no block
// barrier until the block total.
template <class M>
__device__ void update_masses(const InitArgs &a, int par, int weights_only, int first_round, uint32_t clast,
                              const uint32_t *md_in, uint32_t *md_out, uint64_t lo, uint64_t hi,
                              typename M::T *s_w) {
    typedef typename M::T T;
    T *segs = reinterpret_cast<T *>(a.segs) + (size_t)par * ((a.n + kSeg - 1) / kSeg);
    T *parts = reinterpret_cast<T *>(a.parts) + (size_t)par * gridDim.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (hi <= lo + kSeg) {
        // a single segment (small inputs): all warps share it, 4 points per lane
        T loc = 0;
        uint32_t col[4], cnt[4], mi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t i = lo + (uint64_t)u * blockDim.x + threadIdx.x;
            const bool v = i < hi;
            cnt[u] = v ? __ldg(a.counts + i) : 0u;
            col[u] = (v && !weights_only) ? __ldg(a.colors + i) : 0u;
            mi[u] = (v && !weights_only && !first_round) ? md_in[i] : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t i = lo + (uint64_t)u * blockDim.x + threadIdx.x;
            if (i < hi) {
                uint32_t m = kWeightsOnly;
                if (!weights_only) {
                    m = min(mi[u], d2_int(col[u], clast));
                    md_out[i] = m;
                }
                loc += M::mass_c(a, cnt[u], m);
            }
        }
        for (int o = 16; o; o >>= 1) loc += M::shfl(loc, lane ^ o);
        if (lane == 0) s_w[warp] = loc;
        __syncthreads();
        if (threadIdx.x == 0) {
            T t = 0;
            for (int w = 0; w < nw; ++w) t += s_w[w];
            if (lo < hi) segs[lo / kSeg] = t;
            parts[blockIdx.x] = t;
        }
        __syncthreads();
        return;
    }
    T wsum = 0;
    for (uint64_t s0 = lo + (uint64_t)warp * kSeg; s0 < hi; s0 += (uint64_t)nw * kSeg) {
        T loc = 0;
        for (int b = 0; b < kSeg; b += 32 * 8) {
            uint32_t col[8], cnt[8], mi[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t i = s0 + b + u * 32 + lane;
                const bool v = i < hi;
                cnt[u] = v ? __ldg(a.counts + i) : 0u;
                col[u] = (v && !weights_only) ? __ldg(a.colors + i) : 0u;
                mi[u] = (v && !weights_only && !first_round) ? md_in[i] : 0xFFFFFFFFu;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t i = s0 + b + u * 32 + lane;
                if (i < hi) {
                    uint32_t m = kWeightsOnly;
                    if (!weights_only) {
                        m = min(mi[u], d2_int(col[u], clast));
                        md_out[i] = m;
                    }
                    loc += M::mass_c(a, cnt[u], m);
                }
            }
        }
        for (int o = 16; o; o >>= 1) loc += M::shfl(loc, lane ^ o);
        if (lane == 0) segs[s0 / kSeg] = loc;
        wsum += loc;
    }
    if (lane == 0) s_w[warp] = wsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int w = 0; w < nw; ++w) t += s_w[w];
        parts[blockIdx.x] = t;
    }
    __syncthreads();
}

// Every block: locate the draw for unit `nu` over the masses of buffer `par`.
template <class M>
__device__ uint64_t locate_draw(const InitArgs &a, cg::grid_group &grid, int par, double nu, int weights_only,
                                const uint32_t *md, typename M::T *s_w) {
    typedef typename M::T T;
    __shared__ T s_U, s_T, s_before, s_prevE, s_E;
    __shared__ int s_ts;
    __shared__ unsigned long long s_found;
    const uint64_t nseg = (a.n + kSeg - 1) / kSeg;
    const T *parts = reinterpret_cast<const T *>(a.parts) + (size_t)par * gridDim.x;
    const T *segs = reinterpret_cast<const T *>(a.segs) + (size_t)par * nseg;
    if (threadIdx.x < 32) {
        T U = 0, before, tot;
        const int tb = warp_locate<M>(parts, (int)gridDim.x, true, nu, U, &before, &tot);
        int ts = -1;
        T sbefore = before;
        if (tb < (int)gridDim.x) {
            const uint64_t lo = (uint64_t)tb * a.chunk;
            const uint64_t hi = lo + a.chunk < a.n ? lo + a.chunk : a.n;
            const int s0 = (int)(lo / kSeg), s1 = (int)((hi + kSeg - 1) / kSeg);
            if (s1 - s0 == 1) {
                ts = s0;
            } else {
                T U2 = U - before, b2, t2;
                const int j = warp_locate<M>(segs + s0, s1 - s0, false, 0.0, U2, &b2, &t2);
                ts = j < s1 - s0 ? s0 + j : -1;
                sbefore = before + b2;
            }
        }
        if (threadIdx.x == 0) {
            s_U = U;
            s_T = tot;
            s_ts = ts;
            s_before = sbefore;
            s_found = ~0ull;
        }
    }
    __syncthreads();
    const T U = s_U, tot = s_T;
    const int ts = s_ts;
    if (ts >= 0) {
        // block scan inside the 1024-point segment, 4 consecutive points / thread
        const uint64_t base = (uint64_t)ts * kSeg + 4ull * threadIdx.x;
        T m[4];
        T loc = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t i = base + j;
            m[j] = i < a.n ? M::mass(a, i, weights_only ? kWeightsOnly : md_at(a, md, i)) : (T)0;
            loc += m[j];
        }
        T btot;
        const T start = s_before + block_excl<M>(loc, s_w, &btot);
        if (start <= U && start + loc > U) {
            T acc = start;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const T nxt = acc + m[j];
                if (nxt > U) {
                    s_found = base + j;
                    s_prevE = acc;
                    s_E = nxt;
                    break;
                }
                acc = nxt;
            }
        }
    }
    __syncthreads();
    uint64_t idx;
    bool ambiguous = false;
    if (s_found == ~0ull || s_found >= a.n - 1) {
        idx = a.n - 1; // the reference returns n-1 when no i < n-1 qualifies
        if (!M::exact && a.n > 1) {
            const T mlast = M::mass(a, a.n - 1, weights_only ? kWeightsOnly : md_at(a, md, a.n - 1));
            ambiguous = !(U > tot - mlast + M::bound(a.n, tot));
        }
    } else {
        idx = s_found;
        if (!M::exact) {
            const T B2 = M::bound(a.n, tot);
            ambiguous = !(s_E > U + B2) || (idx > 0 && !(U > s_prevE + B2));
        }
    }
    __syncthreads();
    if (ambiguous) { // identical decision in every block -> uniform barrier
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.result[par] = sequential_draw(a, md, nu, weights_only);
            atomicAdd(a.fallbacks, 1ull);
        }
        grid.sync();
        idx = a.result[par];
    }
    return idx;
}

// ---------------------------------------------------------------------------
// Large substrates, record layout: rec[i] = {colour, md} (8 bytes, in place).
// A round reads 8 bytes per point and writes only the points whose min
// distance drops; k-means++ block/segment mass sums change by the exact
// difference of those points' masses (counts are read only for them), so a
// round streams half the bytes of the ping-pong layout. In-place updates need
// a second grid barrier per k-means++ round (nobody updates before every
// block has located the draw); maximin locates through the ping-ponged block
// maxima and keeps one barrier.

constexpr int kRecBatch = 16; // records in flight per lane (32 doubles the registers: 1 block per SM)

#ifdef CQG_INIT_TIMING
__device__ unsigned long long g_coop_timing[8]; // [5] tiles updated, [6] points changed, [7] slowest block's update
__device__ unsigned long long g_tile_round_max;
__device__ unsigned long long g_tile_rounds[1024][2]; // per round: slowest block update, block 0 locate
__device__ unsigned long long g_warp_hist[16][2];    // per warp-round of update_tiles by reached tiles: cycles, count
__device__ int g_warp_hist_on;                       // set by block 0 from round 32 on (steady state)
__device__ unsigned long long g_loc_phase[4];
#define GTIME(slot)                                                                  \
    do {                                                                             \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                   \
            const unsigned long long _n = clock64();                                 \
            g_coop_timing[slot] += _n - _gprev;                                      \
            _gprev = _n;                                                             \
        }                                                                            \
    } while (0)
#else
#define GTIME(slot) \
    do {            \
    } while (0)
#endif

// k-means++ update over this block's segments (full: first round from the
// colours; else incremental). The incremental loop is lean: 8-byte record
// loads, the distance, and a change bitmask; only a warp with a changed point
// loads counts (all at once) and rewrites md. Records past n carry md = 0 and
// never change.
template <class M>
__device__ void update_rec(const InitArgs &a, bool full, uint32_t clast, uint2 *rec, uint64_t lo, uint64_t hi,
                           typename M::T *s_w) {
    typedef typename M::T T;
    T *segs = reinterpret_cast<T *>(a.segs);
    T *parts = reinterpret_cast<T *>(a.parts);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t bb = __dp4a(clast, clast, 0u);
    T bsum = 0;
    for (uint64_t s0 = lo + (uint64_t)warp * kSeg; s0 < hi; s0 += (uint64_t)nw * kSeg) {
        T loc = 0;
        if (full) {
            for (int b = lane; b < kSeg; b += 32) {
                const uint64_t i = s0 + b;
                if (i < hi) {
                    const uint32_t c = __ldg(a.colors + i);
                    const uint32_t d = d2_int_bb(c, clast, bb);
                    rec[i] = make_uint2(c, d);
                    loc += M::mass_c(a, __ldg(a.counts + i), d);
                }
            }
        } else {
            const bool whole = s0 + kSeg <= hi;
            for (int b = 0; b < kSeg; b += 32 * kRecBatch) {
                uint2 r[kRecBatch];
                if (whole) {
#pragma unroll
                    for (int u = 0; u < kRecBatch; ++u) r[u] = rec[s0 + b + u * 32 + lane];
                } else {
#pragma unroll
                    for (int u = 0; u < kRecBatch; ++u) {
                        const uint64_t i = s0 + b + u * 32 + lane;
                        r[u] = i < hi ? rec[i] : make_uint2(0u, 0u);
                    }
                }
                uint32_t chg = 0;
#pragma unroll
                for (int u = 0; u < kRecBatch; ++u)
                    chg |= (d2_int_bb(r[u].x, clast, bb) < r[u].y ? 1u : 0u) << u;
                if (__any_sync(0xffffffffu, chg != 0)) {
                    uint32_t cn[kRecBatch];
#pragma unroll
                    for (int u = 0; u < kRecBatch; ++u)
                        cn[u] = (chg >> u) & 1u ? __ldg(a.counts + s0 + b + u * 32 + lane) : 0u;
#pragma unroll
                    for (int u = 0; u < kRecBatch; ++u) {
                        if ((chg >> u) & 1u) {
                            const uint32_t d = d2_int_bb(r[u].x, clast, bb);
                            loc += M::mass_c(a, cn[u], r[u].y) - M::mass_c(a, cn[u], d); // masses fall with md
                            rec[s0 + b + u * 32 + lane].y = d;
                        }
                    }
                }
            }
        }
        for (int o = 16; o; o >>= 1) loc += M::shfl(loc, lane ^ o);
        if (lane == 0) {
            if (full) segs[s0 / kSeg] = loc;
            else if (loc != (T)0) segs[s0 / kSeg] -= loc;
        }
        bsum += loc;
    }
    if (lane == 0) s_w[warp] = bsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int w = 0; w < nw; ++w) t += s_w[w];
        if (full) parts[blockIdx.x] = t;
        else parts[blockIdx.x] -= t;
    }
    __syncthreads();
}

template <class M>
__global__ void __launch_bounds__(kInitThreads, 3) init_kernel_rec(InitArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ typename M::T s_w[kInitThreads / 32];
    __shared__ unsigned long long s_m[kInitThreads / 32];
    const uint64_t lo = (uint64_t)blockIdx.x * a.chunk;
    const uint64_t hi = lo + a.chunk < a.n ? lo + a.chunk : a.n;
    uint2 *rec = reinterpret_cast<uint2 *>(a.md);
    const uint32_t *mdv = a.md + 1; // md values at stride 2 (a.mds == 2)
    int par = 0;
#ifdef CQG_INIT_TIMING
    unsigned long long _gprev = clock64();
#endif

    uint64_t first;
    if (a.kind == 1 || a.weighted_first) {
        update_masses<M>(a, 0, 1, 0, 0, nullptr, nullptr, lo, hi, s_w);
        grid.sync();
        first = locate_draw<M>(a, grid, 0, a.nu[0], 1, nullptr, s_w);
        grid.sync(); // the block sums are rewritten in place below
    } else {
        first = a.first_index;
    }
    uint32_t clast = __ldg(a.colors + first);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.cen[0] = (double)((clast >> 16) & 255u);
        a.cen[1] = (double)((clast >> 8) & 255u);
        a.cen[2] = (double)(clast & 255u);
    }
    for (int k = 1; k < a.K; ++k) {
        uint64_t pick;
        if (a.kind == 0) {
            const uint32_t bb = __dp4a(clast, clast, 0u);
            // per thread: the largest md and, among equal md, the lowest index
            uint32_t bm = 0, bi = 0xFFFFFFFFu;
            if (k == 1) {
                for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                    const uint32_t c = __ldg(a.colors + i);
                    const uint32_t m = d2_int_bb(c, clast, bb);
                    rec[i] = make_uint2(c, m);
                    if (m > bm || (m == bm && (uint32_t)i < bi)) bm = m, bi = (uint32_t)i;
                }
            } else {
                for (uint64_t i0 = lo + threadIdx.x; i0 < hi; i0 += (uint64_t)kRecBatch * blockDim.x) {
                    uint2 r[kRecBatch];
#pragma unroll
                    for (int u = 0; u < kRecBatch; ++u) {
                        const uint64_t i = i0 + (uint64_t)u * blockDim.x;
                        r[u] = i < hi ? rec[i] : make_uint2(0u, 0u);
                    }
#pragma unroll
                    for (int u = 0; u < kRecBatch; ++u) {
                        const uint32_t d = d2_int_bb(r[u].x, clast, bb);
                        const uint64_t i = i0 + (uint64_t)u * blockDim.x;
                        if (d < r[u].y) { // only reachable for i < hi (padding has md 0)
                            r[u].y = d;
                            rec[i].y = d;
                        }
                        // indices grow with u: strict > keeps the lowest index on ties
                        if (r[u].y > bm || (bi == 0xFFFFFFFFu && i < hi)) bm = r[u].y, bi = (uint32_t)i;
                    }
                }
            }
            unsigned long long best = bi == 0xFFFFFFFFu ? 0ull : (((unsigned long long)bm << 32) | (uint32_t)~bi);
            for (int o = 16; o; o >>= 1) {
                const unsigned long long t = __shfl_xor_sync(0xffffffffu, best, o);
                best = t > best ? t : best;
            }
            if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = best;
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long b = 0;
                for (int i = 0; i < kInitThreads / 32; ++i) b = s_m[i] > b ? s_m[i] : b;
                a.mparts[(size_t)par * gridDim.x + blockIdx.x] = b;
            }
            grid.sync();
            unsigned long long b = 0;
            if (threadIdx.x < 32) {
                for (unsigned i = threadIdx.x; i < gridDim.x; i += 32) {
                    const unsigned long long t = a.mparts[(size_t)par * gridDim.x + i];
                    b = t > b ? t : b;
                }
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
                    b = t > b ? t : b;
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) s_m[0] = b;
            __syncthreads();
            b = s_m[0];
            pick = (uint64_t)(uint32_t)~(uint32_t)(b & 0xFFFFFFFFull);
            par ^= 1;
        } else {
            GTIME(4);
            update_rec<M>(a, k == 1, clast, rec, lo, hi, s_w);
            GTIME(0);
            grid.sync();
            GTIME(1);
            pick = locate_draw<M>(a, grid, 0, a.nu[k], 0, mdv, s_w);
            GTIME(2);
            grid.sync(); // records and sums are updated in place by the next round
            GTIME(3);
        }
        clast = __ldg(a.colors + pick);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.cen[3 * k] = (double)((clast >> 16) & 255u);
            a.cen[3 * k + 1] = (double)((clast >> 8) & 255u);
            a.cen[3 * k + 2] = (double)(clast & 255u);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Large substrates, colour-space tiles. The points are laid out in Morton
// order of their colour (kTile consecutive points per tile, each tile a
// compact colour box), so a round of the update only visits the tiles the new
// centre can reach: a tile whose box is at squared distance >= its largest md
// from the new centre keeps every min distance (md only falls when
// d2(x, c) < md, and d2(x, c) >= d2(box, c) for every x in the box). All in
// exact integers, so the set of updated points -- and every md -- is exactly
// the full sweep's. k-means++ keeps its mass sums in HISTOGRAM order (the
// reference's prefix order): a changed point subtracts its exact mass drop
// from its segment's and its part's sum (atomics); the locate is the record
// kernel's, reading md through hpos. Maximin keeps per-tile maxima of
// (md, ~index); untouched tiles keep theirs.
#ifndef CQG_TILE_POINTS
#define CQG_TILE_POINTS 128 // measured: 64 / 128 / 256 / 512 -> cfg5 init 6.22 / 5.93 / 6.13 / 9.15 ms
#endif
constexpr int kTile = CQG_TILE_POINTS; // points per tile (kTile / 32 per lane of one warp)
constexpr int kFlagStride = 32;  // u64 words between two blocks' release flags (256 B)

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
constexpr int kTileBitmapWords = 1 << 19; // 2^24 Morton slots

__device__ __forceinline__ uint32_t tile_spread8(uint32_t x) {
    x = (x | (x << 8)) & 0x0000F00Fu;
    x = (x | (x << 4)) & 0x000C30C3u;
    x = (x | (x << 2)) & 0x00249249u;
    return x;
}
__device__ __forceinline__ uint32_t tile_morton(uint32_t c) {
    return (tile_spread8((c >> 16) & 255u) << 2) | (tile_spread8((c >> 8) & 255u) << 1) | tile_spread8(c & 255u);
}

// setup 1: one bit per present Morton slot; a second point on a slot
// (duplicate colours: raw-pixel substrates) raises *dup
__global__ void tile_mark_kernel(const uint32_t *__restrict__ colors, uint64_t n, uint32_t *__restrict__ bits,
                                 uint32_t *dup) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = tile_morton(__ldg(colors + i));
        const uint32_t bit = 1u << (m & 31u);
        if (atomicOr(bits + (m >> 5), bit) & bit) *dup = 1u;
    }
}

// setup 2: exclusive popcount prefix of the bitmap words (1024 words per
// block; block offsets from a second, single-block pass over the block sums)
__device__ __forceinline__ uint32_t block_excl_u32(uint32_t v, uint32_t *s_w, uint32_t *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const uint32_t x = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0u;
        uint32_t xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += t;
        }
        s_w[lane] = xi - x;
        if (lane == 31) s_w[32] = xi;
    }
    __syncthreads();
    const uint32_t r = s_w[wid] + incl - v;
    if (total) *total = s_w[32];
    __syncthreads();
    return r;
}
__global__ void __launch_bounds__(1024) tile_scan_blocks(const uint32_t *__restrict__ bits, uint32_t *__restrict__ pref,
                                                         uint32_t *__restrict__ bsum) {
    __shared__ uint32_t s_w[33];
    const uint32_t w = blockIdx.x * 1024u + threadIdx.x;
    uint32_t tot;
    pref[w] = block_excl_u32((uint32_t)__popc(bits[w]), s_w, &tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(1024) tile_scan_top(uint32_t *bsum, int nb) {
    __shared__ uint32_t s_w[33];
    const uint32_t v = (int)threadIdx.x < nb ? bsum[threadIdx.x] : 0u;
    const uint32_t e = block_excl_u32(v, s_w, nullptr);
    if ((int)threadIdx.x < nb) bsum[threadIdx.x] = e;
}

// setup 3: place every point at its Morton rank, one destination array per
// launch (which = 0: colour, 1: histogram index (+ hpos), 2: count), so each
// pass's random 4-byte stores land in an L2-resident 4n-byte array and merge
// into whole sectors before write-back (one pass writing all of them
// thrashed L2 with partial-sector read-modify-writes)
__global__ void tile_place_kernel(const uint32_t *__restrict__ colors, const uint32_t *__restrict__ counts, uint64_t n,
                                  const uint32_t *__restrict__ bits, const uint32_t *__restrict__ pref,
                                  const uint32_t *__restrict__ bsum, uint32_t *__restrict__ dst, int which,
                                  uint32_t *__restrict__ hpos) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = __ldg(colors + i);
        const uint32_t m = tile_morton(c), w = m >> 5;
        const uint32_t pos = bsum[w >> 10] + pref[w] + (uint32_t)__popc(bits[w] & ((1u << (m & 31u)) - 1u));
        dst[pos] = which == 0 ? c : (which == 1 ? (uint32_t)i : __ldg(counts + i));
        if (which == 1 && hpos) hpos[i] = pos;
    }
}

// The tile order is the Morton order of the distinct colours, so the tile-order
// colour array is the bitmap read back (sequential stores, no scatter).
__device__ __forceinline__ uint32_t tile_compact8(uint32_t x) {
    x &= 0x00249249u;
    x = (x | (x >> 2)) & 0x000C30C3u;
    x = (x | (x >> 4)) & 0x0000F00Fu;
    x = (x | (x >> 8)) & 0x000000FFu;
    return x;
}
__global__ void __launch_bounds__(256) tile_expand_kernel(const uint32_t *__restrict__ bits,
                                                          const uint32_t *__restrict__ pref,
                                                          const uint32_t *__restrict__ bsum,
                                                          uint32_t *__restrict__ tcol) {
    // a warp takes 32 words; word by word, lane l writes slot l's colour at
    // the word's prefix + the set bits below it: one coalesced store per word
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t wbase = ((blockIdx.x * 256u + threadIdx.x) >> 5) << 5;
    const uint32_t w = wbase + lane;
    const uint32_t b = bits[w];
    const uint32_t p0 = bsum[w >> 10] + pref[w];
    if (!__any_sync(0xffffffffu, b != 0u)) return;
    const uint32_t below = (1u << lane) - 1u;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
        const uint32_t bj = __shfl_sync(0xffffffffu, b, j);
        const uint32_t pj = __shfl_sync(0xffffffffu, p0, j);
        if ((bj >> lane) & 1u) {
            const uint32_t m = ((wbase + (uint32_t)j) << 5) | lane;
            tcol[pj + (uint32_t)__popc(bj & below)] =
                (tile_compact8(m >> 2) << 16) | (tile_compact8(m >> 1) << 8) | tile_compact8(m);
        }
    }
}
// the tile-order counts: gathered through the placed histogram indices (random
// 4-byte reads cost about half of the scatter pass they replace)
__global__ void tile_count_kernel(const uint32_t *__restrict__ counts, const uint32_t *__restrict__ tidx, uint64_t n,
                                  uint32_t *__restrict__ tcnt) {
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x)
        tcnt[p] = __ldg(counts + tidx[p]);
}

// setup 4: per tile the colour box (one warp per tile)
__global__ void tile_box_kernel(const uint32_t *__restrict__ tcol, uint64_t n, uint64_t ntiles, uint2 *__restrict__ tbox,
                                uint32_t *__restrict__ tmax) {
    const int lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = gw; t < ntiles; t += nw) {
        uint32_t lr = 255, lg = 255, lb = 255, hr = 0, hg = 0, hb = 0;
        for (int u = 0; u < kTile / 32; ++u) {
            const uint64_t p = t * kTile + u * 32 + lane;
            if (p < n) {
                const uint32_t c = tcol[p];
                const uint32_t r = (c >> 16) & 255u, g = (c >> 8) & 255u, b = c & 255u;
                lr = min(lr, r), lg = min(lg, g), lb = min(lb, b);
                hr = max(hr, r), hg = max(hg, g), hb = max(hb, b);
            }
        }
        for (int o = 16; o; o >>= 1) {
            lr = min(lr, __shfl_xor_sync(0xffffffffu, lr, o));
            lg = min(lg, __shfl_xor_sync(0xffffffffu, lg, o));
            lb = min(lb, __shfl_xor_sync(0xffffffffu, lb, o));
            hr = max(hr, __shfl_xor_sync(0xffffffffu, hr, o));
            hg = max(hg, __shfl_xor_sync(0xffffffffu, hg, o));
            hb = max(hb, __shfl_xor_sync(0xffffffffu, hb, o));
        }
        if (lane == 0) {
            tbox[t] = make_uint2((lr << 16) | (lg << 8) | lb, (hr << 16) | (hg << 8) | hb);
            tmax[t] = 0xFFFFFFFFu;
        }
    }
}

// squared distance from colour c to the box {lo, hi} (exact integers)
__device__ __forceinline__ uint32_t box_d2(uint2 box, uint32_t c) {
    uint32_t s = 0;
#pragma unroll
    for (int sh = 16; sh >= 0; sh -= 8) {
        const int v = (int)((c >> sh) & 255u), lo = (int)((box.x >> sh) & 255u), hi = (int)((box.y >> sh) & 255u);
        const int d = v < lo ? lo - v : (v > hi ? v - hi : 0);
        s += (uint32_t)(d * d);
    }
    return s;
}

__device__ __forceinline__ void atomic_sub_mass(unsigned long long *p, unsigned long long v) {
    atomicAdd(p, 0ull - v);
}
__device__ __forceinline__ void atomic_sub_mass(u128 *p, u128 v) {
    // two's complement add of -v, low word first with its carry (the value is
    // consistent again once every update of the round has landed)
    const u128 nv = (u128)0 - v;
    unsigned long long *q = reinterpret_cast<unsigned long long *>(p);
    const unsigned long long lo = (unsigned long long)nv, hi = (unsigned long long)(nv >> 64);
    const unsigned long long old = atomicAdd(q, lo);
    const unsigned long long carry = old + lo < old ? 1ull : 0ull;
    if (hi + carry) atomicAdd(q + 1, hi + carry);
}

// One round of the tile update for the new centre clast. full: first round
// (every tile, md := d2). Each warp owns tiles gw, gw + W, ...; its lanes test
// 32 of them at once, then the warp updates the reached ones (8 points per
// lane). k-means++: changed points subtract their exact mass drop from their
// histogram segment and part sums. Maximin: returns the warp's largest
// (md, ~index) over all its tiles.
template <class M, bool PAIR>
__device__ unsigned long long update_tiles(const InitArgs &a, bool full, uint32_t clast) {
    typedef typename M::T T;
    T *segs = reinterpret_cast<T *>(a.segs);
    const int lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t bb = __dp4a(clast, clast, 0u);
    unsigned long long best = 0;
#ifdef CQG_INIT_TIMING
    const unsigned long long _w0 = clock64();
    int _wn = 0;
#endif
    for (uint64_t j0 = 0; gw + j0 * W < a.ntiles; j0 += 32) {
        const uint64_t t = gw + (j0 + lane) * W;
        // branch-free metadata loads (clamped tile index, masked result)
        const bool tin = t < a.ntiles;
        const uint64_t tc = tin ? t : 0;
        const uint2 bx = a.tbox[tc];
        const uint32_t tm = a.tmax[tc];
        const unsigned long long tk = a.kind == 0 ? a.tkey[tc] : 0ull;
        const bool need = tin && (full || box_d2(bx, clast) < tm);
        if (tin && !need) best = max(best, tk);
        unsigned m = __ballot_sync(0xffffffffu, need);
#ifdef CQG_INIT_TIMING
        _wn += __popc(m);
#endif
        // the reached tiles of this warp; k-means++ (PAIR) takes them two at a time, both tiles' loads in
        // flight before either is updated: a tile costs a DRAM round trip and a round waits for the warp
        // with the most tiles (cfg5 init stage 5.23 -> 5.06 ms). Maximin tiles are cheap and its kernel
        // keeps the smaller register budget (pairing them measured slower: cfg3 1.59 -> 1.73 ms).
        constexpr int TP = kTile / 32;
        auto load_tile = [&](uint64_t tt, uint2 *r, uint32_t *cn, uint32_t *hx) {
            // every load of the tile issued at once (clamped indices: the
            // last tile's padding lanes re-read point n-1 and are masked)
#pragma unroll
            for (int u = 0; u < TP; ++u) {
                const uint64_t p = tt * kTile + u * 32 + lane;
                const uint64_t pc = p < a.n ? p : a.n - 1;
                r[u] = make_uint2(__ldg(a.tcol + pc), a.tmd[pc]);
                cn[u] = (a.kind == 1 && !full) ? __ldg(a.tcnt + pc) : 0u;
                hx[u] = (a.kind == 0 || !full) ? __ldg(a.tidx + pc) : 0u;
            }
        };
        auto update_tile = [&](uint64_t tt, uint2 *r, const uint32_t *cn, const uint32_t *hx) {
            uint32_t mx = 0;
            unsigned long long kb = 0;
            uint32_t dn[TP], chg = 0;
#pragma unroll
            for (int u = 0; u < TP; ++u) {
                const uint64_t p = tt * kTile + u * 32 + lane;
                dn[u] = d2_int_bb(r[u].x, clast, bb);
                if (p < a.n && dn[u] < r[u].y) chg |= 1u << u; // first round: md = 0xFFFFFFFF
            }
#pragma unroll
            for (int u = 0; u < TP; ++u) {
                const uint64_t p = tt * kTile + u * 32 + lane;
                if ((chg >> u) & 1u) {
                    a.tmd[p] = dn[u];
                    if (a.kind == 1 && !full) {
                        const T dm = M::mass_c(a, cn[u], r[u].y) - M::mass_c(a, cn[u], dn[u]);
                        if (dm != (T)0) atomic_sub_mass(segs + hx[u] / kSeg, dm);
                    }
                    r[u].y = dn[u];
                }
                if (p < a.n) {
                    mx = max(mx, r[u].y);
                    if (a.kind == 0) kb = max(kb, ((unsigned long long)r[u].y << 32) | (uint32_t)~hx[u]);
                }
            }
            for (int o = 16; o; o >>= 1) {
                mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                kb = max(kb, __shfl_xor_sync(0xffffffffu, kb, o));
            }
            if (lane == 0) {
                a.tmax[tt] = mx;
                if (a.kind == 0) a.tkey[tt] = kb;
            }
#ifdef CQG_INIT_TIMING
            {
                unsigned nc = __popc(chg);
                for (int o = 16; o; o >>= 1) nc += __shfl_xor_sync(0xffffffffu, nc, o);
                if (lane == 0) {
                    atomicAdd(&g_coop_timing[5], 1ull);
                    atomicAdd(&g_coop_timing[6], (unsigned long long)nc);
                }
            }
#endif
            best = max(best, kb);
        };
        while (m) {
            const int l0 = __ffs(m) - 1;
            m &= m - 1;
            if constexpr (!PAIR) {
                const uint64_t tt = gw + (j0 + l0) * W;
                // every load of the tile issued at once (clamped indices: the
                // last tile's padding lanes re-read point n-1 and are masked)
                uint2 r[kTile / 32];
                uint32_t cn[kTile / 32], hx[kTile / 32];
    #pragma unroll
                for (int u = 0; u < kTile / 32; ++u) {
                    const uint64_t p = tt * kTile + u * 32 + lane;
                    const uint64_t pc = p < a.n ? p : a.n - 1;
                    r[u] = make_uint2(__ldg(a.tcol + pc), a.tmd[pc]);
                    cn[u] = (a.kind == 1 && !full) ? __ldg(a.tcnt + pc) : 0u;
                    hx[u] = (a.kind == 0 || !full) ? __ldg(a.tidx + pc) : 0u;
                }
                uint32_t mx = 0;
                unsigned long long kb = 0;
                uint32_t dn[kTile / 32], chg = 0;
    #pragma unroll
                for (int u = 0; u < kTile / 32; ++u) {
                    const uint64_t p = tt * kTile + u * 32 + lane;
                    dn[u] = d2_int_bb(r[u].x, clast, bb);
                    if (p < a.n && dn[u] < r[u].y) chg |= 1u << u; // first round: md = 0xFFFFFFFF
                }
    #pragma unroll
                for (int u = 0; u < kTile / 32; ++u) {
                    const uint64_t p = tt * kTile + u * 32 + lane;
                    if ((chg >> u) & 1u) {
                        a.tmd[p] = dn[u];
                        if (a.kind == 1 && !full) {
                            const T dm = M::mass_c(a, cn[u], r[u].y) - M::mass_c(a, cn[u], dn[u]);
                            if (dm != (T)0) atomic_sub_mass(segs + hx[u] / kSeg, dm);
                        }
                        r[u].y = dn[u];
                    }
                    if (p < a.n) {
                        mx = max(mx, r[u].y);
                        if (a.kind == 0) kb = max(kb, ((unsigned long long)r[u].y << 32) | (uint32_t)~hx[u]);
                    }
                }
                for (int o = 16; o; o >>= 1) {
                    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    kb = max(kb, __shfl_xor_sync(0xffffffffu, kb, o));
                }
                if (lane == 0) {
                    a.tmax[tt] = mx;
                    if (a.kind == 0) a.tkey[tt] = kb;
                }
    #ifdef CQG_INIT_TIMING
                {
                    unsigned nc = __popc(chg);
                    for (int o = 16; o; o >>= 1) nc += __shfl_xor_sync(0xffffffffu, nc, o);
                    if (lane == 0) {
                        atomicAdd(&g_coop_timing[5], 1ull);
                        atomicAdd(&g_coop_timing[6], (unsigned long long)nc);
                    }
                }
    #endif
                best = max(best, kb);
            } else {
                const bool two = m != 0;
                const int l1 = two ? __ffs(m) - 1 : l0;
                if (two) m &= m - 1;
                const uint64_t t0 = gw + (j0 + l0) * W, t1 = gw + (j0 + l1) * W;
                uint2 r0[TP], r1[TP];
                uint32_t cn0[TP], hx0[TP], cn1[TP], hx1[TP];
                load_tile(t0, r0, cn0, hx0);
                if (two) load_tile(t1, r1, cn1, hx1);
                update_tile(t0, r0, cn0, hx0);
                if (two) update_tile(t1, r1, cn1, hx1);
            }
        }
    }
#ifdef CQG_INIT_TIMING
    if (!full && lane == 0 && *(volatile int *)&g_warp_hist_on) {
        const int b_ = _wn < 15 ? _wn : 15;
        atomicAdd(&g_warp_hist[b_][0], clock64() - _w0);
        atomicAdd(&g_warp_hist[b_][1], 1ull);
    }
#endif
    for (int o = 16; o; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    return best;
}

// first k-means++ round: the segment mass sums in histogram order (one warp
// per kSeg segment), md = d2(x, c0) (the tiles hold the same values)
template <class M>
__device__ void tile_first_sums(const InitArgs &a, uint32_t clast) {
    typedef typename M::T T;
    T *segs = reinterpret_cast<T *>(a.segs);
    const int lane = threadIdx.x & 31;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t bb = __dp4a(clast, clast, 0u);
    const uint64_t nseg = (a.n + kSeg - 1) / kSeg;
    for (uint64_t sg = gw; sg < nseg; sg += W) {
        T loc = 0;
#pragma unroll 4
        for (int b = lane; b < kSeg; b += 32) {
            const uint64_t i = sg * kSeg + b;
            if (i < a.n) loc += M::mass_c(a, __ldg(a.counts + i), d2_int_bb(__ldg(a.colors + i), clast, bb));
        }
        for (int o = 16; o; o >>= 1) loc += M::shfl(loc, lane ^ o);
        if (lane == 0) segs[sg] = loc;
    }
}

// The draw of one k-means++ round, located by ONE block over the segment sums
// (no per-block part sums: those would be the atomics' hot spot): thread
// sums over runs of segments, a block scan, the owner's run, then the
// segment's points (md through hpos) exactly as locate_draw does, including
// its n-1 rule and the fixed-point ambiguity fallback.
template <class M>
__device__ uint64_t locate_one_block(const InitArgs &a, double nu, const uint32_t *md, typename M::T *s_w) {
    typedef typename M::T T;
    __shared__ T s_U, s_T, s_before, s_prevE, s_E;
    __shared__ long long s_ts;
    __shared__ unsigned long long s_found;
    const T *segs = reinterpret_cast<const T *>(a.segs);
    const uint64_t nseg = (a.n + kSeg - 1) / kSeg;
    // The segment sums are read in coalesced waves: wave j covers segments
    // [j*256*V, (j+1)*256*V), thread t the V = 16/sizeof(T) segments at
    // j*256*V + t*V (one 16-byte load). Level 1: per-wave sums (a transposed
    // warp reduction of up to 32 waves per pass, then across warps); level 2:
    // the target wave reloaded and scanned by the block.
    constexpr int V = 16 / (int)sizeof(T);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint64_t per_wave = (uint64_t)kInitThreads * V;
    const int W = (int)((nseg + per_wave - 1) / per_wave); // <= 64 (n <= 2^24)
    __shared__ T s_C[64];
    __shared__ T s_wc[kInitThreads / 32][32];
#ifdef CQG_INIT_TIMING
    unsigned long long _q = clock64();
#define LTIME(i) do { if (threadIdx.x == 0) { const unsigned long long _n = clock64(); g_loc_phase[i] += _n - _q; _q = _n; } } while (0)
#else
#define LTIME(i) do { } while (0)
#endif
    // this thread's V segment sums of wave j (0 past the end): e0, e1 (V == 2)
#define WAVE_ELEM(j, e0, e1)                                                                     \
    do { /* branch-free: clamped address, masked value (loads stay in flight together) */       \
        const uint64_t s_ = (uint64_t)(j) * per_wave + (uint64_t)t * V;                          \
        const bool in0_ = s_ < nseg, in1_ = s_ + 1 < nseg;                                       \
        const uint64_t sc_ = in0_ ? s_ : 0;                                                      \
        if (V == 2) {                                                                            \
            const uint4 q_ = __ldcg(reinterpret_cast<const uint4 *>(segs + sc_));                \
            e0 = in0_ ? (T)(((unsigned long long)q_.y << 32) | q_.x) : (T)0;                     \
            e1 = in1_ ? (T)(((unsigned long long)q_.w << 32) | q_.z) : (T)0;                     \
        } else {                                                                                 \
            const T q_ = segs[sc_];                                                              \
            e0 = in0_ ? q_ : (T)0;                                                               \
            e1 = 0;                                                                              \
        }                                                                                        \
    } while (0)
    for (int g = 0; g < W; g += 32) {
        T v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
            T e0, e1;
            WAVE_ELEM(g + u, e0, e1); // waves past W read as 0 (s_ >= nseg)
            v[u] = e0 + e1;
        }
        // transposed reduction: lane l ends with the warp's sum of v[l]
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int i = 0; i < off; ++i) {
                const T send = up ? v[i] : v[i + off];
                const T keep = up ? v[i + off] : v[i];
                v[i] = keep + M::shfl(send, lane ^ off);
            }
        }
        s_wc[warp][lane] = v[0];
        __syncthreads();
        if (t < 32) {
            T c = 0;
#pragma unroll
            for (int w = 0; w < kInitThreads / 32; ++w) c += s_wc[w][t];
            if (g + t < 64) s_C[g + t] = c;
        }
        __syncthreads();
    }
    LTIME(0);
    // total, target and the wave holding it (warp 0: up to 64 wave sums)
    __shared__ int s_wv;
    __shared__ T s_wbefore;
    if (warp == 0) {
        const T c0 = lane < W ? s_C[lane] : (T)0, c1 = lane + 32 < W ? s_C[lane + 32] : (T)0;
        const T i0 = warp_incl<M>(c0);
        const T tot0 = M::shfl(i0, 31);
        const T i1 = warp_incl<M>(c1) + tot0;
        const T tot = M::shfl(i1, 31);
        const T U = M::target(nu, tot);
        const unsigned m0 = __ballot_sync(0xffffffffu, i0 > U), m1 = __ballot_sync(0xffffffffu, i1 > U);
        int wv = -1;
        T before = 0;
        if (m0) {
            const int l = __ffs(m0) - 1;
            wv = l;
            before = M::shfl(i0 - c0, l);
        } else if (m1) {
            const int l = __ffs(m1) - 1;
            wv = 32 + l;
            before = M::shfl(i1 - c1, l);
        }
        if (lane == 0) {
            s_U = U;
            s_T = tot;
            s_wv = wv;
            s_wbefore = before;
            s_ts = -1;
            s_found = ~0ull;
        }
    }
    __syncthreads();
    const T U = s_U, tot = s_T;
    if (s_wv >= 0) { // the wave: a block scan over the threads' V-segment groups
        T e0, e1;
        WAVE_ELEM(s_wv, e0, e1);
        const T l = e0 + e1;
        T btot;
        const T start = s_wbefore + block_excl<M>(l, s_w, &btot);
        if (start <= U && start + l > U) {
            const uint64_t s0 = (uint64_t)s_wv * per_wave + (uint64_t)t * V;
            if (V == 1 || start + e0 > U) {
                s_ts = (long long)s0;
                s_before = start;
            } else {
                s_ts = (long long)(s0 + 1);
                s_before = start + e0;
            }
        }
    }
    __syncthreads();
    LTIME(1);
    const long long ts = s_ts;
    if (ts >= 0) {
        const uint64_t base = (uint64_t)ts * kSeg + 4ull * threadIdx.x;
        // branch-free gathers (clamped indices, masked masses): all in flight
        T m[4];
        T l4 = 0;
        uint32_t hp[4], cn[4], mv[4];
        bool ok[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t i = base + j;
            ok[j] = 4 * threadIdx.x + j < (unsigned)kSeg && i < a.n;
            const uint64_t ic = ok[j] ? i : 0;
            hp[j] = a.hpos ? __ldg(a.hpos + ic) : (uint32_t)ic;
            cn[j] = __ldg(a.counts + ic);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) mv[j] = md[(uint64_t)hp[j] * (uint64_t)a.mds];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            m[j] = ok[j] ? M::mass_c(a, cn[j], mv[j]) : (T)0;
            l4 += m[j];
        }
        T btot;
        const T start = s_before + block_excl<M>(l4, s_w, &btot);
        if (start <= U && start + l4 > U) {
            T acc = start;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const T nxt = acc + m[j];
                if (nxt > U) {
                    s_found = base + j;
                    s_prevE = acc;
                    s_E = nxt;
                    break;
                }
                acc = nxt;
            }
        }
    }
    __syncthreads();
    LTIME(2);
    uint64_t idx;
    bool ambiguous = false;
    if (s_found == ~0ull || s_found >= a.n - 1) {
        idx = a.n - 1; // the reference returns n-1 when no i < n-1 qualifies
        if (!M::exact && a.n > 1) {
            const T mlast = M::mass(a, a.n - 1, md_at(a, md, a.n - 1));
            ambiguous = !(U > tot - mlast + M::bound(a.n, tot));
        }
    } else {
        idx = s_found;
        if (!M::exact) {
            const T B2 = M::bound(a.n, tot);
            ambiguous = !(s_E > U + B2) || (idx > 0 && !(U > s_prevE + B2));
        }
    }
    if (ambiguous) { // uniform in the block
        __shared__ unsigned long long s_seq;
        if (threadIdx.x == 0) {
            s_seq = sequential_draw(a, md, nu, 0);
            atomicAdd(a.fallbacks, 1ull);
        }
        __syncthreads();
        idx = s_seq;
    }
    __syncthreads();
    return idx;
}

template <class M, int KIND>
__global__ void __launch_bounds__(kInitThreads, KIND == 1 ? 2 : 3) init_kernel_tile(InitArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ typename M::T s_w[kInitThreads / 32];
    __shared__ unsigned long long s_m[kInitThreads / 32];
    const uint32_t *mdv = a.tmd; // md via hpos
#ifdef CQG_INIT_TIMING
    unsigned long long _gprev = clock64();
#endif
    uint64_t first;
    if (a.kind == 1 || a.weighted_first) {
        const uint64_t lo = (uint64_t)blockIdx.x * a.chunk;
        const uint64_t hi = lo + a.chunk < a.n ? lo + a.chunk : a.n;
        update_masses<M>(a, 0, 1, 0, 0, nullptr, nullptr, lo, hi, s_w);
        grid.sync();
        first = locate_draw<M>(a, grid, 0, a.nu[0], 1, nullptr, s_w);
        grid.sync(); // the sums are rewritten below
    } else {
        first = a.first_index;
    }
    uint32_t clast = __ldg(a.colors + first);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.cen[0] = (double)((clast >> 16) & 255u);
        a.cen[1] = (double)((clast >> 8) & 255u);
        a.cen[2] = (double)(clast & 255u);
    }
    if (KIND == 0 && a.kind == 0) { // (the KIND 0 kernel keeps both loops: compiled alone, the maximin loop ran 3% slower)
        // Maximin has no draw to locate: one grid barrier per round, and every block reduces the
        // block maxima itself (ping-ponged by round parity, read past L1), instead of the arrival
        // counter -> block 0 -> release flags hand-off the k-means++ rounds need (cfg3 init stage
        // 1.95 -> 1.59 ms).
        __shared__ unsigned long long s_pickm;
        const unsigned G32 = gridDim.x;
        for (int k = 1; k < a.K; ++k) {
#ifdef CQG_INIT_TIMING
            if (blockIdx.x == 0 && threadIdx.x == 0) g_warp_hist_on = k >= 32;
#endif
            const unsigned long long wb = update_tiles<M, false>(a, k == 1, clast);
            if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = wb;
            __syncthreads();
            unsigned long long *mp = a.mparts + (size_t)(k & 1) * G32;
            if (threadIdx.x == 0) {
                unsigned long long bm = 0;
                for (int i = 0; i < kInitThreads / 32; ++i) bm = s_m[i] > bm ? s_m[i] : bm;
                mp[blockIdx.x] = bm;
            }
            grid.sync();
            if (threadIdx.x < 32) {
                unsigned long long bm = 0;
                for (unsigned i = threadIdx.x; i < G32; i += 32) {
                    const unsigned long long t = __ldcg(mp + i);
                    bm = t > bm ? t : bm;
                }
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long t = __shfl_xor_sync(0xffffffffu, bm, o);
                    bm = t > bm ? t : bm;
                }
                if (threadIdx.x == 0) s_pickm = (unsigned long long)(uint32_t)~(uint32_t)(bm & 0xFFFFFFFFull);
            }
            __syncthreads();
            const uint64_t pick = s_pickm;
            clast = __ldg(a.colors + pick);
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.cen[3 * k] = (double)((clast >> 16) & 255u);
                a.cen[3 * k + 1] = (double)((clast >> 8) & 255u);
                a.cen[3 * k + 2] = (double)(clast & 255u);
            }
        }
        return;
    }
    // k-means++ rounds: every block updates its tiles and arrives on a counter;
    // block 0 alone waits for all arrivals, locates the draw and publishes it;
    // the others poll the published round number with back-off (a spinning grid
    // barrier would load the memory system under block 0's locate).
    __shared__ unsigned long long s_rel;
    unsigned long long *arrive = a.result + 6;
    unsigned long long *flag = a.tflags + (size_t)blockIdx.x * kFlagStride; // this block's release word
    const unsigned long long G = gridDim.x;
    for (int k = 1; k < a.K; ++k) {
        GTIME(4);
        if (k == 1) tile_first_sums<M>(a, clast);
#ifdef CQG_INIT_TIMING
        if (blockIdx.x == 0 && threadIdx.x == 0) g_warp_hist_on = k >= 32;
#endif
#ifdef CQG_INIT_TIMING
        const unsigned long long _u0 = clock64();
#endif
        update_tiles<M, KIND == 1>(a, k == 1, clast);
        __syncthreads();
#ifdef CQG_INIT_TIMING
        if (threadIdx.x == 0) atomicMax(&g_tile_round_max, clock64() - _u0);
#endif
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(arrive, 1ull);
        }
        GTIME(0);
        if (blockIdx.x == 0) {
            if (threadIdx.x == 0)
                while (ld_acquire_u64(arrive) < G * (unsigned long long)k) __nanosleep(32);
            __syncthreads();
            GTIME(1);
#ifdef CQG_INIT_TIMING
            if (threadIdx.x == 0) {
                g_coop_timing[7] += g_tile_round_max;
                if (k < 1024) g_tile_rounds[k][0] += g_tile_round_max;
                g_tile_round_max = 0;
            }
            const unsigned long long _l0 = clock64();
#endif
            const uint64_t v = locate_one_block<M>(a, a.nu[k], mdv, s_w);
#ifdef CQG_INIT_TIMING
            if (threadIdx.x == 0 && k < 1024) g_tile_rounds[k][1] += clock64() - _l0;
#endif
            // The release word carries the picked colour (round << 32 | colour): a released block
            // needs nothing else, so it reads neither the pick nor the colour array. Every block has
            // its own word (no single hot L2 line); the words are relaxed stores (the data travels
            // in the word itself; the md / segment updates of the round were ordered by the arrivals).
            if (threadIdx.x == 0) s_rel = ((unsigned long long)k << 32) | __ldg(a.colors + v);
            __syncthreads();
            const unsigned long long rel = s_rel;
            for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
                st_relaxed_u64(a.tflags + (size_t)b * kFlagStride, rel);
            GTIME(2);
        } else {
            if (threadIdx.x == 0) {
                unsigned long long w;
                while (((w = ld_acquire_u64(flag)) >> 32) < (unsigned long long)k) __nanosleep(64);
                s_rel = w;
            }
            __syncthreads();
            GTIME(3);
        }
        clast = (uint32_t)s_rel;
        __syncthreads(); // every thread has the colour before thread 0 rewrites s_rel next round
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.cen[3 * k] = (double)((clast >> 16) & 255u);
            a.cen[3 * k + 1] = (double)((clast >> 8) & 255u);
            a.cen[3 * k + 2] = (double)(clast & 255u);
        }
    }
}

// ---------------------------------------------------------------------------
// Small substrates: one thread-block CLUSTER (16 CTAs x 1024 threads, one CTA
// per SM) holds every point in shared memory -- colour, count and ping-pong
// min-distances -- and runs all K rounds with one cluster barrier per round.
// Thread t of CTA c owns the contiguous points [c*chunk + t*ppt, +ppt), so
// thread sums -> warp sums -> CTA sums are in histogram order; every CTA
// locates each draw redundantly by reading the other CTAs' sums through DSMEM
// (CTA sums, then the target CTA's 32 warp sums, its 32 thread sums, and the
// target thread's <= 32 point masses). The arithmetic and the exactness
// argument are the cooperative kernel's (ExactMass / FixedMass).
#ifndef CQG_EXP_SKIP_UPDATE
#define CQG_EXP_SKIP_UPDATE 0
#endif
#ifndef CQG_CLUSTER_THREADS
#define CQG_CLUSTER_THREADS 1024
#endif
constexpr int kClusterThreads = CQG_CLUSTER_THREADS;
constexpr int kMaxClusterCtas = 16;

// ---- DSMEM producer/consumer signalling (mbarrier transaction counts) ----
// A consumer CTA arrives once on its local mbarrier and expects N bytes; each
// producer writes into the consumer's shared memory with st.async, which
// completes those bytes on the consumer's mbarrier. The consumer waits on the
// barrier's phase parity: no cluster-wide barrier is needed.
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_complete_local(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.complete_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
// wait for the barrier phase with the given parity. A signal that never comes
// (a protocol bug) traps after 30 s of wall-clock time (%globaltimer, checked
// every 4096 polls), so preemption or time slicing (MPS, a debugger) cannot
// trip it while a slow but valid signal is on its way; the GPU never hangs.
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint64_t t0 = 0;
    for (uint32_t spin = 0;; ++spin) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok)
                     : "r"(a), "r"(parity)
                     : "memory");
        if (ok) return;
        if ((spin & 4095u) == 4095u) {
            const uint64_t t = global_ns();
            if (t0 == 0) t0 = t;
            else if (t - t0 > 30000000000ull) __trap(); // lost signal: abort the kernel, never hang the GPU
        }
    }
}
__device__ __forceinline__ void st_async_u64(uint32_t raddr, unsigned long long v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr), "l"(v),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint32_t x, uint32_t y, uint32_t z, uint32_t w,
                                            uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(x), "r"(y), "r"(z), "r"(w), "r"(rbar)
                 : "memory");
}
// a mass sum (u64, or u128 as two 64-bit halves)
__device__ __forceinline__ void st_async_T(uint32_t raddr, unsigned long long v, uint32_t rbar) { st_async_u64(raddr, v, rbar); }
__device__ __forceinline__ void st_async_T(uint32_t raddr, u128 v, uint32_t rbar) {
    st_async_v4(raddr, (uint32_t)v, (uint32_t)(v >> 32), (uint32_t)(v >> 64), (uint32_t)(v >> 96), rbar);
}

// Phase timing of the cluster initialiser (tools/init_timing.py builds with
// -DCQG_INIT_TIMING): clock64 deltas of CTA 0 / thread 0, summed over rounds.
#ifdef CQG_INIT_TIMING
__device__ unsigned long long g_init_timing[8];
#define ITIME(slot)                                                                  \
    do {                                                                             \
        if (crank == 0 && t == 0) {                                                  \
            const unsigned long long _n = clock64();                                 \
            g_init_timing[slot] += _n - _tprev;                                      \
            _tprev = _n;                                                             \
        }                                                                            \
    } while (0)
#else
#define ITIME(slot) \
    do {            \
    } while (0)
#endif

template <class M>
__device__ uint64_t cluster_sequential_draw(const InitArgs &a, cg::cluster_group &cl, const uint32_t *s_cnt,
                                            const uint32_t *s_md, uint64_t chunk, double nu, int weights_only) {
    double total = 0.0;
    for (uint64_t i = 0; i < a.n; ++i) {
        const uint32_t r = (uint32_t)(i / chunk), li = (uint32_t)(i % chunk);
        const uint32_t cnt = *cl.map_shared_rank(s_cnt + li, r);
        const uint32_t md = weights_only ? kWeightsOnly : *cl.map_shared_rank(s_md + li, r);
        total = __dadd_rn(total, mass_c(cnt, a.inv, md));
    }
    const double u = __dmul_rn(nu, total);
    double acc = 0.0;
    for (uint64_t i = 0; i + 1 < a.n; ++i) {
        const uint32_t r = (uint32_t)(i / chunk), li = (uint32_t)(i % chunk);
        const uint32_t cnt = *cl.map_shared_rank(s_cnt + li, r);
        const uint32_t md = weights_only ? kWeightsOnly : *cl.map_shared_rank(s_md + li, r);
        acc = __dadd_rn(acc, mass_c(cnt, a.inv, md));
        if (u < acc) return i;
    }
    return a.n - 1;
}


// Register-resident variant (the default): thread t keeps its PPT colours and
// min distances in registers, so a round's update reads no shared memory
// (counts are loaded only for points whose distance falls). Every thread
// knows its exclusive mass prefix inside its warp (the publish scan) and its
// warp's prefix inside the CTA, so once the CTA sums arrive each thread tests
// on its own whether it owns the target; the owner scans its PPT register
// masses and pushes (index, colour, ambiguity) to every CTA. No block barrier
// or warp hand-over sits between the sums' arrival and the pick. The rare
// paths (ambiguous fixed-point decisions, a target beyond every prefix) dump
// the registers into s_md and replay the reference sequentially as before.
template <class M, int PPT, int NT>
__global__ void __launch_bounds__(NT, 1) init_cluster_reg_kernel(InitArgs a) {
    typedef typename M::T T;
    cg::cluster_group cl = cg::this_cluster();
    const int C = (int)cl.num_blocks(), crank = (int)cl.block_rank();
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr uint64_t chunk = (uint64_t)NT * PPT;
    const uint64_t lo = (uint64_t)crank * chunk;
    const uint64_t hi = lo + chunk < a.n ? lo + chunk : a.n;
    const int mine = hi > lo ? (int)(hi - lo) : 0;
    extern __shared__ __align__(16) unsigned char sm_raw[];
    uint32_t *s_col = reinterpret_cast<uint32_t *>(sm_raw);
    uint32_t *s_cnt = s_col + chunk;
    uint32_t *s_md = s_cnt + chunk; // written only on the rare sequential paths
    __shared__ T s_wsum[2][32];
    __shared__ T s_allc[2][kMaxClusterCtas];
    __shared__ uint64_t s_bar[4];
    __shared__ __align__(16) uint32_t s_pk4[2][4];                 // pick lo, pick hi, colour, ambiguous
    __shared__ __align__(16) uint32_t s_mk[2][kMaxClusterCtas][4]; // maximin: every CTA's best key + colour
    __shared__ unsigned long long s_wkey[32];
    __shared__ uint32_t s_wcol[32];
    __shared__ unsigned long long s_pick, s_fbv;
    __shared__ uint32_t s_fbc;
    __shared__ T s_U, s_total, s_base;
    __shared__ int s_tw, s_nf;
    for (int i = t; i < (int)chunk; i += NT) { // padding: colour 0, count 0 (mass 0)
        s_col[i] = i < mine ? __ldg(a.colors + lo + i) : 0u;
        s_cnt[i] = i < mine ? __ldg(a.counts + lo + i) : 0u;
    }
    if (t == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&s_bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int p0 = t * PPT;
    uint32_t rc[PPT], rm[PPT];
#pragma unroll
    for (int j = 0; j < PPT; j += 4) {
        const uint4 c4 = *reinterpret_cast<const uint4 *>(s_col + p0 + j);
        rc[j] = c4.x, rc[j + 1] = c4.y, rc[j + 2] = c4.z, rc[j + 3] = c4.w;
        rm[j] = rm[j + 1] = rm[j + 2] = rm[j + 3] = 0u;
    }
    cl.sync(); // every CTA's barriers exist (and its points are loaded) before the first remote access
    uint32_t ph_s = 0, ph_p = 0; // bit par: parity of the next phase to wait for (uniform per CTA)

    auto colour_of = [&](uint64_t gi) -> uint32_t {
        return *cl.map_shared_rank(s_col + (gi % chunk), (unsigned)(gi / chunk));
    };

    // Publish this round's thread sum ts: returns the thread's exclusive prefix
    // inside its warp; warp 0 scans the warp sums (kept in registers for the
    // draw) and pushes the CTA sum into every rank.
    T w_excl = 0, w_sum = 0; // warp 0, lane l: warp l's exclusive prefix in the CTA and its sum
    auto publish = [&](int par, T ts) -> T {
        if (t == 0) { // this round's incoming bytes: C CTA sums, one 16-byte pick
            mbar_arrive_expect(&s_bar[par], (uint32_t)(C * sizeof(T)));
            mbar_arrive_expect(&s_bar[2 + par], 16u);
        }
        const T tincl = warp_incl<M>(ts);
        if (lane == 31) s_wsum[par][warp] = tincl;
        __syncthreads();
        if (warp == 0) {
            w_sum = lane < NT / 32 ? s_wsum[par][lane] : (T)0; // fewer warps than lanes: zero
            const T wincl = warp_incl<M>(w_sum);
            w_excl = wincl - w_sum;
            const T csum = M::shfl(wincl, 31);
            if (lane < C)
                st_async_T(mapa_rank(smem_addr(&s_allc[par][crank]), lane), csum,
                           mapa_rank(smem_addr(&s_bar[par]), lane));
        }
        return tincl - ts;
    };

    // One weighted draw over this round's masses (weights only: counts).
    // Warp 0 waits for the CTA sums, finds the target U and the warp whose
    // range holds it; after one block barrier only that warp's lanes test
    // their own ranges, and the owner scans its registers.
    auto draw = [&](int par, double nu, bool wo, T ts, T tpre, uint32_t &pick_col) -> uint64_t {
        if (warp == 0) {
            mbar_wait(&s_bar[par], (ph_s >> par) & 1u);
            const T cv = lane < C ? s_allc[par][lane] : (T)0;
            const T cincl = warp_incl<M>(cv);
            const T total = M::shfl(cincl, 31);
            const T U = M::target(nu, total);
            const T cpre = M::shfl(cincl - cv, crank);
            const T wlo = cpre + w_excl;
            const unsigned m = __ballot_sync(0xffffffffu, w_sum != (T)0 && !(U < wlo) && U < wlo + w_sum);
            const int tw = m ? __ffs(m) - 1 : -1;
            const T base = M::shfl(wlo, tw < 0 ? 0 : tw);
            if (lane == 0) {
                s_U = U;
                s_total = total;
                s_base = base;
                s_tw = tw;
                s_nf = (U < total && a.force_seq != 2) ? 0 : 1; // no owner anywhere: identical in every CTA
            }
        }
        ph_s ^= 1u << par;
        __syncthreads();
        const bool nf = s_nf != 0;
        const T U = s_U;
        if (warp == s_tw && !nf) {
            const T lo_t = s_base + tpre;
            if (ts != (T)0 && !(U < lo_t) && U < lo_t + ts) { // the owner (exactly one thread in the cluster)
                const T total = s_total;
                T run = lo_t, E = 0, prevE = 0;
                int pl = PPT;
                uint32_t pcol = 0;
#pragma unroll
                for (int j = 0; j < PPT; ++j) {
                    const T m = M::mass_c(a, s_cnt[p0 + j], wo ? kWeightsOnly : rm[j]);
                    if (pl == PPT && U < run + m) {
                        pl = j;
                        prevE = run;
                        E = run + m;
                        pcol = rc[j];
                    }
                    run += m;
                }
                const uint64_t gi = lo + (uint64_t)(p0 + pl);
                bool amb = a.force_seq == 1;
                if (!M::exact) {
                    const T B2 = M::bound(a.n, total);
                    // the reference returns n-1 when no earlier prefix exceeds u
                    amb = amb || (gi == a.n - 1 ? !(U > prevE + B2) : (!(E > U + B2) || (gi > 0 && !(U > prevE + B2))));
                }
                for (int r = 0; r < C; ++r)
                    st_async_v4(mapa_rank(smem_addr(s_pk4[par]), r), (uint32_t)gi, (uint32_t)(gi >> 32), pcol,
                                amb ? 1u : 0u, mapa_rank(smem_addr(&s_bar[2 + par]), r));
            }
        }
        // no owner: complete this CTA's expected pick bytes itself (the phase must end)
        if (nf && t == 0) mbar_complete_local(&s_bar[2 + par], 16u);
        mbar_wait(&s_bar[2 + par], (ph_p >> par) & 1u);
        ph_p ^= 1u << par;
        if (!nf && !s_pk4[par][3]) { // the common case: every thread reads the pushed pick itself
            pick_col = s_pk4[par][2];
            return ((unsigned long long)s_pk4[par][1] << 32) | s_pk4[par][0];
        }
        // rare and uniform across the cluster: a target beyond every prefix (the
        // reference returns n-1) or an ambiguous fixed-point decision
        if (!wo) {
#pragma unroll
            for (int j = 0; j < PPT; ++j) s_md[p0 + j] = rm[j];
        }
        cl.sync(); // every CTA's min distances are in shared memory and stay untouched
        if (crank == 0 && t == 0) {
            bool seq = !nf || a.force_seq == 2;
            unsigned long long v = a.n - 1;
            const T total = s_total;
            if (nf && !seq && !M::exact && a.n > 1) {
                const uint64_t last = a.n - 1;
                const uint32_t r = (uint32_t)(last / chunk), li = (uint32_t)(last % chunk);
                const uint32_t cnt = *cl.map_shared_rank(s_cnt + li, r);
                const uint32_t md = wo ? kWeightsOnly : *cl.map_shared_rank(s_md + li, r);
                seq = !(U > total - M::mass_c(a, cnt, md) + M::bound(a.n, total));
            }
            if (seq) {
                v = cluster_sequential_draw<M>(a, cl, s_cnt, s_md, chunk, nu, wo ? 1 : 0);
                atomicAdd(a.fallbacks, 1ull);
            }
            s_pick = v;
        }
        cl.sync();
        if (t == 0) {
            const unsigned long long v = *cl.map_shared_rank(&s_pick, 0);
            s_fbv = v;
            s_fbc = colour_of(v);
        }
        __syncthreads();
        pick_col = s_fbc;
        return s_fbv;
    };

    int par = 0;
    uint32_t clast;
    if (a.kind == 1 || a.weighted_first) {
        T ts = 0;
#pragma unroll
        for (int j = 0; j < PPT; ++j) ts += M::mass_c(a, s_cnt[p0 + j], kWeightsOnly);
        const T tpre = publish(par, ts);
        draw(par, a.nu[0], true, ts, tpre, clast);
        par ^= 1;
    } else {
        clast = colour_of(a.first_index);
    }
    if (crank == 0 && t == 0) {
        a.cen[0] = (double)((clast >> 16) & 255u);
        a.cen[1] = (double)((clast >> 8) & 255u);
        a.cen[2] = (double)(clast & 255u);
    }
#ifdef CQG_INIT_TIMING
    unsigned long long _tprev = clock64();
#endif
    T ts_run = 0; // this thread's mass sum, kept across rounds (exact deltas)
    for (int k = 1; k < a.K; ++k) {
        uint32_t kcol = 0;
        const uint32_t bb = __dp4a(clast, clast, 0u);
        if (a.kind == 0) {
            unsigned long long best = 0;
            uint32_t bcol = 0;
#pragma unroll
            for (int j = 0; j < PPT; ++j) {
                const uint32_t d = d2_int_bb(rc[j], clast, bb);
                const uint32_t m = k == 1 ? d : min(rm[j], d);
                rm[j] = m;
                const unsigned long long key = ((unsigned long long)m << 32) | (uint32_t)~(uint32_t)(lo + p0 + j);
                if (p0 + j < mine && key > best) {
                    best = key;
                    bcol = rc[j];
                }
            }
            // (key, colour) maxima -> pushed into every CTA; every thread takes the max
            if (t == 0) mbar_arrive_expect(&s_bar[par], (uint32_t)(C * 16));
            for (int o = 16; o; o >>= 1) {
                const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o);
                const uint32_t xc = __shfl_xor_sync(0xffffffffu, bcol, o);
                if (x > best) {
                    best = x;
                    bcol = xc;
                }
            }
            if (lane == 0) {
                s_wkey[warp] = best;
                s_wcol[warp] = bcol;
            }
            __syncthreads();
            if (warp == 0) {
                unsigned long long b = lane < NT / 32 ? s_wkey[lane] : 0ull;
                uint32_t bc = lane < NT / 32 ? s_wcol[lane] : 0u;
                for (int o = 16; o; o >>= 1) {
                    const unsigned long long x = __shfl_xor_sync(0xffffffffu, b, o);
                    const uint32_t xc = __shfl_xor_sync(0xffffffffu, bc, o);
                    if (x > b) {
                        b = x;
                        bc = xc;
                    }
                }
                if (lane < C)
                    st_async_v4(mapa_rank(smem_addr(s_mk[par][crank]), lane), (uint32_t)b, (uint32_t)(b >> 32), bc, 0u,
                                mapa_rank(smem_addr(&s_bar[par]), lane));
            }
            mbar_wait(&s_bar[par], (ph_s >> par) & 1u);
            ph_s ^= 1u << par;
            unsigned long long b = 0;
            uint32_t bc = 0;
            for (int r = 0; r < C; ++r) {
                const unsigned long long x = ((unsigned long long)s_mk[par][r][1] << 32) | s_mk[par][r][0];
                if (x > b) {
                    b = x;
                    bc = s_mk[par][r][2];
                }
            }
            kcol = bc;
        } else {
            const double nu_k = __ldg(a.nu + k); // off the locate's critical path
            if (k == 1) {
#pragma unroll
                for (int j = 0; j < PPT; ++j) {
                    rm[j] = d2_int_bb(rc[j], clast, bb);
                    ts_run += M::mass_c(a, s_cnt[p0 + j], rm[j]);
                }
            } else if (!CQG_EXP_SKIP_UPDATE) {
                // only points closer to the new centre change: their mass
                // difference is subtracted from the running sum (exact)
                T delta = 0;
#pragma unroll
                for (int j = 0; j < PPT; j += 4) {
                    uint32_t d[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) d[u] = d2_int_bb(rc[j + u], clast, bb);
                    if ((d[0] < rm[j]) | (d[1] < rm[j + 1]) | (d[2] < rm[j + 2]) | (d[3] < rm[j + 3])) {
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (d[u] < rm[j + u]) {
                                const uint32_t cnt = s_cnt[p0 + j + u];
                                delta += M::mass_c(a, cnt, rm[j + u]) - M::mass_c(a, cnt, d[u]);
                                rm[j + u] = d[u];
                            }
                        }
                    }
                }
                ts_run -= delta;
            }
            ITIME(0);
            const T tpre = publish(par, ts_run);
            ITIME(1);
            draw(par, nu_k, false, ts_run, tpre, kcol);
            ITIME(3);
        }
        par ^= 1;
        clast = kcol;
        if (crank == 0 && t == 0) {
            a.cen[3 * k] = (double)((clast >> 16) & 255u);
            a.cen[3 * k + 1] = (double)((clast >> 8) & 255u);
            a.cen[3 * k + 2] = (double)(clast & 255u);
        }
        ITIME(4);
    }
    cl.sync(); // no CTA may exit while others still read its shared memory
}

// launch one 16-CTA cluster of `kern`; false when it cannot be resident
template <class... KArgs, class... Args>
static bool launch_cluster(cqg_ctx *ctx, const InitArgs &a, int nt, void (*kern)(KArgs...), size_t smem,
                           Args... args) {
    constexpr int C = 16;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        ensure_smem((const void *)kern, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess || clusters < 1) {
        cudaGetLastError();
        return false;
    }
    const int pb = prof_begin(ctx);
    CQG_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
    prof_end(ctx, CQG_PROF_INIT, pb, (double)a.n * (double)(a.K - 1));
    launched(ctx);
    return true;
}

// Try the cluster initialiser; false when the substrate does not fit.
template <class M>
static bool launch_cluster_init(cqg_ctx *ctx, InitArgs a) {
    constexpr int C = 16;
    const uint64_t per = (a.n + C - 1) / C;
    // Register kernel shape. A round's cost follows the padded point slots per
    // CTA (threads x points per thread, every slot updated and scanned), so
    // pick the (threads, ppt) pair with the fewest slots >= this CTA's share;
    // ppt is capped per size by the register budget (65536 / threads).
    // Measured: cfg2 k-means++ 1024x12 0.648 ms -> 896x12 0.596 ms; cfg1
    // maximin 1024x12 0.104 -> 512x20 0.085 ms. CQG_CLUSTER_NT forces a size.
    if (ctx->cluster_nt != kClusterThreads) {
        static const int kNt[5] = {512, 640, 768, 896, 1024}, kCap[5] = {24, 20, 16, 12, 12};
        int bi = -1, bp = 0;
        uint64_t bslots = ~0ull;
        for (int i = 0; i < 5; ++i) {
            if (ctx->cluster_nt > 0 && kNt[i] != ctx->cluster_nt) continue;
            const int pn = ((int)((per + kNt[i] - 1) / kNt[i]) + 3) & ~3;
            const uint64_t slots = (uint64_t)kNt[i] * pn;
            if (pn <= kCap[i] && slots < bslots) bi = i, bp = pn, bslots = slots;
        }
        if (bi >= 0 && kNt[bi] != kClusterThreads) {
            const size_t smn = bslots * 3 * sizeof(uint32_t);
#define CQG_REG_CASE(NTV, P) \
    if (kNt[bi] == NTV && bp == P) return launch_cluster(ctx, a, NTV, init_cluster_reg_kernel<M, P, NTV>, smn, a);
            CQG_REG_CASE(512, 4) CQG_REG_CASE(512, 8) CQG_REG_CASE(512, 12)
            CQG_REG_CASE(512, 16) CQG_REG_CASE(512, 20) CQG_REG_CASE(512, 24)
            CQG_REG_CASE(640, 4) CQG_REG_CASE(640, 8) CQG_REG_CASE(640, 12)
            CQG_REG_CASE(640, 16) CQG_REG_CASE(640, 20)
            CQG_REG_CASE(768, 4) CQG_REG_CASE(768, 8) CQG_REG_CASE(768, 12) CQG_REG_CASE(768, 16)
            CQG_REG_CASE(896, 4) CQG_REG_CASE(896, 8) CQG_REG_CASE(896, 12)
#undef CQG_REG_CASE
        }
    }
    // kClusterThreads threads per CTA: up to 12 points per thread (the register budget at 1024 threads;
    // up to 24 in a CQG_CLUSTER_THREADS < 1024 experiment build)
    const int ppt = ((int)((per + kClusterThreads - 1) / kClusterThreads) + 3) & ~3; // 128-bit runs
    if (ppt < 1 || !(ppt <= 12 || (kClusterThreads < 1024 && ppt <= 24))) return false;
    const size_t smem = (size_t)kClusterThreads * ppt * 3 * sizeof(uint32_t);
    if (smem > 227 * 1024) return false;
    constexpr int NT = kClusterThreads;
    switch (ppt) {
    case 4: return launch_cluster(ctx, a, NT, init_cluster_reg_kernel<M, 4, NT>, smem, a);
    case 8: return launch_cluster(ctx, a, NT, init_cluster_reg_kernel<M, 8, NT>, smem, a);
#if CQG_CLUSTER_THREADS < 1024
    case 16: return launch_cluster(ctx, a, NT, init_cluster_reg_kernel<M, 16, NT>, smem, a);
    case 20: return launch_cluster(ctx, a, NT, init_cluster_reg_kernel<M, 20, NT>, smem, a);
    case 24: return launch_cluster(ctx, a, NT, init_cluster_reg_kernel<M, 24, NT>, smem, a);
#endif
    default: return launch_cluster(ctx, a, NT, init_cluster_reg_kernel<M, 12, NT>, smem, a);
    }
}

static int tile_grid(const cqg_ctx *ctx, uint64_t threads) {
    uint64_t g = (threads + 255) / 256;
    const uint64_t gmax = (uint64_t)ctx->num_sms * 8;
    return (int)(g < 1 ? 1 : (g > gmax ? gmax : g));
}

void run_init(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n, uint64_t P,
              int K, uint64_t seed, int kind, int weighted_first, double *centers_d) {
    cudaStream_t s = ctx->stream;
    // draws from the reference's generator (rng.hpp:17-39), in consumption order
    std::mt19937_64 gen(seed);
    std::vector<double> nu;
    uint64_t first_index = 0;
    auto unit = [&gen]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
    if (kind == 0 && !weighted_first) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
        uint64_t x;
        do { x = gen(); } while (x >= limit);
        first_index = x % n;
        nu.push_back(0.0);
    } else {
        const int draws = kind == 1 ? K : 1;
        for (int i = 0; i < draws; ++i) nu.push_back(unit());
    }
    const bool exact = (P & (P - 1)) == 0 && P <= (1ull << 32);
    if (ctx->use_cluster_init && n <= 16ull * kClusterThreads * 32) {
        double *nu_c = static_cast<double *>(ctx->unit_draws.ensure(sizeof(double) * nu.size()));
        double *nu_h = static_cast<double *>(ctx->pinned_nu.ensure(sizeof(double) * nu.size()));
        std::memcpy(nu_h, nu.data(), sizeof(double) * nu.size());
        CQG_CUDA(cudaMemcpyAsync(nu_c, nu_h, sizeof(double) * nu.size(), cudaMemcpyHostToDevice, s));
        unsigned long long *resc = static_cast<unsigned long long *>(ctx->status.ensure(64));
        CQG_CUDA(cudaMemsetAsync(resc, 0, 64, s));
        InitArgs c{};
        c.colors = colors_d;
        c.counts = counts_d;
        c.n = n;
        c.inv = 1.0 / static_cast<double>(P);
        c.K = K;
        c.kind = kind;
        c.weighted_first = weighted_first;
        c.exact_sums = exact ? 1 : 0;
        c.first_index = first_index;
        c.nu = nu_c;
        c.result = resc;
        c.fallbacks = resc + 4;
        c.cen = centers_d;
        c.mds = 1;
        c.force_seq = ctx->dbg_init_force_seq;
        if (exact ? launch_cluster_init<ExactMass>(ctx, c) : launch_cluster_init<FixedMass>(ctx, c)) return;
    }
    // colour-space tiles: every colour on its own Morton slot (a duplicate
    // colour -- raw-pixel substrates -- keeps the record layout)
    bool tile = ctx->use_init_tile && n >= ctx->init_tile_min && n <= (1ull << 24);
    const uint64_t ntiles = (n + kTile - 1) / kTile;
    uint32_t *tbits = nullptr, *tpref = nullptr, *tbsum = nullptr;
    if (tile) {
        const size_t words = kTileBitmapWords;
        const size_t need = sizeof(uint32_t) * (2 * words + 1024 + 8) + sizeof(uint2) * n + sizeof(uint32_t) * 3 * n +
                            (sizeof(uint2) + sizeof(uint32_t) + sizeof(unsigned long long)) * ntiles + 512 +
                            sizeof(unsigned long long) * kFlagStride * (kLocateMax + 1);
        unsigned char *base = static_cast<unsigned char *>(ctx->inittile.ensure(need));
        tbits = reinterpret_cast<uint32_t *>(base);
        tpref = tbits + words;
        tbsum = tpref + words;
        uint32_t *dup_d = tbsum + 1024;
        CQG_CUDA(cudaMemsetAsync(tbits, 0, sizeof(uint32_t) * words, s));
        CQG_CUDA(cudaMemsetAsync(dup_d, 0, sizeof(uint32_t), s));
        const int g = tile_grid(ctx, n);
        tile_mark_kernel<<<g, 256, 0, s>>>(colors_d, n, tbits, dup_d);
        launched(ctx);
        uint32_t *dup_h = static_cast<uint32_t *>(ctx->pinned.ensure(4096));
        CQG_CUDA(cudaMemcpyAsync(dup_h, dup_d, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        CQG_CUDA(cudaStreamSynchronize(s));
        tile = *dup_h == 0;
    }
    const void *kern = tile ? (kind == 1 ? (exact ? (const void *)init_kernel_tile<ExactMass, 1> : (const void *)init_kernel_tile<FixedMass, 1>)
                                         : (exact ? (const void *)init_kernel_tile<ExactMass, 0> : (const void *)init_kernel_tile<FixedMass, 0>))
                            : (exact ? (const void *)init_kernel_rec<ExactMass> : (const void *)init_kernel_rec<FixedMass>);
    int occ = 0;
    CQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kInitThreads, 0));
    if (occ < 1) occ = 1;
    // k-means++ record rounds are load-latency bound: 3 blocks per SM (maximin
    // measured faster with 2: one barrier per round, fewer arrivals)
    // (tile rounds: 2 per SM -- fewer arrivals per hand-off; cfg3 2.34 -> 1.97 ms, cfg5 6.33 -> 6.12 ms vs 3)
    const int per_want = tile ? 2 : (kind == 1 ? 3 : 2);
    const int per_sm = occ > per_want ? per_want : occ;
    uint64_t grid = (uint64_t)ctx->num_sms * (uint64_t)per_sm;
    if (grid > (uint64_t)kLocateMax) grid = kLocateMax; // warp_locate scans <= kLocateMax block sums
    const uint64_t want = (n + kSeg - 1) / kSeg;
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    uint64_t chunk = (n + grid - 1) / grid;
    chunk = (chunk + kSeg - 1) / kSeg * kSeg;
    grid = (n + chunk - 1) / chunk;
    if (chunk / kSeg > (uint64_t)kLocateMax) fail(CQG_E_RUNTIME, "init: too many segments per block");
    const uint64_t nseg = (n + kSeg - 1) / kSeg;
    double *nu_d = static_cast<double *>(ctx->unit_draws.ensure(sizeof(double) * nu.size()));
    double *nu_h = static_cast<double *>(ctx->pinned_nu.ensure(sizeof(double) * nu.size()));
    std::memcpy(nu_h, nu.data(), sizeof(double) * nu.size());
    CQG_CUDA(cudaMemcpyAsync(nu_d, nu_h, sizeof(double) * nu.size(), cudaMemcpyHostToDevice, s));
    uint32_t *md = static_cast<uint32_t *>(ctx->mind2.ensure(sizeof(uint32_t) * 2 * n));
    const size_t part_bytes = sizeof(u128) * (2 * grid + 2 * nseg) + 8 * 2 * grid + 64;
    u128 *parts = static_cast<u128 *>(ctx->initpart.ensure(part_bytes));
    u128 *segs = parts + 2 * grid;
    unsigned long long *mparts = reinterpret_cast<unsigned long long *>(segs + 2 * nseg);
    unsigned long long *res = static_cast<unsigned long long *>(ctx->status.ensure(64));
    CQG_CUDA(cudaMemsetAsync(res, 0, 64, s));
    InitArgs a{};
    a.colors = colors_d;
    a.counts = counts_d;
    a.n = n;
    a.inv = 1.0 / static_cast<double>(P);
    a.K = K;
    a.kind = kind;
    a.weighted_first = weighted_first;
    a.exact_sums = exact ? 1 : 0;
    a.first_index = first_index;
    a.chunk = chunk;
    a.nu = nu_d;
    a.md = md;
    a.mds = 2; // {colour, md} records
    a.parts = parts;
    a.segs = segs;
    a.mparts = mparts;
    a.result = res;
    a.fallbacks = res + 4;
    a.cen = centers_d;
    if (tile) {
        unsigned char *tb = reinterpret_cast<unsigned char *>(tbsum + 1024 + 8);
        uint32_t *tcol = reinterpret_cast<uint32_t *>(tb);
        uint32_t *tmd = tcol + n;
        uint32_t *tidx = tmd + n;
        uint32_t *tcnt = tidx + n;
        uint32_t *hpos = tcnt + n;
        uint2 *tbox = reinterpret_cast<uint2 *>((reinterpret_cast<uintptr_t>(hpos + n) + 7) & ~(uintptr_t)7);
        uint32_t *tmax = reinterpret_cast<uint32_t *>(tbox + ntiles);
        unsigned long long *tkey = reinterpret_cast<unsigned long long *>(
            (reinterpret_cast<uintptr_t>(tmax + ntiles) + 7) & ~(uintptr_t)7);
        tile_scan_blocks<<<kTileBitmapWords / 1024, 1024, 0, s>>>(tbits, tpref, tbsum);
        tile_scan_top<<<1, 1024, 0, s>>>(tbsum, kTileBitmapWords / 1024);
        const int g = tile_grid(ctx, n);
        tile_expand_kernel<<<kTileBitmapWords / 256, 256, 0, s>>>(tbits, tpref, tbsum, tcol);
        tile_place_kernel<<<g, 256, 0, s>>>(colors_d, counts_d, n, tbits, tpref, tbsum, tidx, 1,
                                            kind == 1 ? hpos : nullptr);
        if (kind == 1) tile_count_kernel<<<g, 256, 0, s>>>(counts_d, tidx, n, tcnt);
        CQG_CUDA(cudaMemsetAsync(tmd, 0xFF, sizeof(uint32_t) * n, s));
        tile_box_kernel<<<tile_grid(ctx, ntiles * 32), 256, 0, s>>>(tcol, n, ntiles, tbox, tmax);
        launched(ctx, kind == 1 ? 6 : 5);
        a.md = nullptr;
        a.mds = 1;
        a.hpos = kind == 1 ? hpos : nullptr;
        a.tcol = tcol;
        a.tmd = tmd;
        a.tidx = tidx;
        a.tcnt = tcnt;
        a.tbox = tbox;
        a.tmax = tmax;
        a.tkey = tkey;
        a.ntiles = ntiles;
        unsigned long long *fl = reinterpret_cast<unsigned long long *>(
            (reinterpret_cast<uintptr_t>(tkey + ntiles) + 255) & ~(uintptr_t)255);
        CQG_CUDA(cudaMemsetAsync(fl, 0, sizeof(unsigned long long) * kFlagStride * grid, s));
        a.tflags = fl;
    }
    void *args[] = {&a};
    const int pb = prof_begin(ctx);
    CQG_CUDA(launch_cooperative(ctx, kern, dim3((unsigned)grid), dim3(kInitThreads), args, 0));
    prof_end(ctx, CQG_PROF_INIT, pb, (double)n * (double)(K - 1));
    launched(ctx);
}

} // namespace

void init_maximin_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n,
                      uint64_t P, int k, uint64_t seed, int weighted_first, double *centers_d) {
    run_init(ctx, colors_d, counts_d, n, P, k, seed, 0, weighted_first, centers_d);
}

void init_kmeanspp_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d,
                       uint64_t n, uint64_t P, int k, uint64_t seed, double *centers_d) {
    run_init(ctx, colors_d, counts_d, n, P, k, seed, 1, 1, centers_d);
}

} // namespace cqg

#ifdef CQG_INIT_TIMING
extern "C" int cqg_dbg_init_timing(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_init_timing, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(cqg::g_init_timing, z, sizeof(z));
    }
    return 0;
}
#endif

#ifdef CQG_INIT_TIMING
extern "C" int cqg_dbg_warp_hist(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_warp_hist, sizeof(cqg::g_warp_hist)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(cqg::g_warp_hist, z, sizeof(z));
    }
    return 0;
}
#endif

#ifdef CQG_INIT_TIMING
extern "C" int cqg_dbg_loc_phase(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_loc_phase, sizeof(cqg::g_loc_phase)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[4] = {};
        cudaMemcpyToSymbol(cqg::g_loc_phase, z, sizeof(z));
    }
    return 0;
}

extern "C" int cqg_dbg_tile_rounds(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_tile_rounds, sizeof(cqg::g_tile_rounds)) != cudaSuccess) return 1;
    if (reset) {
        static unsigned long long z[1024 * 2];
        cudaMemcpyToSymbol(cqg::g_tile_rounds, z, sizeof(z));
    }
    return 0;
}

extern "C" int cqg_dbg_coop_timing(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, cqg::g_coop_timing, 8 * sizeof(unsigned long long)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(cqg::g_coop_timing, z, sizeof(z));
    }
    return 0;
}
#endif
