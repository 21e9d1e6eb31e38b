// init.cu -- maximin and k-means++ initialisers on the device, bit-exact with
// the reference (src/init.cpp:37-52, 127-138, 295-314; rng.hpp:43-54).
//
// Centres are histogram colours, so every distance is an exact integer and
// min-distances are kept as uint32. One persistent cooperative kernel runs all
// K rounds; each block owns a contiguous index range so block partials are in
// histogram order.
//
//  maximin round:   mind2 = min(mind2, d2(x, c_last)); argmax (lowest index on
//                   ties, init.cpp:43-46) via a packed (mind2, ~index) u64 max.
//  weighted draw:   masses m_i = fl(fl(count_i * (1/P)) * mind2_i) exactly as the
//                   reference forms them; their sum is taken EXACTLY in 128-bit
//                   fixed point (2^-88 units), the draw u = fl(unit * total) is
//                   located by a prefix search, and the decision is accepted
//                   only when u lies farther than a rigorous bound on the
//                   reference's sequential-FP64 rounding from every prefix
//                   boundary; otherwise one thread replays the reference's
//                   sequential weighted_draw in FP64 (never observed; counted).
#include <cooperative_groups.h>

#include <random>

#include "cqg_internal.cuh"

namespace cg = cooperative_groups;

namespace cqg {
namespace {

typedef unsigned __int128 u128;
constexpr int kFix = 88;     // fixed-point fraction bits
constexpr int kInitThreads = 256;

struct InitArgs {
    const uint32_t *colors;
    const uint32_t *counts;
    uint64_t n;
    double inv;
    int K;
    int kind;           // 0 maximin, 1 k-means++
    int weighted_first; // maximin only
    uint64_t first_index;
    const double *nu;   // unit draws, in consumption order
    uint32_t *mind2;
    u128 *parts;                 // 2 x gridDim
    unsigned long long *mparts;  // 2 x gridDim
    unsigned long long *result;  // [0] chosen index of the current draw, [1] inexact flag
    unsigned long long *fallbacks;
    double *cen;
};

__device__ __forceinline__ u128 to_fixed(double m, int *inexact) {
    if (m == 0.0) return 0;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(m);
    const int e = (int)((bits >> 52) & 0x7FF);
    const unsigned long long mant = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    const int s = e - 1075 + kFix;
    if (s < 0) {
        *inexact = 1;
        return (u128)(mant >> (-s > 63 ? 63 : -s));
    }
    return ((u128)mant) << s;
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

__device__ __forceinline__ uint32_t d2_int(uint32_t a, uint32_t b) {
    const int dr = (int)((a >> 16) & 255u) - (int)((b >> 16) & 255u);
    const int dg = (int)((a >> 8) & 255u) - (int)((b >> 8) & 255u);
    const int db = (int)(a & 255u) - (int)(b & 255u);
    return (uint32_t)(dr * dr + dg * dg + db * db);
}

// mass of point i (mind2 == 0xFFFFFFFF means "weights only")
__device__ __forceinline__ double mass_of(const InitArgs &a, uint64_t i, uint32_t md) {
    const double w = __dmul_rn((double)a.counts[i], a.inv);
    return md == 0xFFFFFFFFu ? w : __dmul_rn(w, (double)md);
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

// block-wide sum (all threads get the result)
__device__ u128 block_sum_u128(u128 v, u128 *s_w) {
    for (int o = 16; o; o >>= 1) v += shfl_u128(v, (threadIdx.x & 31) ^ o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = v;
    __syncthreads();
    u128 t = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += s_w[i];
    __syncthreads();
    return t;
}

// block-wide exclusive scan; *total receives the block total
__device__ u128 block_excl_u128(u128 v, u128 *s_w, u128 *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    u128 incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const u128 t = shfl_up_u128(incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    u128 off = 0, tot = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
        if (i < wid) off += s_w[i];
        tot += s_w[i];
    }
    __syncthreads();
    *total = tot;
    return off + incl - v;
}

// Exact replay of rng.hpp:43-54 (one thread). Used only when the fast path
// cannot certify its decision.
__device__ uint64_t sequential_draw(const InitArgs &a, double nu, int weights_only) {
    double total = 0.0;
    for (uint64_t i = 0; i < a.n; ++i) total = __dadd_rn(total, mass_of(a, i, weights_only ? 0xFFFFFFFFu : a.mind2[i]));
    const double u = __dmul_rn(nu, total);
    double acc = 0.0;
    for (uint64_t i = 0; i + 1 < a.n; ++i) {
        acc = __dadd_rn(acc, mass_of(a, i, weights_only ? 0xFFFFFFFFu : a.mind2[i]));
        if (u < acc) return i;
    }
    return a.n - 1;
}

// Weighted draw over the current masses. Phase A (block sums) must already be
// in parts[par * gridDim.x + b]. Returns the chosen index in every block.
__device__ uint64_t draw(const InitArgs &a, cg::grid_group &grid, int par, double nu, int weights_only,
                         uint64_t lo, uint64_t hi, u128 *s_w, unsigned long long *s_res) {
    const u128 *parts = a.parts + (size_t)par * gridDim.x;
    // every block: total, u, target block
    __shared__ u128 s_before;
    __shared__ int s_tblock;
    __shared__ u128 s_U, s_T;
    if (threadIdx.x == 0) {
        u128 T = 0;
        for (unsigned b = 0; b < gridDim.x; ++b) T += parts[b];
        const double u = __dmul_rn(nu, fixed_to_double(T));
        const u128 U = floor_fixed(u);
        u128 run = 0;
        int tb = -1;
        u128 before = 0;
        for (unsigned b = 0; b < gridDim.x; ++b) {
            if (run + parts[b] > U) {
                tb = (int)b;
                before = run;
                break;
            }
            run += parts[b];
        }
        s_tblock = tb;
        s_before = before;
        s_U = U;
        s_T = T;
    }
    __syncthreads();
    const int tb = s_tblock;
    const u128 U = s_U, T = s_T;
    // rigorous bound on |reference prefix / u - exact| (units 2^-88), doubled
    const u128 B2 = (u128)2 * (u128)(a.n + 4) * ((T >> 52) + 1) + 2;
    // the block holding the crossing (or the last block if u >= total) searches
    const int searcher = tb >= 0 ? tb : (int)gridDim.x - 1;
    if ((int)blockIdx.x == searcher) {
        __shared__ unsigned long long s_found;
        __shared__ u128 s_prevE, s_E;
        if (threadIdx.x == 0) s_found = ~0ull;
        __syncthreads();
        int inexact = 0;
        if (tb >= 0) {
            u128 run = s_before;
            for (uint64_t base = lo; base < hi; base += 8ull * blockDim.x) {
                u128 m[8];
                u128 loc = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint64_t i = base + 8ull * threadIdx.x + j;
                    m[j] = i < hi ? to_fixed(mass_of(a, i, weights_only ? 0xFFFFFFFFu : a.mind2[i]), &inexact) : 0;
                    loc += m[j];
                }
                u128 btot;
                const u128 start = run + block_excl_u128(loc, s_w, &btot);
                if (start <= U && start + loc > U) {
                    u128 acc = start;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const u128 nxt = acc + m[j];
                        if (nxt > U) {
                            s_found = base + 8ull * threadIdx.x + j;
                            s_prevE = acc;
                            s_E = nxt;
                            break;
                        }
                        acc = nxt;
                    }
                }
                __syncthreads();
                if (s_found != ~0ull) break;
                run += btot;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t idx;
            bool ambiguous;
            if (s_found == ~0ull || s_found >= a.n - 1) {
                // reference returns n-1: need U clearly above E_{n-2}
                idx = a.n - 1;
                int ix = 0;
                const u128 mlast = to_fixed(mass_of(a, a.n - 1, weights_only ? 0xFFFFFFFFu : a.mind2[a.n - 1]), &ix);
                inexact |= ix;
                const u128 Enm2 = T - mlast;
                ambiguous = a.n > 1 && !(U > Enm2 + B2);
            } else {
                idx = s_found;
                ambiguous = !(s_E > U + B2) || (idx > 0 && !(U > s_prevE + B2));
            }
            s_res[0] = idx;
            s_res[1] = (ambiguous || inexact) ? 1ull : 0ull;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_res[1]) {
                s_res[0] = sequential_draw(a, nu, weights_only);
                atomicAdd(a.fallbacks, 1ull);
            }
            a.result[par] = s_res[0];
        }
    }
    grid.sync();
    return a.result[par];
}

__global__ void __launch_bounds__(kInitThreads) init_kernel(InitArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ u128 s_w[kInitThreads / 32];
    __shared__ unsigned long long s_res[2];
    __shared__ unsigned long long s_m[kInitThreads / 32];
    const uint64_t chunk = (a.n + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = (uint64_t)blockIdx.x * chunk;
    const uint64_t hi = lo + chunk < a.n ? lo + chunk : a.n;
    int par = 0;
    int inexact = 0;

    // ---- first centre ---------------------------------------------------
    uint64_t first;
    if (a.kind == 1 || a.weighted_first) {
        u128 loc = 0;
        for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) loc += to_fixed(mass_of(a, i, 0xFFFFFFFFu), &inexact);
        const u128 t = block_sum_u128(loc, s_w);
        if (threadIdx.x == 0) a.parts[(size_t)par * gridDim.x + blockIdx.x] = t;
        grid.sync();
        first = draw(a, grid, par, a.nu[0], 1, lo, hi, s_w, s_res);
        par ^= 1;
    } else {
        first = a.first_index;
    }
    uint32_t clast = a.colors[first];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.cen[0] = (double)((clast >> 16) & 255u);
        a.cen[1] = (double)((clast >> 8) & 255u);
        a.cen[2] = (double)(clast & 255u);
    }

    for (int k = 1; k < a.K; ++k) {
        // update min distances with the last centre; per-block partial
        if (a.kind == 0) {
            unsigned long long best = 0;
            for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const uint32_t d = d2_int(a.colors[i], clast);
                const uint32_t md = (k == 1) ? d : min(a.mind2[i], d);
                a.mind2[i] = md;
                const unsigned long long key = ((unsigned long long)md << 32) | (uint32_t)~(uint32_t)i;
                best = key > best ? key : best;
            }
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
            for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
                const unsigned long long t = a.mparts[(size_t)par * gridDim.x + i];
                b = t > b ? t : b;
            }
            for (int o = 16; o; o >>= 1) {
                const unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
                b = t > b ? t : b;
            }
            if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = b;
            __syncthreads();
            b = 0;
            for (int i = 0; i < kInitThreads / 32; ++i) b = s_m[i] > b ? s_m[i] : b;
            __syncthreads();
            // index = ~low32 (indices < 2^32)
            const uint64_t pick = (uint64_t)(uint32_t)~(uint32_t)(b & 0xFFFFFFFFull);
            clast = a.colors[pick];
        } else {
            u128 loc = 0;
            for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
                const uint32_t d = d2_int(a.colors[i], clast);
                const uint32_t md = (k == 1) ? d : min(a.mind2[i], d);
                a.mind2[i] = md;
                loc += to_fixed(mass_of(a, i, md), &inexact);
            }
            const u128 t = block_sum_u128(loc, s_w);
            if (threadIdx.x == 0) a.parts[(size_t)par * gridDim.x + blockIdx.x] = t;
            grid.sync();
            const uint64_t pick = draw(a, grid, par, a.nu[k], 0, lo, hi, s_w, s_res);
            clast = a.colors[pick];
        }
        par ^= 1;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.cen[3 * k] = (double)((clast >> 16) & 255u);
            a.cen[3 * k + 1] = (double)((clast >> 8) & 255u);
            a.cen[3 * k + 2] = (double)(clast & 255u);
        }
    }
    if (inexact) atomicAdd(a.fallbacks, 0ull); // masses below 2^-36 only for P > 2^32
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
    int occ = 0;
    CQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, init_kernel, kInitThreads, 0));
    if (occ < 1) occ = 1;
    uint64_t grid = (uint64_t)ctx->num_sms * (uint64_t)(occ > 2 ? 2 : occ);
    const uint64_t want = (n + 4 * kInitThreads - 1) / (4 * kInitThreads);
    if (grid > want) grid = want;
    if (grid < 1) grid = 1;
    double *nu_d = static_cast<double *>(ctx->unit_draws.ensure(sizeof(double) * nu.size()));
    CQG_CUDA(cudaMemcpyAsync(nu_d, nu.data(), sizeof(double) * nu.size(), cudaMemcpyHostToDevice, s));
    uint32_t *mind2 = static_cast<uint32_t *>(ctx->mind2.ensure(sizeof(uint32_t) * n));
    u128 *parts = static_cast<u128 *>(ctx->initpart.ensure(sizeof(u128) * 2 * grid + 16 * 2 * grid + 64));
    unsigned long long *mparts = reinterpret_cast<unsigned long long *>(parts + 2 * grid);
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
    a.first_index = first_index;
    a.nu = nu_d;
    a.mind2 = mind2;
    a.parts = parts;
    a.mparts = mparts;
    a.result = res;
    a.fallbacks = res + 4;
    a.cen = centers_d;
    void *args[] = {&a};
    const int pb = prof_begin(ctx);
    CQG_CUDA(cudaLaunchCooperativeKernel((const void *)init_kernel, dim3((unsigned)grid), dim3(kInitThreads),
                                         args, 0, s));
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
