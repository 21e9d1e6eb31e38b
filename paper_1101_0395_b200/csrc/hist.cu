// hist.cu -- stage 1: distinct colours in first-occurrence order.
//
// Replaces quant::build_histogram (reference src/histogram.cpp:69-104). The
// reference dedups through a seeded chained hash and appends colours on first
// sight, so its output order is "by first pixel index". Here:
//
//   A  hist_count   per pixel (16 pixels / thread, 3 x 128-bit loads):
//                   atomicAdd(count[c]) with return -> the lane that sees 0
//                   appends c to an (unordered) list (warp-aggregated append);
//                   atomicMax(~first[c], ~p) keeps the minimum index.
//                   Small images: both in one pass over an interleaved
//                   {count, ~first} table. Large images (P >= 2^22): two passes
//                   of fire-and-forget reductions (hist_count_red, hist_first)
//                   over split 64 MiB tables (each fits the 126 MB L2), then a
//                   third pass marks the first occurrences straight from the
//                   image (~first[c] == p) -- no unique-colour list, no global
//                   append counter; N' is the bitmap's popcount from the scan.
//   B  hist_mark    per listed colour: set bit first(c) in a P-bit bitmap.
//   C  scan         popcount prefix over the bitmap words (2 small kernels).
//   D  emit         small: per listed colour, rank = prefix(first(c)), write at
//                   that rank and zero the table entry. Large: one thread per
//                   pixel in pixel order -- a set bit is a first occurrence with
//                   rank = word prefix + bits below, so stores are sequential;
//                   the tables are reset with one 128 MiB memset.
//
// The tables (2^24 counts | 2^24 ~first) are 128 MiB and live in the context;
// they are zero between calls. HBM bound: 6P bytes read + 8N' written + atomics.
#include "cqg_internal.cuh"

namespace cqg {
namespace {

constexpr int kThreads = 256;
constexpr int kWordsPerThread = 16;                         // scan granularity
constexpr int kWordsPerBlock = kThreads * kWordsPerThread;  // 4096 words = 131072 pixels

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// Decode 16 packed RGB pixels from 48 bytes (little-endian words).
__device__ __forceinline__ void decode16(const uint4 &a, const uint4 &b, const uint4 &d, uint32_t *col) {
    const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int o = 3 * j;
        const uint32_t b0 = (w[o >> 2] >> (8 * (o & 3))) & 255u;
        const uint32_t b1 = (w[(o + 1) >> 2] >> (8 * ((o + 1) & 3))) & 255u;
        const uint32_t b2 = (w[(o + 2) >> 2] >> (8 * ((o + 2) & 3))) & 255u;
        col[j] = (b0 << 16) | (b1 << 8) | b2;
    }
}

__device__ __forceinline__ void append(bool isnew, uint32_t c, uint32_t *list, uint32_t *list_n) {
    const uint32_t active = __activemask();
    const uint32_t m = __ballot_sync(active, isnew);
    if (m == 0) return;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(list_n, (uint32_t)__popc(m));
    base = __shfl_sync(active, base, leader);
    if (isnew) list[base + __popc(m & lanemask_lt())] = c;
}

// ---- small images: one interleaved table {count, ~first} (one sector per colour)

__global__ void __launch_bounds__(kThreads) hist_count_fused(const uint8_t *__restrict__ rgb, uint64_t P,
                                                            uint2 *__restrict__ tab, uint32_t *__restrict__ list,
                                                            uint32_t *__restrict__ list_n, int aligned) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t groups = aligned ? P / 16 : 0;
    for (uint64_t g = tid; g < groups; g += stride) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rgb + g * 48);
        uint32_t col[16];
        decode16(ld_stream(src), ld_stream(src + 1), ld_stream(src + 2), col);
        bool isnew[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            isnew[j] = atomicAdd(&tab[col[j]].x, 1u) == 0;
            atomicMax(&tab[col[j]].y, ~(uint32_t)(g * 16 + j));
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) append(isnew[j], col[j], list, list_n);
    }
    // tail (or everything when the input is not 16-byte aligned)
    for (uint64_t p = groups * 16 + tid; p < P; p += stride) {
        const uint32_t c = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
        const bool isnew = atomicAdd(&tab[c].x, 1u) == 0;
        atomicMax(&tab[c].y, ~(uint32_t)p);
        append(isnew, c, list, list_n);
    }
}

__global__ void hist_mark_fused(const uint32_t *__restrict__ list, const uint32_t *__restrict__ list_n,
                                const uint2 *__restrict__ tab, uint32_t *__restrict__ bitmap) {
    const uint32_t n = *list_n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t f = ~tab[list[i]].y;
        atomicOr(&bitmap[f >> 5], 1u << (f & 31));
    }
}

// per listed colour: rank = prefix(first(c)); write at that rank, reset tab[c]
__global__ void hist_emit_fused(const uint32_t *__restrict__ list, const uint32_t *__restrict__ list_n,
                                uint2 *__restrict__ tab, const uint32_t *__restrict__ bitmap,
                                const uint32_t *__restrict__ wpref, uint32_t *__restrict__ colors,
                                uint32_t *__restrict__ counts, uint32_t *__restrict__ first) {
    const uint32_t n = *list_n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t c = list[i];
        const uint2 t = tab[c];
        const uint32_t f = ~t.y;
        const uint32_t w = f >> 5;
        const uint32_t rank = wpref[w] + __popc(bitmap[w] & ((1u << (f & 31)) - 1u));
        colors[rank] = c;
        counts[rank] = t.x;
        if (first) first[rank] = f;
        tab[c] = make_uint2(0u, 0u);
    }
}

// ---- large images: split tables cnt | negf (64 MiB each), two passes

// large images: counts by reductions (no return value, no list)
__global__ void __launch_bounds__(kThreads) hist_count_red(const uint8_t *__restrict__ rgb, uint64_t P,
                                                          uint32_t *__restrict__ cnt, int aligned) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t groups = aligned ? P / 16 : 0;
    for (uint64_t g = tid; g < groups; g += stride) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rgb + g * 48);
        uint32_t col[16];
        decode16(ld_stream(src), ld_stream(src + 1), ld_stream(src + 2), col);
#pragma unroll
        for (int j = 0; j < 16; ++j) atomicAdd(cnt + col[j], 1u);
    }
    for (uint64_t p = groups * 16 + tid; p < P; p += stride) {
        const uint32_t c = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
        atomicAdd(cnt + c, 1u);
    }
}

// large images: first-occurrence bitmap from the ~first table instead of a
// third image pass: every present colour sets the bit of its first pixel
// (coalesced 16-byte reads of the 64 MiB table, one reduction per colour into
// the L2-resident bitmap; a pass over the image re-read it and looked up the
// table per pixel: 865 MB of DRAM reads on an 8192^2 image)
__global__ void __launch_bounds__(kThreads) hist_mark_table(const uint32_t *__restrict__ negf,
                                                           uint32_t *__restrict__ bitmap) {
    const uint4 *t4 = reinterpret_cast<const uint4 *>(negf);
    constexpr uint32_t n4 = (1u << 24) / 4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(t4 + i);
        const uint32_t f[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (f[j]) {
                const uint32_t p = ~f[j];
                atomicOr(&bitmap[p >> 5], 1u << (p & 31));
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) hist_first(const uint8_t *__restrict__ rgb, uint64_t P,
                                                      uint32_t *__restrict__ negf, int aligned) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t groups = aligned ? P / 16 : 0;
    for (uint64_t g = tid; g < groups; g += stride) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rgb + g * 48);
        uint32_t col[16];
        decode16(ld_stream(src), ld_stream(src + 1), ld_stream(src + 2), col);
#pragma unroll
        for (int j = 0; j < 16; ++j) atomicMax(negf + col[j], ~(uint32_t)(g * 16 + j));
    }
    for (uint64_t p = groups * 16 + tid; p < P; p += stride) {
        const uint32_t c = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
        atomicMax(negf + c, ~(uint32_t)p);
    }
}


// one thread per pixel, in pixel order: a set bit is a first occurrence whose
// rank is the word prefix plus the set bits below it, so the stores of a warp
// land on consecutive ranks (the colour comes from the image itself)
__global__ void __launch_bounds__(kThreads) hist_emit(const uint8_t *__restrict__ rgb, uint64_t P,
                                                     const uint32_t *__restrict__ bitmap,
                                                     const uint32_t *__restrict__ wpref,
                                                     const uint32_t *__restrict__ cnt,
                                                     uint32_t *__restrict__ colors, uint32_t *__restrict__ counts,
                                                     uint32_t *__restrict__ first) {
    for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = p >> 5;
        const uint32_t bits = __ldg(bitmap + w);
        const uint32_t b = (uint32_t)(p & 31);
        if (!((bits >> b) & 1u)) continue;
        const uint32_t rank = __ldg(wpref + w) + __popc(bits & ((1u << b) - 1u));
        const uint32_t c = ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2];
        colors[rank] = c;
        counts[rank] = __ldg(cnt + c);
        if (first) first[rank] = (uint32_t)p;
    }
}

// block sums of popcounts over kWordsPerBlock words
__global__ void __launch_bounds__(kThreads) scan_blocksum(const uint32_t *__restrict__ bitmap,
                                                          uint64_t words, uint32_t *__restrict__ bsum) {
    __shared__ uint32_t red[kThreads / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kWordsPerBlock + (uint64_t)threadIdx.x * kWordsPerThread;
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kWordsPerThread; ++i)
        if (base + i < words) s += __popc(bitmap[base + i]);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int i = 0; i < kThreads / 32; ++i) t += red[i];
        bsum[blockIdx.x] = t;
    }
}

// exclusive scan of the block sums (one block, sequential chunks)
__global__ void scan_blocks(uint32_t *__restrict__ bsum, uint32_t nblocks, uint32_t *__restrict__ n_out) {
    __shared__ uint32_t carry;
    __shared__ uint32_t tmp[1024];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint32_t base = 0; base < nblocks; base += 1024) {
        const uint32_t i = base + threadIdx.x;
        const uint32_t v = i < nblocks ? bsum[i] : 0;
        tmp[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < 1024; off <<= 1) {
            const uint32_t add = threadIdx.x >= (unsigned)off ? tmp[threadIdx.x - off] : 0;
            __syncthreads();
            tmp[threadIdx.x] += add;
            __syncthreads();
        }
        if (i < nblocks) bsum[i] = carry + tmp[threadIdx.x] - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry += tmp[1023];
        __syncthreads();
    }
    if (n_out && threadIdx.x == 0) *n_out = carry; // the number of set bits: N'
}

// per-word exclusive prefix (global)
__global__ void __launch_bounds__(kThreads) scan_words(const uint32_t *__restrict__ bitmap, uint64_t words,
                                                       const uint32_t *__restrict__ bsum,
                                                       uint32_t *__restrict__ wpref) {
    __shared__ uint32_t wsum[kThreads / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kWordsPerBlock + (uint64_t)threadIdx.x * kWordsPerThread;
    uint32_t pc[kWordsPerThread];
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < kWordsPerThread; ++i) {
        pc[i] = (base + i < words) ? __popc(bitmap[base + i]) : 0;
        s += pc[i];
    }
    // exclusive scan of s across the block
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    uint32_t woff = 0;
    for (int i = 0; i < wid; ++i) woff += wsum[i];
    uint32_t run = bsum[blockIdx.x] + woff + incl - s;
#pragma unroll
    for (int i = 0; i < kWordsPerThread; ++i) {
        if (base + i < words) wpref[base + i] = run;
        run += pc[i];
    }
}

// subsample_2to1 (histogram.cpp:60-67): pixels at even (x, y), row-major
__global__ void subsample_kernel(const uint8_t *__restrict__ rgb, int w, int h, uint8_t *__restrict__ out) {
    const int ws = (w + 1) / 2, hs = (h + 1) / 2;
    const uint64_t S = (uint64_t)ws * hs;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t y = i / ws, x = i - y * ws;
        const uint64_t src = 3 * (2 * y * (uint64_t)w + 2 * x);
        out[3 * i] = rgb[src];
        out[3 * i + 1] = rgb[src + 1];
        out[3 * i + 2] = rgb[src + 2];
    }
}

// raw substrate (pipeline.cpp:103-108): every sampled pixel is a point of count 1
__global__ void pack_kernel(const uint8_t *__restrict__ rgb, uint64_t S, uint32_t *__restrict__ colors,
                            uint32_t *__restrict__ counts) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += (uint64_t)gridDim.x * blockDim.x) {
        colors[i] = ((uint32_t)rgb[3 * i] << 16) | ((uint32_t)rgb[3 * i + 1] << 8) | rgb[3 * i + 2];
        counts[i] = 1u;
    }
}

} // namespace

void histogram_dev(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t P, uint32_t *colors_d,
                   uint32_t *counts_d, uint32_t *first_d, uint32_t *n_dev) {
    cudaStream_t s = ctx->stream;
    if (ctx->tab.cap < (sizeof(uint2) << 24)) {
        ctx->tab.ensure(sizeof(uint2) << 24);
        CQG_CUDA(cudaMemsetAsync(ctx->tab.p, 0, sizeof(uint2) << 24, s));
    }
    const uint64_t cap = P < (1ull << 24) ? P : (1ull << 24);
    uint32_t *list = static_cast<uint32_t *>(ctx->list.ensure(cap * 4));
    const uint64_t words = (P + 31) / 32;
    const uint32_t nblk = ceil_div(words, kWordsPerBlock);
    uint32_t *bitmap = static_cast<uint32_t *>(ctx->bitmap.ensure(words * 4 + 16));
    uint32_t *wpref = static_cast<uint32_t *>(ctx->wordpref.ensure(words * 4 + 16 + (size_t)nblk * 4));
    uint32_t *bsum = wpref + words + 4;

    const int pb = prof_begin(ctx);
    CQG_CUDA(cudaMemsetAsync(n_dev, 0, 4, s));
    CQG_CUDA(cudaMemsetAsync(bitmap, 0, words * 4, s));

    const int aligned = (reinterpret_cast<uintptr_t>(rgb_d) & 15) == 0;
    const uint64_t work = aligned ? (P / 16 > 0 ? P / 16 : P) : P;
    unsigned grid = ceil_div(work, kThreads);
    const unsigned gmax = (unsigned)ctx->num_sms * 8;
    if (grid > gmax) grid = gmax;
    if (grid == 0) grid = 1;
    unsigned lgrid = ceil_div(cap, kThreads);
    if (lgrid > gmax) lgrid = gmax;
    // small images: one pass over the interleaved table (L2-resident anyway),
    // emit + reset per listed colour. Large images: two passes over split
    // 64 MiB tables (each fits the L2), emit in pixel order, one memset reset.
    const bool large = P >= (1ull << 22);
    uint2 *tab = ctx->tab.as<uint2>();
    uint32_t *cnt = ctx->tab.as<uint32_t>(), *negf = cnt + (1u << 24);
    if (!large) {
        hist_count_fused<<<grid, kThreads, 0, s>>>(rgb_d, P, tab, list, n_dev, aligned);
        hist_mark_fused<<<lgrid, kThreads, 0, s>>>(list, n_dev, tab, bitmap);
    } else {
        // counts and minimum indices by reductions; the bitmap from the
        // first-index table (no unique-colour list, no global append counter)
        hist_count_red<<<grid, kThreads, 0, s>>>(rgb_d, P, cnt, aligned);
        hist_first<<<grid, kThreads, 0, s>>>(rgb_d, P, negf, aligned);
        hist_mark_table<<<(unsigned)ctx->num_sms * 8, kThreads, 0, s>>>(negf, bitmap);
    }
    scan_blocksum<<<nblk, kThreads, 0, s>>>(bitmap, words, bsum);
    scan_blocks<<<1, 1024, 0, s>>>(bsum, nblk, large ? n_dev : nullptr);
    scan_words<<<nblk, kThreads, 0, s>>>(bitmap, words, bsum, wpref);
    if (!large) {
        hist_emit_fused<<<lgrid, kThreads, 0, s>>>(list, n_dev, tab, bitmap, wpref, colors_d, counts_d, first_d);
    } else {
        const unsigned egrid = (unsigned)ctx->num_sms * 8;
        hist_emit<<<egrid, kThreads, 0, s>>>(rgb_d, P, bitmap, wpref, cnt, colors_d, counts_d, first_d);
        CQG_CUDA(cudaMemsetAsync(ctx->tab.p, 0, sizeof(uint2) << 24, s));
    }
    prof_end(ctx, CQG_PROF_HIST, pb, 3.0 * (double)P); // + 8 N' added by the caller
    CQG_CUDA(cudaGetLastError());
    launched(ctx, large ? 7 : 6);
}

void subsample_2to1_dev(cqg_ctx *ctx, const uint8_t *rgb_d, int w, int h, uint8_t *out_d) {
    const uint64_t S = (uint64_t)((w + 1) / 2) * ((h + 1) / 2);
    unsigned grid = ceil_div(S, kThreads);
    if (grid > (unsigned)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    subsample_kernel<<<grid ? grid : 1, kThreads, 0, ctx->stream>>>(rgb_d, w, h, out_d);
    CQG_CUDA(cudaGetLastError());
    launched(ctx);
}

void pack_pixels_dev(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t S, uint32_t *colors_d, uint32_t *counts_d) {
    unsigned grid = ceil_div(S, kThreads);
    if (grid > (unsigned)ctx->num_sms * 8) grid = ctx->num_sms * 8;
    pack_kernel<<<grid ? grid : 1, kThreads, 0, ctx->stream>>>(rgb_d, S, colors_d, counts_d);
    CQG_CUDA(cudaGetLastError());
    launched(ctx);
}

} // namespace cqg

// ---------------------------------------------------------------------------
// Coarse 32x32x32 histogram (quant::build_coarse_histogram,
// src/precluster.cpp:13-47): per bin (r>>3, g>>3, b>>3) the pixel count and
// exact sums of r, g, b and r^2+g^2+b^2. Built from the distinct colours and
// their counts (5 reductions per colour instead of per pixel; the totals are
// the same integers), straight into the L2-resident 1.3 MiB table as
// fire-and-forget u64 adds (the colours come in first-occurrence order, not
// grouped by bin, so a shared-memory slice per block would not localise them).
namespace cqg {
namespace {
__global__ void __launch_bounds__(256) coarse_hist_kernel(const uint32_t *__restrict__ colors,
                                                         const uint32_t *__restrict__ counts, uint64_t n,
                                                         unsigned long long *__restrict__ tab) {
    // tab: 5 x 32768 u64 -- count | sum_r | sum_g | sum_b | sum_sq
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = __ldg(colors + i);
        const unsigned long long cnt = __ldg(counts + i);
        const uint32_t r = (c >> 16) & 255u, g = (c >> 8) & 255u, b = c & 255u;
        const uint32_t bin = ((r >> 3) << 10) | ((g >> 3) << 5) | (b >> 3);
        atomicAdd(tab + bin, cnt);
        atomicAdd(tab + 32768 + bin, cnt * r);
        atomicAdd(tab + 2 * 32768 + bin, cnt * g);
        atomicAdd(tab + 3 * 32768 + bin, cnt * b);
        atomicAdd(tab + 4 * 32768 + bin, cnt * (unsigned long long)(r * r + g * g + b * b));
    }
}
} // namespace

void coarse_hist_dev(cqg_ctx *ctx, const uint32_t *colors_d, const uint32_t *counts_d, uint64_t n,
                     unsigned long long *tab_d) {
    cudaStream_t s = ctx->stream;
    CQG_CUDA(cudaMemsetAsync(tab_d, 0, sizeof(unsigned long long) * 5 * 32768, s));
    unsigned grid = (unsigned)((n + 255) / 256);
    const unsigned gmax = (unsigned)ctx->num_sms * 8;
    if (grid > gmax) grid = gmax;
    if (grid == 0) grid = 1;
    coarse_hist_kernel<<<grid, 256, 0, s>>>(colors_d, counts_d, n, tab_d);
    CQG_CUDA(cudaGetLastError());
    launched(ctx);
}
} // namespace cqg
