// hist.cu -- stage 1: distinct colours in first-occurrence order.
//
// Replaces quant::build_histogram (reference src/histogram.cpp:69-104). The
// reference dedups through a seeded chained hash and appends colours on first
// sight, so its output order is "by first pixel index". Here:
//
// Small images (P < 2^22): one pass over an interleaved {count, ~first} table
//   of 2^24 entries (L2-resident): per pixel atomicAdd(count) with return (the
//   lane that sees 0 appends the colour to a list, warp-aggregated) and
//   atomicMax(~first); per listed colour one bit at its first pixel in a P-bit
//   bitmap; popcount scan; per listed colour rank = prefix(first), write at
//   that rank and zero the table entry.
// Large images (P >= 2^22): the random L2 atomics per pixel (two per pixel,
//   ~156 G/s on B200) are replaced by a colour-bucketed partition with the
//   aggregation in shared memory (part_count -> part_scatter -> bucket_agg,
//   below); bucket_agg writes the dense per-colour counts and marks each
//   colour's first pixel in the bitmap; popcount scan; one pass over the
//   pixels in pixel order emits every first occurrence at rank = word prefix
//   + bits below (sequential stores), its count gathered from the table.
// Only distinct colours touch L2 at random (bitmap mark, count gather).
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
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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

// The per-colour counts come from bucket_agg as a saturating u8 table (16 MiB:
// it stays in L2 between the aggregation and the emit, where the 64 MiB u32
// table was re-read from DRAM by one sector per gather); a count >= 255 is in
// the sparse u32 side table.
__device__ __forceinline__ uint32_t count_of(const uint8_t *__restrict__ cnt8, const uint32_t *__restrict__ cnt32,
                                             uint32_t c) {
    const uint32_t n = __ldg(cnt8 + c);
    return n == 255u ? __ldg(cnt32 + c) : n;
}

// pixel order, 512 pixels per warp pass (16 per lane: 48 bytes and one bitmap
// half-word). A set bit is a first occurrence whose rank is the word prefix
// plus the set bits below it. Each lane drops its first occurrences (colour,
// pixel offset) into the warp's shared-memory row at rank - warp base; the warp
// then walks the row with all lanes busy: count gathers in flight together,
// stores on consecutive ranks. The image loads do not depend on the preceding
// kernels and are issued before the dependency wait.
constexpr int kEmitWarps = kThreads / 32;
__global__ void __launch_bounds__(kThreads) hist_emit16(const uint8_t *__restrict__ rgb, uint64_t groups,
                                                       const uint32_t *__restrict__ bitmap,
                                                       const uint32_t *__restrict__ wpref,
                                                       const uint8_t *__restrict__ cnt8,
                                                       const uint32_t *__restrict__ cnt32,
                                                       uint32_t *__restrict__ colors, uint32_t *__restrict__ counts,
                                                       uint32_t *__restrict__ first) {
    __shared__ uint32_t s_col[kEmitWarps][512];
    __shared__ uint16_t s_off[kEmitWarps][512];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x; // a multiple of 32: a warp's groups stay consecutive
    uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint4 a = {}, b = {}, d = {};
    if (g < groups) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rgb + g * 48);
        a = ld_stream(src);
        b = ld_stream(src + 1);
        d = ld_stream(src + 2);
    }
    pdl_wait();
    pdl_trigger();
    for (uint64_t g0 = g - lane; g0 < groups; g0 += stride, g += stride) { // warp-uniform trip count
        const bool v = g < groups;
        const uint32_t word = v ? __ldg(bitmap + (g >> 1)) : 0u;
        const uint32_t hi = (uint32_t)(g & 1);
        const uint32_t bits = (word >> (16 * hi)) & 0xFFFFu;
        const uint32_t rank = v ? __ldg(wpref + (g >> 1)) + (hi ? __popc(word & 0xFFFFu) : 0u) : 0u;
        uint4 na = {}, nb = {}, nd = {};
        if (g + stride < groups) {
            const uint4 *src = reinterpret_cast<const uint4 *>(rgb + (g + stride) * 48);
            na = ld_stream(src);
            nb = ld_stream(src + 1);
            nd = ld_stream(src + 2);
        }
        const uint32_t base = __shfl_sync(0xffffffffu, rank, 0);
        // the warp's first occurrences: the last valid lane's rank + its bits
        uint32_t endr = rank + __popc(bits);
        endr = __reduce_max_sync(0xffffffffu, v ? endr : 0u);
        const uint32_t total = endr > base ? endr - base : 0u;
        if (bits) {
            uint32_t col[16];
            decode16(a, b, d, col);
            uint32_t r = rank - base;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if ((bits >> j) & 1u) {
                    s_col[warp][r] = col[j];
                    s_off[warp][r] = (uint16_t)(lane * 16 + j);
                    ++r;
                }
        }
        __syncwarp();
        for (uint32_t i0 = 0; i0 < total; i0 += 128) {
            uint32_t c[4], n[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + u * 32 + lane;
                c[u] = i < total ? s_col[warp][i] : 0u;
                n[u] = i < total ? __ldg(cnt8 + c[u]) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t i = i0 + u * 32 + lane;
                if (i < total) {
                    colors[base + i] = c[u];
                    counts[base + i] = n[u] == 255u ? __ldg(cnt32 + c[u]) : n[u];
                    if (first) first[base + i] = (uint32_t)(g0 * 16 + s_off[warp][i]);
                }
            }
        }
        __syncwarp();
        a = na;
        b = nb;
        d = nd;
    }
}

// one thread per pixel from p0 on: the tail of hist_emit16, or the whole image
// when it is not 16-byte aligned
__global__ void __launch_bounds__(kThreads) hist_emit(const uint8_t *__restrict__ rgb, uint64_t p0, uint64_t P,
                                                     const uint32_t *__restrict__ bitmap,
                                                     const uint32_t *__restrict__ wpref,
                                                     const uint8_t *__restrict__ cnt8,
                                                     const uint32_t *__restrict__ cnt32,
                                                     uint32_t *__restrict__ colors, uint32_t *__restrict__ counts,
                                                     uint32_t *__restrict__ first) {
    pdl_wait();
    pdl_trigger();
    for (uint64_t p = p0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P;
         p += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = p >> 5;
        const uint32_t bits = __ldg(bitmap + w);
        const uint32_t b = (uint32_t)(p & 31);
        if (!((bits >> b) & 1u)) continue;
        const uint32_t rank = __ldg(wpref + w) + __popc(bits & ((1u << b) - 1u));
        const uint32_t c = ((uint32_t)__ldcs(rgb + 3 * p) << 16) | ((uint32_t)__ldcs(rgb + 3 * p + 1) << 8) |
                           __ldcs(rgb + 3 * p + 2);
        colors[rank] = c;
        counts[rank] = count_of(cnt8, cnt32, c);
        if (first) first[rank] = (uint32_t)p;
    }
}


// ---- large images: colour-bucketed partition, aggregation in shared memory
//
// Colour c splits into bucket c >> 14 (1024 buckets) and slot c & 0x3FFF
// (16384 colours, whose count and minimum pixel index fit one block's shared
// memory). The image is cut into G chunks of at most 2^18 pixels, so a pixel
// travels as one u32 entry (chunk offset << 14 | slot):
//   part_count    per chunk: pixels per bucket (shared-memory counters)
//   seg_scan      per bucket: chunk segment offsets; bucket sizes
//   bucket_scan   bucket starts; buckets ordered by size (largest first)
//   part_scatter  per chunk, 8192-pixel tiles: counting sort by bucket in
//                 shared memory, then runs of consecutive entries per bucket
//   bucket_agg    one block per bucket: count (add) and first pixel (min) per
//                 colour with shared-memory atomics; dense per-colour counts
//                 out, and the first pixel of every present colour marked in
//                 the P-bit first-occurrence bitmap
// then the scan and the pixel-order emit as before. Every pixel costs shared-
// memory atomics and streamed bytes; only distinct colours touch L2 randomly.
constexpr int kBucketBits = 10;
constexpr int kSlotBits = 14;
constexpr int kBuckets = 1 << kBucketBits;
constexpr int kSlots = 1 << kSlotBits;
constexpr int kChunkBits = 18; // offset within a chunk: 18 bits + slot: 14 bits
constexpr int kPartThreads = 1024;
constexpr int kTilePix = kPartThreads * 16; // 16384 pixels per scatter tile: runs of ~16 entries per bucket
constexpr int kAggThreads = 1024;

__device__ __forceinline__ void decode_group(const uint8_t *rgb, uint64_t p0, int n, bool vec, uint32_t *col) {
    if (vec && n == 16) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rgb + p0 * 3);
        decode16(ld_stream(src), ld_stream(src + 1), ld_stream(src + 2), col);
    } else {
        for (int j = 0; j < 16; ++j) {
            const uint64_t p = p0 + j;
            col[j] = j < n ? ((uint32_t)rgb[3 * p] << 16) | ((uint32_t)rgb[3 * p + 1] << 8) | rgb[3 * p + 2] : 0u;
        }
    }
}

__global__ void __launch_bounds__(kPartThreads) part_count(const uint8_t *__restrict__ rgb, uint64_t P, uint64_t chunk,
                                                           int vec, uint32_t *__restrict__ gcnt, int G) {
    pdl_trigger();
    __shared__ uint32_t s_cnt[kBuckets];
    for (int b = threadIdx.x; b < kBuckets; b += kPartThreads) s_cnt[b] = 0;
    __syncthreads();
    const uint64_t base = (uint64_t)blockIdx.x * chunk;
    const uint64_t end = base + chunk < P ? base + chunk : P;
    for (uint64_t p0 = base + 16ull * threadIdx.x; p0 < end; p0 += 16ull * kPartThreads) {
        const int n = end - p0 < 16 ? (int)(end - p0) : 16;
        uint32_t col[16];
        decode_group(rgb, p0, n, vec, col);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < n) atomicAdd(&s_cnt[col[j] >> kSlotBits], 1u);
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kBuckets; b += kPartThreads) gcnt[(size_t)b * G + blockIdx.x] = s_cnt[b];
}

// per bucket: exclusive scan of its G chunk counts (in place) and the bucket size
__global__ void __launch_bounds__(256) seg_scan(uint32_t *__restrict__ gcnt, int G, uint32_t *__restrict__ bsize) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint32_t s_w[8];
    __shared__ uint32_t s_carry;
    uint32_t *row = gcnt + (size_t)blockIdx.x * G;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int base = 0; base < G; base += 256) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < G ? row[i] : 0u;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= (unsigned)o) x += t;
        }
        if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = x;
        __syncthreads();
        uint32_t woff = 0;
        for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) woff += s_w[w];
        const uint32_t carry = s_carry;
        if (i < G) row[i] = carry + woff + x - v;
        __syncthreads();
        if (threadIdx.x == 255) s_carry = carry + woff + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) bsize[blockIdx.x] = s_carry;
}

// bucket starts (exclusive scan of the sizes) and the aggregation order:
// buckets by decreasing size, so the largest start first (one block)
__global__ void __launch_bounds__(kBuckets) bucket_scan(const uint32_t *__restrict__ bsize,
                                                        uint32_t *__restrict__ bstart, uint32_t *__restrict__ border) {
    pdl_wait();
    pdl_trigger();
    __shared__ uint32_t s_x[kBuckets];
    __shared__ unsigned long long s_k[kBuckets];
    const int t = threadIdx.x;
    const uint32_t v = bsize[t];
    s_x[t] = v;
    s_k[t] = ((unsigned long long)(~v) << 32) | (uint32_t)t; // ascending key = descending size
    __syncthreads();
    for (int o = 1; o < kBuckets; o <<= 1) {
        const uint32_t add = t >= o ? s_x[t - o] : 0u;
        __syncthreads();
        s_x[t] += add;
        __syncthreads();
    }
    bstart[t] = s_x[t] - v;
    for (int size = 2; size <= kBuckets; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int o = t ^ stride;
            if (o > t) {
                const bool up = (t & size) == 0;
                const unsigned long long a = s_k[t], b = s_k[o];
                if ((a > b) == up) {
                    s_k[t] = b;
                    s_k[o] = a;
                }
            }
            __syncthreads();
        }
    border[t] = (uint32_t)(s_k[t] & 0xFFFFFFFFu);
}

constexpr size_t kScatterSmem = sizeof(uint32_t) * (3 * kBuckets + kPartThreads / 32 + kTilePix) +
                                sizeof(uint16_t) * kTilePix;
__global__ void __launch_bounds__(kPartThreads) part_scatter(const uint8_t *__restrict__ rgb, uint64_t P,
                                                             uint64_t chunk, int vec,
                                                             const uint32_t *__restrict__ gcnt, int G,
                                                             const uint32_t *__restrict__ bstart,
                                                             uint32_t *__restrict__ ent) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ uint32_t s_part[];
    uint32_t *s_cur = s_part;             // next global slot of this chunk's segment per bucket
    uint32_t *s_tc = s_cur + kBuckets;    // tile: entries per bucket
    uint32_t *s_ts = s_tc + kBuckets;     // tile: exclusive start per bucket
    uint32_t *s_w = s_ts + kBuckets;      // scan: warp totals
    uint32_t *s_e = s_w + kPartThreads / 32; // tile entries sorted by bucket
    uint16_t *s_b = reinterpret_cast<uint16_t *>(s_e + kTilePix); // their buckets
    for (int b = threadIdx.x; b < kBuckets; b += kPartThreads)
        s_cur[b] = bstart[b] + gcnt[(size_t)b * G + blockIdx.x];
    const uint64_t base = (uint64_t)blockIdx.x * chunk;
    const uint64_t end = base + chunk < P ? base + chunk : P;
    // the next tile's 48 bytes per thread are loaded while this tile is sorted
    uint4 nx[3] = {};
    auto prefetch = [&](uint64_t t) {
        const uint64_t q = t + 16ull * threadIdx.x;
        if (vec && q + 16 <= end) {
            const uint4 *src = reinterpret_cast<const uint4 *>(rgb + q * 3);
            nx[0] = ld_stream(src);
            nx[1] = ld_stream(src + 1);
            nx[2] = ld_stream(src + 2);
        }
    };
    if (base < end) prefetch(base);
    for (uint64_t t0 = base; t0 < end; t0 += kTilePix) {
        for (int b = threadIdx.x; b < kBuckets; b += kPartThreads) s_tc[b] = 0;
        __syncthreads();
        const uint64_t p0 = t0 + 16ull * threadIdx.x;
        const int n = p0 < end ? (end - p0 < 16 ? (int)(end - p0) : 16) : 0;
        uint32_t col[16], rank[16];
        if (vec && n == 16) decode16(nx[0], nx[1], nx[2], col);
        else decode_group(rgb, p0, n, false, col);
        if (t0 + kTilePix < end) prefetch(t0 + kTilePix);
#pragma unroll
        for (int j = 0; j < 16; ++j)
            rank[j] = j < n ? atomicAdd(&s_tc[col[j] >> kSlotBits], 1u) : 0u;
        __syncthreads();
        // exclusive scan of the 1024 tile counts: one per thread
        static_assert(kPartThreads == kBuckets, "one bucket per thread in the tile scan");
        const uint32_t a0 = s_tc[threadIdx.x];
        uint32_t x = a0;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
            if ((threadIdx.x & 31) >= (unsigned)o) x += t;
        }
        if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = x;
        __syncthreads();
        uint32_t woff = 0;
        for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) woff += s_w[w];
        s_ts[threadIdx.x] = woff + x - a0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < n) {
                const uint32_t b = col[j] >> kSlotBits;
                const uint32_t pos = s_ts[b] + rank[j];
                s_e[pos] = ((uint32_t)(p0 + j - base) << kSlotBits) | (col[j] & (kSlots - 1));
                s_b[pos] = (uint16_t)b;
            }
        __syncthreads();
        // runs of consecutive entries per bucket go to consecutive global slots
        const int tn = end - t0 < (uint64_t)kTilePix ? (int)(end - t0) : kTilePix;
        for (int j = threadIdx.x; j < tn; j += kPartThreads) {
            const uint32_t b = s_b[j];
            ent[s_cur[b] + (j - s_ts[b])] = s_e[j];
        }
        __syncthreads();
        for (int b = threadIdx.x; b < kBuckets; b += kPartThreads) s_cur[b] += s_tc[b];
        __syncthreads();
    }
}

// one block per bucket (largest first): count and first pixel per colour in
// shared memory. Each warp takes a contiguous slice of the bucket's entries;
// a lane tracks the chunk segment its entry falls in (the segment starts are
// in shared memory, entries only move forward). The minimum is kept on the key
// (chunk << 18 | offset), which orders as the pixel index does (offset < chunk
// size <= 2^18), and decoded to chunk * g + offset at the end.
__global__ void __launch_bounds__(kAggThreads) bucket_agg(const uint32_t *__restrict__ ent,
                                                          const uint32_t *__restrict__ gcnt, int G, uint64_t chunk,
                                                          const uint32_t *__restrict__ bstart,
                                                          const uint32_t *__restrict__ bsize,
                                                          const uint32_t *__restrict__ border,
                                                          uint8_t *__restrict__ cnt8, uint32_t *__restrict__ cnt32,
                                                          uint32_t *__restrict__ bitmap) {
    pdl_wait();
    pdl_trigger();
    extern __shared__ __align__(16) uint32_t s_tab[]; // kSlots counts | kSlots minimum keys | G + 1 segment starts
    uint32_t *s_cnt = s_tab, *s_min = s_tab + kSlots, *s_seg = s_tab + 2 * kSlots;
    const uint32_t b = border[blockIdx.x];
    const uint32_t bs = bstart[b], bn = bsize[b];
    for (int i = threadIdx.x; i < kSlots; i += kAggThreads) {
        s_cnt[i] = 0u;
        s_min[i] = 0xFFFFFFFFu;
    }
    for (int g = threadIdx.x; g < G; g += kAggThreads) s_seg[g] = gcnt[(size_t)b * G + g];
    if (threadIdx.x == 0) s_seg[G] = bn;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kWarps = kAggThreads / 32, U = 8; // U entries per lane in flight
    const uint32_t per = (bn + kWarps - 1) / kWarps;
    const uint32_t w0 = per * warp < bn ? per * warp : bn, w1 = w0 + per < bn ? w0 + per : bn;
    // the segment of entry w0 + lane: first g with s_seg[g + 1] > e
    uint32_t g = 0;
    {
        int lo = 0, hi = G - 1;
        const uint32_t e = w0 + lane;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_seg[mid] <= e) lo = mid;
            else hi = mid - 1;
        }
        g = (uint32_t)lo;
    }
    for (uint32_t e0 = w0;; e0 += 32) { // warp-uniform control flow throughout
        // full batches: no bounds tests. One vote per batch looks for a first
        // row of a single colour (flat regions): that row takes the careful
        // path below, which folds a one-colour row into one update.
        for (; e0 < w1 && w1 - e0 >= 32 * U; e0 += 32 * U) {
            uint32_t x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = __ldcs(ent + bs + e0 + u * 32 + lane);
            const uint32_t x0slot = x[0] & (kSlots - 1);
            if (__all_sync(0xffffffffu, x0slot == __shfl_sync(0xffffffffu, x0slot, 0))) break;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = e0 + u * 32 + lane;
                while (s_seg[g + 1] <= e) ++g;
                const uint32_t slot = x[u] & (kSlots - 1);
                const uint32_t key = (g << kChunkBits) | (x[u] >> kSlotBits);
                atomicAdd(&s_cnt[slot], 1u);
                if (key < s_min[slot]) atomicMin(&s_min[slot], key); // most later occurrences skip the atomic
            }
        }
        if (e0 >= w1) break;
        const uint32_t e = e0 + lane;
        const bool v = e < w1;
        const uint32_t xe = v ? __ldcs(ent + bs + e) : 0u;
        if (v)
            while (s_seg[g + 1] <= e) ++g;
        const uint32_t slot = xe & (kSlots - 1);
        const uint32_t key = (g << kChunkBits) | (xe >> kSlotBits);
        const uint32_t act = __ballot_sync(0xffffffffu, v);
        const int lead = __ffs(act) - 1;
        const uint32_t s_first = __shfl_sync(0xffffffffu, slot, lead);
        if (__all_sync(0xffffffffu, !v || slot == s_first)) {
            // one colour across the warp: one update per warp
            const uint32_t km = __reduce_min_sync(0xffffffffu, v ? key : 0xFFFFFFFFu);
            if (lane == lead) {
                atomicAdd(&s_cnt[slot], (uint32_t)__popc(act));
                atomicMin(&s_min[slot], km);
            }
        } else if (v) {
            atomicAdd(&s_cnt[slot], 1u);
            if (key < s_min[slot]) atomicMin(&s_min[slot], key);
        }
    }
    __syncthreads();
    // four slots per thread: one packed u8x4 store; the u32 side table only
    // where a count saturates
    uint32_t *dst8 = reinterpret_cast<uint32_t *>(cnt8 + ((size_t)b << kSlotBits));
    uint32_t *dst32 = cnt32 + ((size_t)b << kSlotBits);
    for (int q = threadIdx.x; q < kSlots / 4; q += kAggThreads) {
        const uint4 c4 = reinterpret_cast<const uint4 *>(s_cnt)[q];
        const uint4 m4 = reinterpret_cast<const uint4 *>(s_min)[q];
        const uint32_t c[4] = {c4.x, c4.y, c4.z, c4.w}, m[4] = {m4.x, m4.y, m4.z, m4.w};
        uint32_t packed = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            packed |= (c[j] < 255u ? c[j] : 255u) << (8 * j);
            if (c[j] >= 255u) dst32[4 * q + j] = c[j];
            if (c[j]) {
                const uint64_t f = (uint64_t)(m[j] >> kChunkBits) * chunk + (m[j] & ((1u << kChunkBits) - 1u));
                atomicOr(&bitmap[f >> 5], 1u << (f & 31));
            }
        }
        dst8[q] = packed;
    }
}

// block sums of popcounts over kWordsPerBlock words
__global__ void __launch_bounds__(kThreads) scan_blocksum(const uint32_t *__restrict__ bitmap,
                                                          uint64_t words, uint32_t *__restrict__ bsum) {
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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
    pdl_wait();
    pdl_trigger();
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

// large images: the bucketed partition (part_count .. bucket_agg) into the
// first-occurrence bitmap and the per-colour counts
static void histogram_partitioned(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t P, uint32_t *bitmap,
                                  uint8_t *&cnt8, uint32_t *&cnt32) {
    cudaStream_t s = ctx->stream;
    // chunks of at most 2^18 pixels (an entry's offset field), a multiple of 16
    // pixels (48-byte vector loads), about 4 per SM
    uint64_t chunk = (P + (uint64_t)ctx->num_sms * 4 - 1) / ((uint64_t)ctx->num_sms * 4);
    chunk = (chunk + 15) & ~15ull;
    if (chunk > (1ull << kChunkBits)) chunk = 1ull << kChunkBits;
    const int G = (int)((P + chunk - 1) / chunk);
    const int vec = (reinterpret_cast<uintptr_t>(rgb_d) & 15) == 0;
    uint32_t *gcnt = static_cast<uint32_t *>(ctx->pseg.ensure(sizeof(uint32_t) * ((size_t)kBuckets * G + 3 * kBuckets)));
    uint32_t *bsize = gcnt + (size_t)kBuckets * G, *bstart = bsize + kBuckets, *border = bstart + kBuckets;
    uint32_t *ent = static_cast<uint32_t *>(ctx->pent.ensure(sizeof(uint32_t) * P));
    // per-colour counts: u32 side table (only saturated entries are written or read) | u8 table
    cnt32 = static_cast<uint32_t *>(ctx->pcnt.ensure((sizeof(uint32_t) + sizeof(uint8_t)) << 24));
    cnt8 = reinterpret_cast<uint8_t *>(cnt32 + (1u << 24));
    part_count<<<G, kPartThreads, 0, s>>>(rgb_d, P, chunk, vec, gcnt, G);
    launch_pdl(seg_scan, kBuckets, 256, 0, s, gcnt, G, bsize);
    launch_pdl(bucket_scan, 1, kBuckets, 0, s, bsize, bstart, border);
    CQG_CUDA(ensure_smem((const void *)part_scatter, kScatterSmem));
    launch_pdl(part_scatter, G, kPartThreads, kScatterSmem, s, rgb_d, P, chunk, vec, gcnt, G, bstart, ent);
    const size_t agg_smem = sizeof(uint32_t) * (2 * kSlots + (size_t)G + 1);
    CQG_CUDA(ensure_smem((const void *)bucket_agg, agg_smem));
    launch_pdl(bucket_agg, kBuckets, kAggThreads, agg_smem, s, ent, gcnt, G, chunk, bstart, bsize, border, cnt8, cnt32, bitmap);
    launched(ctx, 5);
}

void histogram_dev(cqg_ctx *ctx, const uint8_t *rgb_d, uint64_t P, uint32_t *colors_d,
                   uint32_t *counts_d, uint32_t *first_d, uint32_t *n_dev) {
    cudaStream_t s = ctx->stream;
    const uint64_t cap = P < (1ull << 24) ? P : (1ull << 24);
    const uint64_t words = (P + 31) / 32;
    const uint32_t nblk = ceil_div(words, kWordsPerBlock);
    uint32_t *bitmap = static_cast<uint32_t *>(ctx->bitmap.ensure(words * 4 + 16));
    uint32_t *wpref = static_cast<uint32_t *>(ctx->wordpref.ensure(words * 4 + 16 + (size_t)nblk * 4));
    uint32_t *bsum = wpref + words + 4;
    const bool large = P >= (1ull << 22);
    if (!large && ctx->tab.cap < (sizeof(uint2) << 24)) {
        ctx->tab.ensure(sizeof(uint2) << 24);
        CQG_CUDA(cudaMemsetAsync(ctx->tab.p, 0, sizeof(uint2) << 24, s));
    }
    uint32_t *list = large ? nullptr : static_cast<uint32_t *>(ctx->list.ensure(cap * 4));

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
    // emit + reset per listed colour. Large images: the bucketed partition,
    // emit in pixel order.
    uint2 *tab = ctx->tab.as<uint2>();
    uint8_t *cnt8 = nullptr;
    uint32_t *cnt32 = nullptr;
    if (!large) {
        hist_count_fused<<<grid, kThreads, 0, s>>>(rgb_d, P, tab, list, n_dev, aligned);
        launch_pdl(hist_mark_fused, lgrid, kThreads, 0, s, list, n_dev, tab, bitmap);
    } else {
        histogram_partitioned(ctx, rgb_d, P, bitmap, cnt8, cnt32);
    }
    launch_pdl(scan_blocksum, nblk, kThreads, 0, s, bitmap, words, bsum);
    launch_pdl(scan_blocks, 1, 1024, 0, s, bsum, nblk, large ? n_dev : nullptr);
    launch_pdl(scan_words, nblk, kThreads, 0, s, bitmap, words, bsum, wpref);
    if (!large) {
        launch_pdl(hist_emit_fused, lgrid, kThreads, 0, s, list, n_dev, tab, bitmap, wpref, colors_d, counts_d, first_d);
    } else {
        const unsigned egrid = (unsigned)ctx->num_sms * 8;
        const uint64_t groups = aligned ? P / 16 : 0;
        if (groups)
            launch_pdl(hist_emit16, egrid, kThreads, 0, s, rgb_d, groups, bitmap, wpref, (const uint8_t *)cnt8,
                       (const uint32_t *)cnt32, colors_d, counts_d, first_d);
        if (groups * 16 < P) {
            unsigned tgrid = ceil_div(P - groups * 16, kThreads);
            if (tgrid > egrid) tgrid = egrid;
            launch_pdl(hist_emit, tgrid, kThreads, 0, s, rgb_d, groups * 16, P, bitmap, wpref, (const uint8_t *)cnt8,
                       (const uint32_t *)cnt32, colors_d, counts_d, first_d);
        }
    }
    prof_end(ctx, CQG_PROF_HIST, pb, 3.0 * (double)P); // + 8 N' added by the caller
    CQG_CUDA(cudaGetLastError());
    launched(ctx, large ? 3 + (aligned && P >= 16) + ((aligned ? P / 16 * 16 : 0) < P) : 6);
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
