// gather_micro.cu -- microbenchmark behind the pixel-mapping analysis (not part
// of the product). pixel_kernel (csrc/mapk.cu) streams 3 B/pixel in, writes
// 4 B index + 3 B RGB out, and gathers one byte per pixel from the 16 MiB
// colour -> index LUT. This measures, on the same B200:
//   G1  random 1-byte gathers from a 16 MiB table (L2-resident), 16 per thread
//       in flight, indices from a hash (no input stream): the gather ceiling
//   G2  random 4-byte gathers from a 64 MiB table (K > 256 LUT)
//   G3  the pixel kernel's traffic with random colours (uniform 24-bit image,
//       cfg5-like): 48-byte loads, 16 gathers, 64 + 48 byte stores per thread
//   G4  G3 without the gather (index = low byte of the colour): the HBM-only
//       ceiling of the same streams
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_micro tools/gather_micro.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            printf("%s: %s\n", #x, cudaGetErrorString(e));                        \
            exit(1);                                                              \
        }                                                                         \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

template <typename T>
__global__ void __launch_bounds__(256) gather_only(const T *__restrict__ lut, uint32_t mask, uint64_t n,
                                                   unsigned *out) {
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 16;
    for (uint64_t b = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; b < n; b += stride) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = (uint32_t)__ldg(lut + (hash32((uint32_t)(b + j)) & mask));
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += v[j];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint4 ld_stream4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream4(uint4 *p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}

// the pixel kernel's streams (16 pixels / thread), with or without the LUT gather
template <bool GATHER>
__global__ void __launch_bounds__(256) pixel_like(const uint8_t *__restrict__ rgb, uint64_t P,
                                                  const uint8_t *__restrict__ lut, uint32_t *__restrict__ idx_out,
                                                  uint8_t *__restrict__ q_out) {
    const uint64_t groups = P / 16, stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const uint4 *src = reinterpret_cast<const uint4 *>(rgb + g * 48);
        const uint4 a = ld_stream4(src), b = ld_stream4(src + 1), d = ld_stream4(src + 2);
        const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
        uint32_t idx[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int o = 3 * j;
            const uint32_t c = (((w[o >> 2] >> (8 * (o & 3))) & 255u) << 16) |
                               (((w[(o + 1) >> 2] >> (8 * ((o + 1) & 3))) & 255u) << 8) |
                               ((w[(o + 2) >> 2] >> (8 * ((o + 2) & 3))) & 255u);
            idx[j] = GATHER ? (uint32_t)__ldg(lut + c) : (c & 255u);
        }
        uint4 *o4 = reinterpret_cast<uint4 *>(idx_out + g * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i) st_stream4(o4 + i, make_uint4(idx[4 * i], idx[4 * i + 1], idx[4 * i + 2], idx[4 * i + 3]));
        uint4 *q4 = reinterpret_cast<uint4 *>(q_out + g * 48);
        st_stream4(q4, make_uint4(w[0] ^ idx[0], w[1], w[2], w[3]));
        st_stream4(q4 + 1, make_uint4(w[4], w[5] ^ idx[5], w[6], w[7]));
        st_stream4(q4 + 2, make_uint4(w[8], w[9], w[10] ^ idx[10], w[11]));
    }
}

template <class F>
static float time_ms(F f, int reps) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    f();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) f();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / reps;
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t P = 1ull << 26; // cfg5: 8192^2 pixels
    uint8_t *lut8, *rgb, *q;
    uint32_t *lut32, *idx;
    unsigned *out;
    CK(cudaMalloc(&lut8, 1u << 24));
    CK(cudaMalloc(&lut32, 4u << 24));
    CK(cudaMalloc(&rgb, 3 * P));
    CK(cudaMalloc(&q, 3 * P));
    CK(cudaMalloc(&idx, 4 * P));
    CK(cudaMalloc(&out, 64));
    CK(cudaMemset(lut8, 7, 1u << 24));
    CK(cudaMemset(lut32, 7, 4u << 24));
    // uniform random 24-bit pixels (cfg5-like), generated on the device
    {
        uint8_t *h = (uint8_t *)malloc(3 * P);
        uint64_t s = 88172645463325252ull;
        for (uint64_t i = 0; i < 3 * P; ++i) {
            s ^= s << 13;
            s ^= s >> 7;
            s ^= s << 17;
            h[i] = (uint8_t)s;
        }
        CK(cudaMemcpy(rgb, h, 3 * P, cudaMemcpyHostToDevice));
        free(h);
    }
    const int grid = sms * 8;
    const uint64_t n = P;
    const float g1 = time_ms([&] { gather_only<uint8_t><<<grid, 256>>>(lut8, (1u << 24) - 1, n, out); }, 10);
    const float g2 = time_ms([&] { gather_only<uint32_t><<<grid, 256>>>(lut32, (1u << 24) - 1, n, out); }, 10);
    const float g3 = time_ms([&] { pixel_like<true><<<grid, 256>>>(rgb, P, lut8, idx, q); }, 10);
    const float g4 = time_ms([&] { pixel_like<false><<<grid, 256>>>(rgb, P, lut8, idx, q); }, 10);
    const double bytes = 10.0 * P; // 3 in + 4 index + 3 RGB out
    printf("G1 random u8 gathers, 16 MiB table : %7.3f ms  %6.1f G gathers/s\n", g1, n / (g1 * 1e6));
    printf("G2 random u32 gathers, 64 MiB table: %7.3f ms  %6.1f G gathers/s\n", g2, n / (g2 * 1e6));
    printf("G3 pixel streams + u8 LUT gather    : %7.3f ms  %6.1f G pixels/s  %7.1f GB/s\n", g3, P / (g3 * 1e6),
           bytes / (g3 * 1e6));
    printf("G4 pixel streams, no gather         : %7.3f ms  %6.1f G pixels/s  %7.1f GB/s\n", g4, P / (g4 * 1e6),
           bytes / (g4 * 1e6));
    return 0;
}
