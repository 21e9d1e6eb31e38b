// sweep_variants.cu -- microbenchmark of the Lloyd sweep inner loop on B200
// (not part of the product). Measures distances/s for variants of the
// per-(point, centre) work to locate the pipe limit:
//   V0  product loop: point pairs, FADD2 + 3 FFMA2 (broadcast centre scalar),
//       exact best/second tracking (5 min/max per 2 candidates), group index
//   V1  V0 with best-only tracking (3-input min), no second-best
//   V2  FP only (sum of distances, no tracking)  -> FP pipe limit
//   V3  V0 with 4 points per thread (higher occupancy)
//   V4  group-minimum tracking: 3-input min chain per 8-centre group, then
//       (best, second) over group minima; the winning group's own second value
//       comes from the index-recovery recompute (not timed here: per point)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sweep_variants tools/sweep_variants.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void track_pair(float2 v, float &b1, float &b2) {
    const float lo = fminf(v.x, v.y), hi = fmaxf(v.x, v.y);
    b2 = fminf(fminf(b2, hi), fmaxf(b1, lo));
    b1 = fminf(b1, lo);
}

template <int VAR, int PPT>
__global__ void __launch_bounds__(256, 2) kern(const unsigned *colors, int n, const float *fc, int Kp, float *out) {
    constexpr int PP = PPT / 2;
    extern __shared__ __align__(16) float sm[];
    for (int i = threadIdx.x; i < 4 * Kp; i += blockDim.x) sm[i] = fc[i];
    __syncthreads();
    const float *m2r = sm, *m2g = sm + Kp, *m2b = sm + 2 * Kp, *cc = sm + 3 * Kp;
    const int tile = 256 * PPT;
    for (int base = blockIdx.x * tile; base < n; base += gridDim.x * tile) {
        float2 xr2[PP], xg2[PP], xb2[PP], xx2[PP];
        float b1[PPT], b2[PPT];
        int g1[PPT];
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const int idx = base + threadIdx.x + i * 256;
            const unsigned c = idx < n ? colors[idx] : 0u;
            float r = (float)((c >> 16) & 255u), g = (float)((c >> 8) & 255u), b = (float)(c & 255u);
            float xx = r * r + g * g + b * b;
            asm volatile("" : "+f"(r), "+f"(g), "+f"(b), "+f"(xx));
            if (i & 1) { xr2[i / 2].y = r; xg2[i / 2].y = g; xb2[i / 2].y = b; xx2[i / 2].y = xx; }
            else { xr2[i / 2].x = r; xg2[i / 2].x = g; xb2[i / 2].x = b; xx2[i / 2].x = xx; }
            b1[i] = 3e38f;
            b2[i] = 3e38f;
            g1[i] = 0;
        }
        for (int j = 0; j < Kp; j += 8) {
            float before[PPT], gm[PPT];
#pragma unroll
            for (int i = 0; i < PPT; ++i) before[i] = b1[i], gm[i] = 3e38f;
#pragma unroll
            for (int q = 0; q < 8; q += 4) {
                const float4 r4 = *reinterpret_cast<const float4 *>(m2r + j + q);
                const float4 g4 = *reinterpret_cast<const float4 *>(m2g + j + q);
                const float4 b4 = *reinterpret_cast<const float4 *>(m2b + j + q);
                const float4 c4 = *reinterpret_cast<const float4 *>(cc + j + q);
#pragma unroll
                for (int p = 0; p < PP; ++p) {
                    float2 A0 = __fadd2_rn(xx2[p], make_float2(c4.x, c4.x));
                    A0 = __ffma2_rn(xr2[p], make_float2(r4.x, r4.x), A0);
                    A0 = __ffma2_rn(xg2[p], make_float2(g4.x, g4.x), A0);
                    A0 = __ffma2_rn(xb2[p], make_float2(b4.x, b4.x), A0);
                    float2 A1 = __fadd2_rn(xx2[p], make_float2(c4.y, c4.y));
                    A1 = __ffma2_rn(xr2[p], make_float2(r4.y, r4.y), A1);
                    A1 = __ffma2_rn(xg2[p], make_float2(g4.y, g4.y), A1);
                    A1 = __ffma2_rn(xb2[p], make_float2(b4.y, b4.y), A1);
                    float2 A2 = __fadd2_rn(xx2[p], make_float2(c4.z, c4.z));
                    A2 = __ffma2_rn(xr2[p], make_float2(r4.z, r4.z), A2);
                    A2 = __ffma2_rn(xg2[p], make_float2(g4.z, g4.z), A2);
                    A2 = __ffma2_rn(xb2[p], make_float2(b4.z, b4.z), A2);
                    float2 A3 = __fadd2_rn(xx2[p], make_float2(c4.w, c4.w));
                    A3 = __ffma2_rn(xr2[p], make_float2(r4.w, r4.w), A3);
                    A3 = __ffma2_rn(xg2[p], make_float2(g4.w, g4.w), A3);
                    A3 = __ffma2_rn(xb2[p], make_float2(b4.w, b4.w), A3);
                    if (VAR == 0 || VAR == 3) {
                        track_pair(make_float2(A0.x, A1.x), b1[2 * p], b2[2 * p]);
                        track_pair(make_float2(A2.x, A3.x), b1[2 * p], b2[2 * p]);
                        track_pair(make_float2(A0.y, A1.y), b1[2 * p + 1], b2[2 * p + 1]);
                        track_pair(make_float2(A2.y, A3.y), b1[2 * p + 1], b2[2 * p + 1]);
                    } else if (VAR == 4) {
                        gm[2 * p] = fminf(fminf(fminf(gm[2 * p], A0.x), A1.x), fminf(A2.x, A3.x));
                        gm[2 * p + 1] = fminf(fminf(fminf(gm[2 * p + 1], A0.y), A1.y), fminf(A2.y, A3.y));
                    } else if (VAR == 1) {
                        b1[2 * p] = fminf(fminf(b1[2 * p], A0.x), A1.x);
                        b1[2 * p] = fminf(fminf(b1[2 * p], A2.x), A3.x);
                        b1[2 * p + 1] = fminf(fminf(b1[2 * p + 1], A0.y), A1.y);
                        b1[2 * p + 1] = fminf(fminf(b1[2 * p + 1], A2.y), A3.y);
                    } else {
                        float2 s = __fadd2_rn(__fadd2_rn(A0, A1), __fadd2_rn(A2, A3));
                        b1[2 * p] += s.x;
                        b1[2 * p + 1] += s.y;
                    }
                }
            }
            if (VAR == 4) {
#pragma unroll
                for (int i = 0; i < PPT; ++i) {
                    const float lo = gm[i];
                    g1[i] = lo < b1[i] ? j : g1[i];
                    b2[i] = fminf(b2[i], fmaxf(b1[i], lo));
                    b1[i] = fminf(b1[i], lo);
                }
            } else if (VAR != 2) {
#pragma unroll
                for (int i = 0; i < PPT; ++i) g1[i] = b1[i] < before[i] ? j : g1[i];
            }
        }
#pragma unroll
        for (int i = 0; i < PPT; ++i) {
            const int idx = base + threadIdx.x + i * 256;
            if (idx < n) out[idx] = b1[i] + b2[i] + (float)g1[i];
        }
    }
}

template <int VAR, int PPT>
double run(const unsigned *d_col, int n, const float *d_fc, int K, float *d_out, int sms) {
    const int Kp = (K + 7) & ~7;
    const size_t smem = 16 * Kp;
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kern<VAR, PPT>, 256, smem));
    const int grid = sms * bps;
    kern<VAR, PPT><<<grid, 256, smem>>>(d_col, n, d_fc, Kp, d_out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 10;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) kern<VAR, PPT><<<grid, 256, smem>>>(d_col, n, d_fc, Kp, d_out);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double dps = (double)n * K * reps / (ms / 1e3);
    printf("V%d PPT=%d bps=%d grid=%d  %.3f ms/launch  %.3e dist/s  %.1f%% of 9.31e12\n", VAR, PPT, bps, grid,
           ms / reps, dps, 100.0 * dps / 9.31e12);
    return dps;
}

int main() {
    const int n = 6295531, K = 256;
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<unsigned> col(n);
    unsigned s = 12345;
    for (auto &c : col) { s = s * 1664525u + 1013904223u; c = s >> 8; }
    std::vector<float> fc(4 * K);
    for (int k = 0; k < K; ++k) {
        s = s * 1664525u + 1013904223u;
        const float r = (s >> 24), g = ((s >> 16) & 255), b = ((s >> 8) & 255);
        fc[k] = -2 * r; fc[K + k] = -2 * g; fc[2 * K + k] = -2 * b; fc[3 * K + k] = r * r + g * g + b * b;
    }
    unsigned *d_col; float *d_fc, *d_out;
    CK(cudaMalloc(&d_col, 4 * n)); CK(cudaMalloc(&d_fc, 16 * K)); CK(cudaMalloc(&d_out, 4 * n));
    CK(cudaMemcpy(d_col, col.data(), 4 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_fc, fc.data(), 16 * K, cudaMemcpyHostToDevice));
    run<0, 8>(d_col, n, d_fc, K, d_out, sms);
    run<1, 8>(d_col, n, d_fc, K, d_out, sms);
    run<2, 8>(d_col, n, d_fc, K, d_out, sms);
    run<3, 4>(d_col, n, d_fc, K, d_out, sms);
    run<0, 2>(d_col, n, d_fc, K, d_out, sms);
    run<4, 8>(d_col, n, d_fc, K, d_out, sms);
    run<4, 4>(d_col, n, d_fc, K, d_out, sms);
    return 0;
}
