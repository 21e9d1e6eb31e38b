// Microbenchmark: the walk-row sort of the persistent Lloyd kernel in isolation
// (one 256-thread block sorts 256 (key, index) pairs; clock64 around the sort).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/sort_micro tools/sort_micro.cu
#include <cstdio>
#include <cstdint>

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
            if (other_less == (low == up)) {
                key = ok;
                r = orr;
            }
        }
    }
}

// Warp bitonic (15 stages over 32 lanes) + rank merge: an element's rank is its
// lane plus, for each of the other 7 sorted warp lists, the number of keys
// below it (binary searches interleaved across the lists, branch-free).
template <int NL>
__device__ __forceinline__ int warp_sort_rank(unsigned long long &key, int &r, int t, unsigned long long *s_key,
                                              int *s_idx) {
    const int lane = t & 31, w = t >> 5;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, stride);
            const int orr = __shfl_xor_sync(0xffffffffu, r, stride);
            const bool up = (lane & size) == 0;
            const bool low = (lane & stride) == 0;
            const bool other_less = ok < key || (ok == key && orr < r);
            if (other_less == (low == up)) {
                key = ok;
                r = orr;
            }
        }
    }
    s_key[t] = key;
    s_idx[t] = r;
    __syncthreads();
    int c[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) c[l] = 0;
#pragma unroll
    for (int step = 32; step >= 1; step >>= 1) {
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            const int q = c[l] + step - 1;
            const int qc = q < 32 ? q : 31;
            const unsigned long long lk = s_key[l * 32 + qc];
            const int li = s_idx[l * 32 + qc];
            const bool below = q < 32 && (lk < key || (lk == key && li < r));
            c[l] += below ? step : 0;
        }
    }
    int rank = lane;
#pragma unroll
    for (int l = 0; l < NL; ++l) rank += l == w ? 0 : c[l];
    return rank;
}

__global__ void sort2_kernel(const double *d, unsigned long long *out, long long *cycles, int reps) {
    __shared__ unsigned long long s_key[256];
    __shared__ int s_idx[256];
    __shared__ unsigned long long s_out[256];
    const int t = threadIdx.x;
    unsigned long long key = (unsigned long long)__double_as_longlong(d[t]);
    int r = t;
    __syncthreads();
    long long c0 = clock64();
    for (int i = 0; i < reps; ++i) {
        const int rank = warp_sort_rank<8>(key, r, t, s_key, s_idx);
        s_out[rank] = key;
        __syncthreads();
        key = s_out[t] ^ (unsigned long long)i;
        r = t;
        __syncthreads();
    }
    long long c1 = clock64();
    out[t] = key + r;
    if (t == 0) cycles[blockIdx.x] = (c1 - c0) / reps;
}

__global__ void sort_kernel(const double *d, unsigned long long *out, long long *cycles, int reps) {
    __shared__ unsigned long long s_key[256];
    __shared__ int s_idx[256];
    const int t = threadIdx.x;
    unsigned long long key = (unsigned long long)__double_as_longlong(d[t]);
    int r = t;
    __syncthreads();
    long long c0 = clock64();
    for (int i = 0; i < reps; ++i) {
        bitonic_reg<256>(key, r, t, s_key, s_idx);
        key ^= (unsigned long long)i; // keep the loop honest
    }
    __syncthreads();
    long long c1 = clock64();
    out[t] = key + r;
    if (t == 0) cycles[blockIdx.x] = (c1 - c0) / reps;
}

int main() {
    const int blocks = 296;
    double h[256];
    for (int i = 0; i < 256; ++i) h[i] = (double)((i * 7919) % 256) * 1.5;
    double *d;
    unsigned long long *o;
    long long *c;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 8 * 256);
    cudaMalloc(&c, 8 * blocks);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int b : {1, 148, 296}) {
        sort2_kernel<<<b, 256>>>(d, o, c, 20);
        cudaDeviceSynchronize();
        long long hc2[296];
        cudaMemcpy(hc2, c, 8 * b, cudaMemcpyDeviceToHost);
        long long s2 = 0;
        for (int i = 0; i < b; ++i) s2 += hc2[i];
        printf("blocks %3d: warp sort + rank merge of 256 in %lld cycles (mean)\n", b, s2 / b);
        sort_kernel<<<b, 256>>>(d, o, c, 20);
        cudaDeviceSynchronize();
        long long hc[296];
        cudaMemcpy(hc, c, 8 * b, cudaMemcpyDeviceToHost);
        long long mx = 0, sum = 0;
        for (int i = 0; i < b; ++i) { sum += hc[i]; mx = hc[i] > mx ? hc[i] : mx; }
        printf("blocks %3d: sort of 256 in %lld cycles (mean), %lld (max)\n", b, sum / b, mx);
    }
    return 0;
}
