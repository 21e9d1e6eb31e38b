// gridsync_micro.cu -- grid barrier latency on B200 (not part of the product).
// A cooperative grid of 2 x SMs blocks x 256 threads runs R barriers:
//   cg    cooperative_groups grid.sync()
//   flat  one counter: thread 0 red.release.gpu.add, spin on ld.acquire.gpu
//         until the count reaches the generation target
//   tree  blocks of one SM pair up: the last of every group of 8 blocks to
//         arrive adds to the top counter (fewer arrivals on one L2 line)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_micro tools/gridsync_micro.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned long long *p, unsigned long long v) {
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_acqrel(unsigned long long *p, unsigned long long v) {
    unsigned long long o;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;" : "=l"(o) : "l"(p), "l"(v) : "memory");
    return o;
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) kern(int R, unsigned long long *ctr, unsigned long long *out) {
    cg::grid_group grid = cg::this_grid();
    const unsigned long long G = gridDim.x;
    unsigned long long acc = 0;
    for (int r = 1; r <= R; ++r) {
        acc += clock64() & 1; // a little per-round work
        if (MODE == 0) {
            grid.sync();
        } else if (MODE == 1) {
            __syncthreads();
            if (threadIdx.x == 0) {
                red_rel(ctr, 1ull);
                while (ld_acq(ctr) < G * (unsigned long long)r) { }
            }
            __syncthreads();
        } else {
            // two levels: groups of 8 blocks, the last arriver of a group forwards
            __syncthreads();
            if (threadIdx.x == 0) {
                const unsigned grp = blockIdx.x >> 3, ngrp = (gridDim.x + 7) >> 3;
                const unsigned gsz = min(8u, gridDim.x - grp * 8);
                const unsigned long long o = atom_add_acqrel(ctr + 16 + grp * 16, 1ull);
                if (o + 1 == (unsigned long long)gsz * r) red_rel(ctr, 1ull);
                while (ld_acq(ctr) < (unsigned long long)ngrp * r) { }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int G = 2 * sms, R = 2000;
    unsigned long long *ctr, *out;
    cudaMalloc(&ctr, 1 << 20);
    cudaMalloc(&out, 8 * G);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char *names[3] = {"cg grid.sync", "flat counter", "two-level (8)"};
    void (*ks[3])(int, unsigned long long *, unsigned long long *) = {kern<0>, kern<1>, kern<2>};
    for (int m = 0; m < 3; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemset(ctr, 0, 1 << 20);
            int Rv = R;
            void *args[] = {&Rv, &ctr, &out};
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)ks[m], G, 256, args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) printf("%-14s %d blocks: %.3f us per barrier\n", names[m], G, ms * 1e3 / R);
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
