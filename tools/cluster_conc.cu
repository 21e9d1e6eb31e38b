// How many 16-CTA clusters run side by side on a B200? (design tool)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_conc tools/cluster_conc.cu && /tmp/cluster_conc
// A spinning cluster kernel (cluster size C, T threads, S bytes of dynamic shared memory) is launched on
// n streams at once; wall time of n launches / time of one = how many were serialised.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void spin(long long cycles, int *sink) {
    extern __shared__ int sm[];
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
    if (sink && threadIdx.x == 0 && cycles < 0) sink[0] = sm[0];
    cl.sync();
}

static float run(int n, int C, int T, size_t S, long long cycles) {
    cudaStream_t st[32];
    for (int i = 0; i < n; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
    cudaFuncSetAttribute(spin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(T);
    cfg.dynamicSmemBytes = S;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int maxc = 0;
    cudaOccupancyMaxActiveClusters(&maxc, spin, &cfg);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        for (int i = 0; i < n; ++i) {
            cudaStreamWaitEvent(st[i], e0, 0);
            cfg.stream = st[i];
            cudaLaunchKernelEx(&cfg, spin, cycles, (int *)nullptr);
        }
        cudaDeviceSynchronize();
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    printf("C=%2d T=%4d smem=%6zu: max active clusters (occupancy API) %2d; %2d streams: %.3f ms\n", C, T, S, maxc, n,
           best);
    for (int i = 0; i < n; ++i) cudaStreamDestroy(st[i]);
    return best;
}

int main() {
    const long long cycles = 1000000; // ~0.5 ms
    for (int C : {16, 8}) {
        for (size_t S : {(size_t)0, (size_t)150 * 1024}) {
            for (int T : {896, 512}) {
                for (int n : {1, 2, 4, 8, 16}) run(n, C, T, S, cycles);
            }
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
