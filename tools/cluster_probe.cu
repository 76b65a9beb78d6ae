// How many 2- / 4-CTA clusters of one-CTA-per-SM kernels (the backward ring's 256 threads and
// ~225 KB of shared memory) can be co-resident on this GPU (cudaOccupancyMaxActiveClusters), and a
// launch check: G CTAs that each spin ~1 ms finish in ~1 ms only if they all run at once.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_spin(long long cycles, int *smid) {
    extern __shared__ int sm[];
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
    if (threadIdx.x == 0) { unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); smid[blockIdx.x] = s; sm[0] = s; }
}
int main() {
    const size_t smem = 225 * 1024;
    cudaFuncSetAttribute(k_spin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_spin, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int *smid; cudaMalloc(&smid, 4096 * 4);
    for (int cs : {1, 2, 4, 8}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(148 / cs * cs); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
        cfg.attrs = at; cfg.numAttrs = 1;
        int ncl = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void *)k_spin, &cfg);
        printf("cluster %d: max active clusters %d (%d CTAs) %s\n", cs, ncl, ncl * cs, cudaGetErrorString(e));
        for (int g : {ncl * cs, 148 / cs * cs}) {
            if (g <= 0) continue;
            cfg.gridDim = dim3(g);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaLaunchKernelEx(&cfg, k_spin, 2000000LL, smid);
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, k_spin, 2000000LL, smid);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("   grid %3d: %.3f ms (%s)\n", g, ms, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
