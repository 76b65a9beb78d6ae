// Minimal, obviously-correct programs that use the two synchronisation / data-movement mechanisms the
// ring kernels rely on, to show what compute-sanitizer reports for them:
//  (1) racecheck: warp 0 writes shared memory and arrives on an mbarrier; warp 1 waits on the mbarrier
//      (try_wait.parity loop, acquire semantics) and reads it. Correct by the mbarrier's
//      release/acquire ordering.
//  (2) initcheck: a CTA fills shared memory, writes it to global with cp.async.bulk (TMA bulk copy)
//      and waits for completion; a second kernel reads the global buffer. Every byte is written.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/sanitizer_probe tools/sanitizer_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2106_00003_b200/csrc/common.cuh"

__global__ void k_mbar_handoff(float *out) {
    __shared__ float buf[32];
    __shared__ uint64_t bar;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        gk::mbar_init(&bar, 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        buf[lane] = (float)lane;
        gk::mbar_arrive(&bar);  // release: this lane's write happens-before the phase completes
    } else {
        gk::mbar_wait(&bar, 0);  // acquire
        out[lane] = buf[lane];
    }
}

// (3) the ring pattern of the backward kernel's dtheta stage: NW warps write their slice of ring
// buffer bi = g % 2, arrive on rfull[bi]; then every warp waits rfull[bi], reads all slices, and
// arrives on rempty[bi]; group g + 2 reuses buffer bi after waiting rempty[bi] (pre-armed once, so the
// first use of each buffer passes). Multi-phase reuse of the same two mbarriers, as in k_ring.
__global__ void k_mbar_ring(float *out, int groups) {
    constexpr int NW = 8, NG = 2;
    __shared__ float ring[NG][NW][32];
    __shared__ uint64_t rfull[NG], rempty[NG];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NG; i++) { gk::mbar_init(&rfull[i], NW); gk::mbar_init(&rempty[i], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (lane == 0) for (int i = 0; i < NG; i++) gk::mbar_arrive(&rempty[i]);
    float acc = 0.f;
    for (int g = 0; g < groups; g++) {
        const int bi = g % NG;
        gk::mbar_wait(&rempty[bi], (uint32_t)((g / NG) & 1));
        __syncwarp();
        ring[bi][warp][lane] = (float)(g + warp + lane);
        __syncwarp();
        if (lane == 0) gk::mbar_arrive(&rfull[bi]);
        gk::mbar_wait(&rfull[bi], (uint32_t)((g / NG) & 1));
        for (int w = 0; w < NW; w++) acc += ring[bi][w][lane];
        __syncwarp();
        if (lane == 0) gk::mbar_arrive(&rempty[bi]);
    }
    out[threadIdx.x] = acc;
}

__global__ void k_bulk_store(float *dst) {
    __shared__ __align__(128) float buf[256];
    buf[threadIdx.x] = (float)threadIdx.x;
    gk::fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
        gk::bulk_s2g_store(dst, buf, 256 * 4);
        gk::bulk_commit();
        gk::bulk_wait_all();
    }
}

__global__ void k_read(const float *src, float *out) { out[threadIdx.x] = src[threadIdx.x] + 1.f; }

int main() {
    float *a, *b, *o;
    cudaMalloc(&a, 256 * 4); cudaMalloc(&b, 256 * 4); cudaMalloc(&o, 256 * 4);
    k_mbar_handoff<<<1, 64>>>(o);
    k_mbar_ring<<<1, 256>>>(a, 10);
    k_bulk_store<<<1, 256>>>(b);
    k_read<<<1, 256>>>(b, o);
    cudaError_t e = cudaDeviceSynchronize();
    float h[256];
    cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    printf("probe done: %s, out[5] = %g (expect 6)\n", cudaGetErrorString(e), h[5]);
    return 0;
}
