// Does tcgen05.mma.kind::tf32 truncate or round its fp32 smem operands? A = 1 + 3 * 2^-12 (0.75 TF32
// ulp above 1), B = 1, K = 32, no hi/lo split (TCG_NO_CONVERT, TCG_ONE_MMA): D = 32 (truncation) or
// 32 * (1 + 2^-10) = 32.03125 (round to nearest).
#define TCG_NO_CONVERT 1
#define TCG_ONE_MMA 1
#include <cstdio>
#include <vector>
#include "../paper_2106_00003_b200/csrc/tc_gemm.cuh"
int main() {
    const int M = 128, N = 128, K = 32;
    std::vector<float> ha(M * K, 1.0f + 3.0f / 4096.0f), hb(N * K, 1.0f);
    float *da, *db, *dd;
    cudaMalloc(&da, M * K * 4); cudaMalloc(&db, N * K * 4); cudaMalloc(&dd, M * N * 4);
    cudaMemcpy(da, ha.data(), M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), N * K * 4, cudaMemcpyHostToDevice);
    tcg::gemm3({da, K, false}, {db, K, false}, M, N, K, 1 << 20, dd, M, M * N, 0);
    cudaDeviceSynchronize();
    float d;
    cudaMemcpy(&d, dd, 4, cudaMemcpyDeviceToHost);
    printf("D = %.6f (trunc 32, rn 32.03125) %s\n", d, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
