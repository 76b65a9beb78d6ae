#define TCG_DEBUG 1
#include <cstdio>
#include <vector>
#include "../paper_2106_00003_b200/csrc/tc_gemm.cuh"
int main() {
    const int M = 128, N = 128, K = 32;
    for (int amn = 0; amn < 2; amn++) {
        std::vector<float> ha(M * K), hb(N * K);
        for (int i = 0; i < M * K; i++) ha[i] = 1.0f + (i % 7);
        for (int i = 0; i < N * K; i++) hb[i] = 1.0f;
        float *da, *db, *dd;
        cudaMalloc(&da, M * K * 4); cudaMalloc(&db, N * K * 4); cudaMalloc(&dd, M * N * 4);
        cudaMemcpy(da, ha.data(), M * K * 4, cudaMemcpyHostToDevice);
        cudaMemcpy(db, hb.data(), N * K * 4, cudaMemcpyHostToDevice);
        cudaMemset(dd, 0xFF, M * N * 4);
        cudaError_t e = tcg::gemm3({da, amn ? M : K, (bool)amn}, {db, K, false}, M, N, K, 1 << 20, dd, M, M * N, 0);
        cudaError_t e2 = cudaDeviceSynchronize();
        std::vector<float> hd(M * N);
        cudaMemcpy(hd.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
        // expected D[m][n] = sum_k A(m,k) * 1
        double ref0 = 0;
        for (int k = 0; k < K; k++) ref0 += amn ? ha[k * M + 0] : ha[0 * K + k];
        printf("amn=%d %s %s D[0][0]=%g (ref %g) D[1][0]=%g D[0][1]=%g\n", amn, cudaGetErrorString(e), cudaGetErrorString(e2),
               hd[0], ref0, hd[1], hd[M]);
    }
    return 0;
}
