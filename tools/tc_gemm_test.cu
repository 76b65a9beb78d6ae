// Standalone check + timing of the hand-written tcgen05 3xTF32 GEMM (csrc/tc_gemm.cuh):
// every operand-major combination against an fp64 host reference on a ragged size, then timings
// at the GEMM-path shapes of C3 (n = 1024, m = 65536).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_gemm_test tools/tc_gemm_test.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2106_00003_b200/csrc/tc_gemm.cuh"

static float frand(uint64_t &s) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    return ((s >> 40) & 0xFFFFFF) / 8388608.0f - 1.0f;
}

// host reference of D[m][n] = sum_k A(m,k) B(n,k)
static double check(bool amn, bool bmn, int M, int N, int K, int kchunk) {
    int64_t lda = amn ? ((M + 3) / 4 * 4 + 4) : ((K + 3) / 4 * 4 + 8);
    int64_t ldb = bmn ? ((N + 3) / 4 * 4 + 4) : ((K + 3) / 4 * 4);
    size_t na = (size_t)lda * (amn ? K : M), nb = (size_t)ldb * (bmn ? K : N);
    std::vector<float> ha(na), hb(nb);
    uint64_t s = 42;
    for (auto &x : ha) x = frand(s);
    for (auto &x : hb) x = frand(s);
    auto A = [&](int m, int k) { return (double)(amn ? ha[(size_t)k * lda + m] : ha[(size_t)m * lda + k]); };
    auto B = [&](int n, int k) { return (double)(bmn ? hb[(size_t)k * ldb + n] : hb[(size_t)n * ldb + k]); };
    float *da, *db, *dd;
    int nz = (K + kchunk - 1) / kchunk;
    int64_t ldo = M + 5;
    size_t zs = (size_t)ldo * N;
    cudaMalloc(&da, na * 4); cudaMalloc(&db, nb * 4); cudaMalloc(&dd, zs * nz * 4);
    cudaMemcpy(da, ha.data(), na * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(db, hb.data(), nb * 4, cudaMemcpyHostToDevice);
    cudaMemset(dd, 0, zs * nz * 4);
    cudaError_t e = tcg::gemm3({da, lda, amn}, {db, ldb, bmn}, M, N, K, kchunk, dd, ldo, zs, 0);
    cudaError_t e2 = cudaDeviceSynchronize();
    std::vector<float> hd(zs * nz);
    cudaMemcpy(hd.data(), dd, zs * nz * 4, cudaMemcpyDeviceToHost);
    double num = 0, den = 0, emax = 0;
    for (int m = 0; m < M; m++)
        for (int n = 0; n < N; n++) {
            double ref = 0, got = 0;
            for (int k = 0; k < K; k++) ref += A(m, k) * B(n, k);
            for (int z = 0; z < nz; z++) got += hd[z * zs + (size_t)n * ldo + m];
            num += (got - ref) * (got - ref);
            den += ref * ref;
            emax = fmax(emax, fabs(got - ref));
        }
    printf("AMN=%d BMN=%d M=%d N=%d K=%d kchunk=%d: launch=%s sync=%s rel=%.3e maxabs=%.3e\n", amn, bmn, M, N, K,
           kchunk, cudaGetErrorString(e), cudaGetErrorString(e2), sqrt(num / den), emax);
    cudaFree(da); cudaFree(db); cudaFree(dd);
    return sqrt(num / den);
}

static double timeit(const char *name, bool amn, bool bmn, int M, int N, int K, int kchunk) {
    int64_t lda = amn ? M : K, ldb = bmn ? N : K;
    size_t na = (size_t)lda * (amn ? K : M), nb = (size_t)ldb * (bmn ? K : N);
    float *da, *db, *dd;
    int nz = (K + kchunk - 1) / kchunk;
    cudaMalloc(&da, na * 4); cudaMalloc(&db, nb * 4); cudaMalloc(&dd, (size_t)M * N * nz * 4);
    cudaMemset(da, 0, na * 4); cudaMemset(db, 0, nb * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    tcg::gemm3({da, lda, amn}, {db, ldb, bmn}, M, N, K, kchunk, dd, M, (int64_t)M * N, 0);
    cudaDeviceSynchronize();
    const int reps = 10;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; r++) tcg::gemm3({da, lda, amn}, {db, ldb, bmn}, M, N, K, kchunk, dd, M, (int64_t)M * N, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    double fl = 3.0 * 2.0 * M * N * (double)K;
    printf("%-34s M=%6d N=%5d K=%6d: %.3f ms  %.1f TF/s (3xTF32: %.1f TF/s of TF32 MMA)  %s\n", name, M, N, K, ms,
           fl / 3 / ms / 1e9, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(da); cudaFree(db); cudaFree(dd);
    return ms;
}

int main(int argc, char **argv) {
    double worst = 0;
    for (int amn = 0; amn < 2; amn++)
        for (int bmn = 0; bmn < 2; bmn++) {
            worst = fmax(worst, check(amn, bmn, 200, 150, 100, 1 << 20));
            worst = fmax(worst, check(amn, bmn, 128, 128, 32, 1 << 20));
            worst = fmax(worst, check(amn, bmn, 300, 260, 1000, 256));
        }
    printf("worst rel %.3e\n", worst);
    timeit("Y^T = X^T U^T   (A MN, B K)", true, false, 65536, 1024, 1024, 1 << 20);
    timeit("dX^T = dY^T U   (A MN, B MN)", true, true, 65536, 1024, 1024, 1 << 20);
    timeit("M^T = Y dY^T    (A K, B K, split)", false, false, 1024, 1024, 65536, 2048);
    timeit("Gam^T = U^T M^T (A MN, B K)", true, false, 1024, 1024, 1024, 1 << 20);
    // The north_star's k-round dense-tile family at C3 (n = 1024, m = 65536): k consecutive blocks of
    // the circle method compose into a matrix that is banded in slot coordinates (every round moves a
    // value at most one slot, so a 128-row output tile depends on a window of w = 128 + 2 (2k + 2) input
    // rows). The forward is then ceil(1023 / k) GEMMs of the shape Y^T (m x n) over K = w each (the
    // k = 1023 member is the dense U: one GEMM over K = n). Time the GEMM at each window; the build of
    // the band matrices (k rounds of the ring on identity columns, ~ one U-build) comes on top.
    printf("k-round banded-tile forward (C3), 3xTF32 GEMMs over the band window:\n");
    for (int k : {16, 32, 64, 128, 256, 1023}) {
        int w = k >= 1023 ? 1024 : 128 + 2 * (2 * k + 2);
        if (w > 1024) w = 1024;
        const int groups = (1023 + k - 1) / k;
        char nm[64];
        snprintf(nm, sizeof nm, "band k=%d (window %d)", k, w);
        double ms = timeit(nm, true, false, 65536, 1024, w, 1 << 20);
        printf("  k=%4d: %2d GEMMs x %.3f ms = %.3f ms forward (+ band build)\n", k, groups, ms, groups * ms);
    }
    return 0;
}
