// Microbenchmark: FFMA2 throughput vs operand pattern (immediate, register scalar, pair coefficient, scalar FFMA, shared scalar, FSEL-interleaved). DESIGN.md §10a.
#include <cstdio>
#include <cuda_runtime.h>

#define NCH 16
template <int MODE>
__global__ void __launch_bounds__(256, 1) k(float *out, const float *__restrict__ cin, int iters) {
    float2 x[NCH], y[NCH];
    float c[NCH];
#pragma unroll
    for (int i = 0; i < NCH; i++) {
        x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        y[i] = make_float2(i * 0.25f, threadIdx.x * 1e-4f);
        c[i] = cin[(threadIdx.x + i) & 63];
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < NCH; i++) {
            if (MODE == 0) {  // distinct register scalar per instruction (three-shear, 1 pack)
                x[i] = __ffma2_rn(make_float2(c[i], c[i]), y[i], x[i]);
                y[i] = __ffma2_rn(make_float2(c[(i + 1) % NCH], c[(i + 1) % NCH]), x[i], y[i]);
                x[i] = __ffma2_rn(make_float2(c[i], c[i]), y[i], x[i]);
            } else if (MODE == 1) {  // immediates
                x[i] = __ffma2_rn(make_float2(0.01f * i, 0.01f * i), y[i], x[i]);
                y[i] = __ffma2_rn(make_float2(-0.02f * i, -0.02f * i), x[i], y[i]);
                x[i] = __ffma2_rn(make_float2(0.01f * i, 0.01f * i), y[i], x[i]);
            } else if (MODE == 2) {  // pair-valued coefficient (t, t') as a full register pair
                const float2 cc = make_float2(c[i], c[(i + 3) % NCH]);
                x[i] = __ffma2_rn(cc, y[i], x[i]);
                y[i] = __ffma2_rn(make_float2(c[(i + 1) % NCH], c[(i + 5) % NCH]), x[i], y[i]);
                x[i] = __ffma2_rn(cc, y[i], x[i]);
            } else if (MODE == 3) {  // scalar FFMA, 3 distinct regs, 2 columns (same flops)
                x[i].x = fmaf(c[i], y[i].x, x[i].x);
                x[i].y = fmaf(c[i], y[i].y, x[i].y);
                y[i].x = fmaf(c[(i + 1) % NCH], x[i].x, y[i].x);
                y[i].y = fmaf(c[(i + 1) % NCH], x[i].y, y[i].y);
                x[i].x = fmaf(c[i], y[i].x, x[i].x);
                x[i].y = fmaf(c[i], y[i].y, x[i].y);
            } else if (MODE == 5) {  // immediates + 2 FSEL per FFMA2 on the same data
                x[i] = __ffma2_rn(make_float2(0.01f * i, 0.01f * i), y[i], x[i]);
                const bool pr = c[i] > 0.f;
                float2 t = make_float2(pr ? x[i].x : y[i].x, pr ? x[i].y : y[i].y);
                y[i] = __ffma2_rn(make_float2(-0.02f * i, -0.02f * i), t, y[i]);
                t = make_float2(pr ? y[i].x : x[i].x, pr ? y[i].y : x[i].y);
                x[i] = __ffma2_rn(make_float2(0.01f * i, 0.01f * i), t, x[i]);
            } else if (MODE == 4) {  // FMUL2-free: scalar register coefficient shared by 2 packs (reuse)
                const int j = (i + NCH / 2) % NCH;
                x[i] = __ffma2_rn(make_float2(c[i], c[i]), y[i], x[i]);
                x[j] = __ffma2_rn(make_float2(c[i], c[i]), y[j], x[j]);
                y[i] = __ffma2_rn(make_float2(c[(i + 1) % NCH], c[(i + 1) % NCH]), x[i], y[i]);
                y[j] = __ffma2_rn(make_float2(c[(i + 1) % NCH], c[(i + 1) % NCH]), x[j], y[j]);
                x[i] = __ffma2_rn(make_float2(c[i], c[i]), y[i], x[i]);
                x[j] = __ffma2_rn(make_float2(c[i], c[i]), y[j], x[j]);
            }
        }
        // (coefficients are loop-invariant registers the compiler cannot fold: loaded from memory)
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < NCH; i++) s += x[i].x + y[i].y + x[i].y + y[i].x;
    if (s == 1234.5f) out[0] = s;
}

template <int MODE>
void run(float *out, const float *cin) {
    const int iters = 4000;
    k<MODE><<<148, 256>>>(out, cin, 10);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<148, 256>>>(out, cin, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double per = (MODE == 4) ? 6.0 * 2 * NCH : 6.0 * NCH;  // FMA-ops per thread per iteration (2 cols)
    const double fma = 148.0 * 256 * iters * per * (MODE == 4 ? 1 : 1);
    printf("mode %d: %.2f TFMA/s (%.0f%% of 37.2 nominal) %s\n", MODE, fma / ms / 1e9, fma / ms / 1e9 / 37.22 * 100,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float *out, *cin; cudaMalloc(&out, 4); cudaMalloc(&cin, 256);
    float h[64]; for (int i = 0; i < 64; i++) h[i] = 0.01f * (i + 1);
    cudaMemcpy(cin, h, 256, cudaMemcpyHostToDevice);
    run<0>(out, cin); run<1>(out, cin); run<2>(out, cin); run<3>(out, cin); run<4>(out, cin); run<5>(out, cin);
    return 0;
}
