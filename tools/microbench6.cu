// microbench2's three-shear FFMA2 pattern with and without ring-style register renaming across the
// W steps of an unrolled body (slot q of step u uses T[(q+u)%W], B[(q-u)%W]): is the kernels'
// operand cost a consequence of the renaming?
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>
template <typename F, int... I> __device__ __forceinline__ void unroll_impl(F &&f, std::integer_sequence<int, I...>) { (f(std::integral_constant<int, I>{}), ...); }
template <int N, typename F> __device__ __forceinline__ void unroll(F &&f) { unroll_impl(f, std::make_integer_sequence<int, N>{}); }
template <int W, int KP, bool REN>
__global__ void __launch_bounds__(256, 1) k(float *out, const float4 *__restrict__ coef, int iters) {
    float2 T[KP][W], B[KP][W];
#pragma unroll
    for (int p = 0; p < KP; p++)
#pragma unroll
        for (int q = 0; q < W; q++) { T[p][q] = make_float2(threadIdx.x + q, p); B[p][q] = make_float2(q, threadIdx.x); }
    float4 c[W / 2];
#pragma unroll
    for (int i = 0; i < W / 2; i++) c[i] = coef[(threadIdx.x + i) & 255];
    for (int it = 0; it < iters / W; it++) {
        unroll<W>([&](auto uc) {
            constexpr int u = decltype(uc)::value;
#pragma unroll
            for (int pp = 0; pp < W / 2; pp++) {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int q = 2 * pp + h;
                    const int qt = REN ? (q + u) % W : q, qb = REN ? (q + W - u) % W : q;
                    const float tq = h ? c[pp].z : c[pp].x, sq = h ? c[pp].w : c[pp].y;
#pragma unroll
                    for (int p = 0; p < KP; p++) {
                        T[p][qt] = __ffma2_rn(make_float2(-tq, -tq), B[p][qb], T[p][qt]);
                        B[p][qb] = __ffma2_rn(make_float2(sq, sq), T[p][qt], B[p][qb]);
                        T[p][qt] = __ffma2_rn(make_float2(-tq, -tq), B[p][qb], T[p][qt]);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < W / 2; i++) c[i] = make_float4(c[i].y, c[i].x, c[i].w, c[i].z);
        });
    }
    float s = 0;
#pragma unroll
    for (int p = 0; p < KP; p++)
#pragma unroll
        for (int q = 0; q < W; q++) s += T[p][q].x + B[p][q].y;
    if (s == 1234.5f) out[0] = s;
}
template <int W, int KP, bool REN> void run(float *out, float4 *coef) {
    const int iters = 2048;
    k<W, KP, REN><<<148, 256>>>(out, coef, 32);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<W, KP, REN><<<148, 256>>>(out, coef, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = 148.0 * 256 * (iters / W * W) * W * KP * 2 * 3;
    printf("W=%d KP=%d renaming=%d: %.1f%% of 37.2 TFMA/s %s\n", W, KP, (int)REN, fma / ms / 1e9 / 37.22 * 100, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    float *out; float4 *coef; cudaMalloc(&out, 4); cudaMalloc(&coef, 256 * 16);
    float4 h[256]; for (int i = 0; i < 256; i++) h[i] = make_float4(0.01f * i, 0.02f, -0.03f, 0.004f * i);
    cudaMemcpy(coef, h, sizeof h, cudaMemcpyHostToDevice);
    run<16, 2, false>(out, coef); run<16, 2, true>(out, coef); run<16, 1, false>(out, coef); run<16, 1, true>(out, coef);
}
