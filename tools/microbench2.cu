// Microbenchmark: achievable FMA-pipe rate of the three-shear rotation pattern (FFMA2 with a
// scalar coefficient) at different warps/SMSP and columns/thread, without shuffles/LDS.
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int KP>
__global__ void k_rot(float* out, const float4* __restrict__ coef, int iters) {
  float2 T[KP][W], B[KP][W];
#pragma unroll
  for (int p = 0; p < KP; p++)
#pragma unroll
    for (int q = 0; q < W; q++) { T[p][q] = make_float2(threadIdx.x + q, p); B[p][q] = make_float2(q, threadIdx.x); }
  float4 c[W / 2];
#pragma unroll
  for (int i = 0; i < W / 2; i++) c[i] = coef[i];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int pp = 0; pp < W / 2; pp++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        int q = 2 * pp + h;
        float tq = h ? c[pp].z : c[pp].x, sq = h ? c[pp].w : c[pp].y;
#pragma unroll
        for (int p = 0; p < KP; p++) {
          T[p][q] = __ffma2_rn(make_float2(-tq, -tq), B[p][q], T[p][q]);
          B[p][q] = __ffma2_rn(make_float2(sq, sq), T[p][q], B[p][q]);
          T[p][q] = __ffma2_rn(make_float2(-tq, -tq), B[p][q], T[p][q]);
        }
      }
    }
    // rotate coefficient roles so the compiler cannot hoist
#pragma unroll
    for (int i = 0; i < W / 2; i++) c[i] = make_float4(c[i].y, c[i].x, c[i].w, c[i].z);
  }
  float s = 0;
#pragma unroll
  for (int p = 0; p < KP; p++)
#pragma unroll
    for (int q = 0; q < W; q++) s += T[p][q].x + B[p][q].y;
  if (s == 1234.5f) out[0] = s;
}

template <int W, int KP>
void run(int warps_per_sm, float* out, float4* coef) {
  int iters = 2000;
  int tpb = 32 * warps_per_sm;
  int blocks = 148;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_rot<W, KP><<<blocks, tpb>>>(out, coef, 10);
  cudaEventRecord(e0);
  k_rot<W, KP><<<blocks, tpb>>>(out, coef, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = (double)blocks * tpb * iters * W * KP * 2 * 3;
  cudaFuncAttributes a; cudaFuncGetAttributes(&a, k_rot<W, KP>);
  printf("W=%2d KP=%d warps/SM=%2d regs=%3d: %.2f TFMA/s (%.0f%% of 35.9 measured FFMA peak) err=%s\n", W, KP, warps_per_sm,
         a.numRegs, fma / ms / 1e9, fma / ms / 1e9 / 35.9 * 100, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float* out; cudaMalloc(&out, 4);
  float4* coef; cudaMalloc(&coef, 1024 * 16);
  cudaMemset(coef, 0, 1024 * 16);
  for (int w : {4, 8, 12, 16}) run<16, 2>(w, out, coef);
  for (int w : {8, 16, 24}) run<16, 1>(w, out, coef);
  for (int w : {8, 16}) run<8, 2>(w, out, coef);
  return 0;
}
