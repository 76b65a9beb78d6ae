// Microbenchmark: the forward ring step's instruction mix without the ring (96 FFMA2 three-shear
// rotations + 8 LDS.128 coefficient loads + 8 SHFL + 12 FSEL per warp-step), 8 warps/SM, to see
// whether the FMA pipe can be kept busy next to this much smem/shuffle traffic.
#include <cstdio>
#include <cuda_runtime.h>

template <int NLDS, int NSHFL, bool SEL>
__global__ void __launch_bounds__(256, 1) k_mix(float* out, int iters) {
  __shared__ float4 sm[8 * 8 * 32];
  for (int i = threadIdx.x; i < 8 * 8 * 32; i += blockDim.x) sm[i] = make_float4(0.001f * i, 0.002f, 0.003f, 0.004f);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float2 T[2][16], B[2][16];
#pragma unroll
  for (int p = 0; p < 2; p++)
#pragma unroll
    for (int q = 0; q < 16; q++) { T[p][q] = make_float2(threadIdx.x + q, p); B[p][q] = make_float2(q, threadIdx.x); }
  for (int it = 0; it < iters; it++) {
    const float4* row = sm + (it & 7) * 256;
#pragma unroll
    for (int pp = 0; pp < 8; pp++) {
      float4 cf = (pp < NLDS) ? row[pp * 32 + lane] : make_float4(0.1f, 0.2f, 0.3f, 0.4f);
#pragma unroll
      for (int h = 0; h < 2; h++) {
        int q = 2 * pp + h;
        float tq = h ? cf.z : cf.x, sq = h ? cf.w : cf.y;
#pragma unroll
        for (int p = 0; p < 2; p++) {
          T[p][q] = __ffma2_rn(make_float2(-tq, -tq), B[p][q], T[p][q]);
          B[p][q] = __ffma2_rn(make_float2(sq, sq), T[p][q], B[p][q]);
          T[p][q] = __ffma2_rn(make_float2(-tq, -tq), B[p][q], T[p][q]);
        }
      }
    }
    // shift-like data movement
#pragma unroll
    for (int p = 0; p < 2; p++) {
      float a = T[p][0].x, b = T[p][0].y, c = B[p][15].x, d = B[p][15].y;
      if (NSHFL >= 4) {
        a = __shfl_down_sync(0xffffffffu, a, 1); b = __shfl_down_sync(0xffffffffu, b, 1);
        c = __shfl_up_sync(0xffffffffu, c, 1); d = __shfl_up_sync(0xffffffffu, d, 1);
      }
      if (SEL) {
        bool f = lane == 0, l = lane == 31;
        a = l ? B[p][15].x : a; b = l ? B[p][15].y : b;
        c = f ? T[p][1].x : c; d = f ? T[p][1].y : d;
        T[p][1].x = f ? T[p][0].x : T[p][1].x; T[p][1].y = f ? T[p][0].y : T[p][1].y;
      }
#pragma unroll
      for (int q = 0; q < 15; q++) T[p][q] = T[p][q + 1];
      T[p][15] = make_float2(a, b);
#pragma unroll
      for (int q = 15; q > 0; q--) B[p][q] = B[p][q - 1];
      B[p][0] = make_float2(c, d);
    }
  }
  float s = 0;
#pragma unroll
  for (int p = 0; p < 2; p++)
#pragma unroll
    for (int q = 0; q < 16; q++) s += T[p][q].x + B[p][q].y;
  if (s == 1234.5f) out[0] = s;
}

template <int NLDS, int NSHFL, bool SEL>
void run(float* out) {
  int iters = 4096;  // must be a multiple of 16 for the register renaming to close (unrolled 16x below)
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k_mix<NLDS, NSHFL, SEL><<<148, 256>>>(out, 16);
  cudaEventRecord(e0);
  k_mix<NLDS, NSHFL, SEL><<<148, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = 148.0 * 256 * iters * 96 * 2;
  printf("LDS128=%d SHFL=%d SEL=%d: %.2f TFMA/s (%.0f%% of 35.9)\n", NLDS, NSHFL * 2, SEL, fma / ms / 1e9, fma / ms / 1e9 / 35.9 * 100);
}

int main() {
  float* out; cudaMalloc(&out, 4);
  run<0, 0, false>(out);
  run<8, 0, false>(out);
  run<0, 4, false>(out);
  run<0, 4, true>(out);
  run<8, 4, true>(out);
  run<4, 4, true>(out);
  return 0;
}
