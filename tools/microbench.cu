// Microbenchmarks for the FP32 issue model the Givens kernels rely on (sm_100a):
// FFMA vs FFMA2 (packed f32x2) throughput, FFMA2 mixed with SHFL / LDS.128 / SEL.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 16

__global__ void k_ffma(float* out, float a, float b) {
  float x[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = fmaf(x[i], a, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += x[i];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma2(float* out, float a, float b) {
  float2 x[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) x[i] = make_float2(threadIdx.x + i, i);
  float2 aa = make_float2(a, a);
  float2 bb = make_float2(b, b);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = __ffma2_rn(aa, x[i], bb);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CH; i++) s += x[i].x + x[i].y;
  if (s == 1234.5f) out[0] = s;
}

// FFMA2 with a per-iteration SHFL every `ratio` FFMA2s
template <int NSHFL>
__global__ void k_ffma2_shfl(float* out, float a, float b) {
  float2 x[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) x[i] = make_float2(threadIdx.x + i, i);
  float2 aa = make_float2(a, a);
  float y = threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = __ffma2_rn(aa, x[i], x[(i + 1) % CH]);
#pragma unroll
    for (int j = 0; j < NSHFL; j++) y = __shfl_down_sync(0xffffffffu, y, 1) + x[j].x;
  }
  float s = y;
#pragma unroll
  for (int i = 0; i < CH; i++) s += x[i].x + x[i].y;
  if (s == 1234.5f) out[0] = s;
}

template <int NLDS>
__global__ void k_ffma2_lds(float* out, float a, float b) {
  __shared__ float4 sm[32 * 16];
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) sm[i] = make_float4(i, i, i, i);
  __syncthreads();
  float2 x[CH];
#pragma unroll
  for (int i = 0; i < CH; i++) x[i] = make_float2(threadIdx.x + i, i);
  float2 acc = make_float2(0, 0);
  int lane = threadIdx.x & 31;
  for (int it = 0; it < ITERS; it++) {
    float4 v[NLDS > 0 ? NLDS : 1];
#pragma unroll
    for (int j = 0; j < NLDS; j++) v[j] = sm[((it + j) & 15) * 32 + lane];
#pragma unroll
    for (int i = 0; i < CH; i++) x[i] = __ffma2_rn(make_float2(a, a), x[i], x[(i + 1) % CH]);
#pragma unroll
    for (int j = 0; j < NLDS; j++) acc = __ffma2_rn(make_float2(v[j].x, v[j].y), acc, make_float2(v[j].z, v[j].w));
  }
  float s = acc.x + acc.y;
#pragma unroll
  for (int i = 0; i < CH; i++) s += x[i].x + x[i].y;
  if (s == 1234.5f) out[0] = s;
}

template <typename F>
double timeit(F f, int reps = 5) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clockRate %d kHz\n", p.name, p.multiProcessorCount, clk_khz);
  float* out; cudaMalloc(&out, 4);
  int sms = p.multiProcessorCount;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb);
    double threads = (double)blocks * tpb;
    double ms = timeit([&] { k_ffma<<<blocks, tpb>>>(out, 1.0001f, 0.5f); });
    double fma = threads * ITERS * CH;
    printf("FFMA  tpb=%4d: %.3f ms  %.2f TFMA/s  -> %.1f TFLOP/s\n", tpb, ms, fma / ms / 1e9, 2 * fma / ms / 1e9);
    ms = timeit([&] { k_ffma2<<<blocks, tpb>>>(out, 1.0001f, 0.5f); });
    fma = threads * ITERS * CH * 2;
    printf("FFMA2 tpb=%4d: %.3f ms  %.2f TFMA/s  -> %.1f TFLOP/s\n", tpb, ms, fma / ms / 1e9, 2 * fma / ms / 1e9);
  }
  int tpb = 256, blocks = sms * 8;
  double threads = (double)blocks * tpb;
#define SH(N) { double ms = timeit([&] { k_ffma2_shfl<N><<<blocks, tpb>>>(out, 1.0001f, 0.5f); }); \
    double fma = threads * ITERS * CH * 2; printf("FFMA2x%d + SHFLx%d: %.3f ms  %.2f TFMA/s\n", CH, N, ms, fma / ms / 1e9); }
  SH(0) SH(2) SH(4) SH(8) SH(16)
#define LD(N) { double ms = timeit([&] { k_ffma2_lds<N><<<blocks, tpb>>>(out, 1.0001f, 0.5f); }); \
    double fma = threads * ITERS * CH * 2; printf("FFMA2x%d + LDS128x%d: %.3f ms  %.2f TFMA/s (lds %.1f B/clk/SM @1.965GHz)\n", CH, N, ms, fma / ms / 1e9, threads*ITERS*N*16/(ms*1e-3)/sms/1.965e9); }
  LD(0) LD(1) LD(2) LD(4) LD(8) LD(16)
  return 0;
}
