// FP32 peak microbenchmark (the A6/A7 roofline denominator is the derived
// 148 x 128 x 2 x clock figure AND a measured FMA rate from independent chains on all SMs).
// mode 0: scalar FFMA (3-register form), mode 1: packed FFMA2 (FP32x2).  Each thread runs
// 16 independent FMA chains (8 float2 chains in mode 1) for `iters` iterations.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pgsag {
namespace {

__global__ void __launch_bounds__(256) ffma_kernel(int iters, float a, float b, float* out) {
  float acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = (float)(threadIdx.x + k);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = fmaf(acc[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += acc[k];
  if (s == 1.2345f) out[threadIdx.x] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) ffma2_kernel(int iters, float a, float b, float* out) {
  float2 acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = make_float2((float)(threadIdx.x + k), (float)(k - threadIdx.x));
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(acc[k], a2, b2);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y;
  if (s == 1.2345f) out[threadIdx.x] = s;
}

}  // namespace

cudaError_t launch_fp32_microbench(int mode, int iters, float* scratch, float* ms, double* flops, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // warm-up, then the timed launch
  for (int rep = 0; rep < 2; ++rep) {
    if (rep == 1) cudaEventRecord(e0, st);
    if (mode == 0)
      ffma_kernel<<<blocks, 256, 0, st>>>(iters, 0.999f, 1e-3f, scratch);
    else
      ffma2_kernel<<<blocks, 256, 0, st>>>(iters, 0.999f, 1e-3f, scratch);
  }
  cudaEventRecord(e1, st);
  cudaError_t e = cudaEventSynchronize(e1);
  float t = 0.f;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = t;
  *flops = 2.0 * 16.0 * (double)iters * (double)blocks * 256.0;  // 16 FMAs per thread-iteration either way
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace pgsag
