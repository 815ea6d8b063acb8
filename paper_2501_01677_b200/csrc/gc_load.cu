// NEXT-1: L_GC-load weights (Eq. 9 "w_i is a gradient-dependent weight
// nabla I for pixel i"; reading R23).  Two HBM-bound passes over the image:
//   (1) gray -> 3x3 Sobel magnitude (replicated borders) written to w, plus the
//       mask-pixel sum and count (block reduction -> f64 atomics spread over 8 slots);
//   (2) w <- clamp(w / mean, 0.1, 10) on mask pixels (floor if mean == 0), 1 off-mask.
// The per-pixel statistics (N, sum r, sum r^2 of r = g / w) are fused into A6's
// epilogue and the surrogate gradient into A7 (render_fwd.cu / render_bwd.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kGX = 32, kGY = 32;  // 32x32 pixel blocks (256 threads, 4 rows each), halo 1
constexpr int kGSlots = 8;         // the mask-pixel sums are spread over 8 (sum, count) slots

__global__ void __launch_bounds__(256) sobel_kernel(const float* __restrict__ img, const uint8_t* __restrict__ mask,
                                                    int W, int H, float* __restrict__ w, double* __restrict__ acc) {
  __shared__ float s_g[kGY + 2][kGX + 2];
  __shared__ float s_red[8][2];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * kGX, y0 = blockIdx.y * kGY;
  const size_t HW = (size_t)W * H;
  for (int ly = ty; ly < kGY + 2; ly += 8) {
    const int gy = min(max(y0 + ly - 1, 0), H - 1);
    for (int lx = tx; lx < kGX + 2; lx += 32) {
      const int gx = min(max(x0 + lx - 1, 0), W - 1);
      const size_t p = (size_t)gy * W + gx;
      s_g[ly][lx] = 0.299f * __ldg(img + p) + 0.587f * __ldg(img + HW + p) + 0.114f * __ldg(img + 2 * HW + p);
    }
  }
  __syncthreads();
  float sum = 0.f, cnt = 0.f;
  const int x = x0 + tx, lx = tx + 1;
#pragma unroll
  for (int k = 0; k < kGY / 8; ++k) {
    const int ly = ty + 8 * k + 1, y = y0 + ly - 1;
    if (x < W && y < H) {
      const float gx = (s_g[ly - 1][lx + 1] + 2.f * s_g[ly][lx + 1] + s_g[ly + 1][lx + 1]) -
                       (s_g[ly - 1][lx - 1] + 2.f * s_g[ly][lx - 1] + s_g[ly + 1][lx - 1]);
      const float gy = (s_g[ly + 1][lx - 1] + 2.f * s_g[ly + 1][lx] + s_g[ly + 1][lx + 1]) -
                       (s_g[ly - 1][lx - 1] + 2.f * s_g[ly - 1][lx] + s_g[ly - 1][lx + 1]);
      const float mag = sqrtf(gx * gx + gy * gy);
      const size_t p = (size_t)y * W + x;
      w[p] = mag;
      if (__ldg(mask + p)) { sum += mag; cnt += 1.f; }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if (tx == 0) { s_red[ty][0] = sum; s_red[ty][1] = cnt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sd = 0.0, c = 0.0;
    for (int k = 0; k < 8; ++k) { sd += s_red[k][0]; c += s_red[k][1]; }
    const int slot = (blockIdx.x + blockIdx.y) & (kGSlots - 1);  // fewer same-address atomics
    if (c > 0.0) { atomicAdd(acc + 2 * slot, sd); atomicAdd(acc + 2 * slot + 1, c); }
  }
}

__global__ void gc_normalize_kernel(const uint8_t* __restrict__ mask, size_t HW, float* __restrict__ w,
                                    const double* __restrict__ acc) {
  double S = 0.0, Nn = 0.0;
#pragma unroll
  for (int k = 0; k < kGSlots; ++k) { S += acc[2 * k]; Nn += acc[2 * k + 1]; }
  const double m = Nn > 0.0 ? S / Nn : 0.0;
  const float inv = m > 0.0 ? (float)(1.0 / m) : 0.f;
  for (size_t p = blockIdx.x * (size_t)blockDim.x + threadIdx.x; p < HW; p += (size_t)gridDim.x * blockDim.x) {
    if (!mask[p]) { w[p] = 1.0f; continue; }
    w[p] = m > 0.0 ? fminf(fmaxf(w[p] * inv, 0.1f), 10.0f) : 0.1f;
  }
}

}  // namespace

cudaError_t launch_gc_weights(const float* image, const uint8_t* mask, int W, int H, float* w, double* acc,
                              cudaStream_t st) {
  cudaMemsetAsync(acc, 0, 2 * kGSlots * sizeof(double), st);
  {
    KTimer kt_("N1_gc_sobel", st);
    dim3 grid((W + kGX - 1) / kGX, (H + kGY - 1) / kGY);
    sobel_kernel<<<grid, 256, 0, st>>>(image, mask, W, H, w, acc);
  }
  {
    KTimer kt_("N1_gc_normalize", st);
    const size_t HW = (size_t)W * H;
    const int blocks = (int)((HW + 1023) / 1024 < 148 * 8 ? (HW + 1023) / 1024 : 148 * 8);
    gc_normalize_kernel<<<blocks > 0 ? blocks : 1, 1024, 0, st>>>(mask, HW, w, acc);
  }
  return cudaGetLastError();
}

}  // namespace pgsag
