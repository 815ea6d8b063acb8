// Per-pair alpha evaluation shared by the forward (A6) and backward (A7)
// compositors.  Every operation is an explicit round-to-nearest intrinsic, so both
// kernels take bit-identical skip / clamp / termination decisions whatever the
// compiler does elsewhere (the backward must retrace exactly the forward's list).
//
// power = -0.5 (ca dx^2 + cc dy^2) - cb dx dy  (P:78 2D Gaussian; R5 pixel centres)
// alpha = min(0.99, o exp(power)), skipped if power > 0 or alpha < 1/255 (R6).
// Evaluated as p2 = log2(e) * power = dx (A' dx + B' dy) + C' dy^2 with the
// pre-scaled conic (A', B', C') = log2(e) * (-0.5 ca, -cb, -0.5 cc), and
// exp(power) = ex2(p2) on the MUFU unit.
#pragma once
#include <cuda_runtime.h>

namespace pgsag {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kAlphaMin = 1.0f / 255.0f;
constexpr float kAlphaMax = 0.99f;
constexpr float kTmin = 1e-4f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// (A', B', C', o) from (ca, cb, cc, o)
__device__ __forceinline__ float4 scaled_conic(float4 co) {
  return make_float4(__fmul_rn(-0.5f * kLog2e, co.x), __fmul_rn(-kLog2e, co.y), __fmul_rn(-0.5f * kLog2e, co.z),
                     co.w);
}

__device__ __forceinline__ float power2(const float4& sc, float dx, float dy) {
  const float t = __fmaf_rn(sc.y, dy, __fmul_rn(sc.x, dx));  // A'dx + B'dy
  return __fmaf_rn(dx, t, __fmul_rn(__fmul_rn(sc.z, dy), dy));
}

}  // namespace pgsag
