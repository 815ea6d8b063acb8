// Adam (Kingma & Ba, bias-corrected) on the raw parameters (R30), shared by pgsag_adam_step
// (train.cu) and the fused A8 + Adam of pgsag_render_bwd_adam (preprocess_bwd.cu).  Every
// operation is an explicit round-to-nearest intrinsic, so both paths produce bitwise the same
// parameters and moments from the same float32 gradients.
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "internal.cuh"

namespace pgsag {

struct AdamP {
  float lr_mean, lr_scale, lr_rot, lr_op, lr_dc, lr_rest;
  float b1, b2, eps, flat_w;
  float ibc1, isbc2;  // 1 / (1 - b1^t), 1 / sqrt(1 - b2^t)
};

inline AdamP adam_params(const pgsag_adam_hparams* hp) {
  AdamP P;
  P.lr_mean = hp->lr_mean; P.lr_scale = hp->lr_scale; P.lr_rot = hp->lr_rot; P.lr_op = hp->lr_opacity;
  P.lr_dc = hp->lr_sh_dc; P.lr_rest = hp->lr_sh_rest;
  P.b1 = hp->beta1; P.b2 = hp->beta2; P.eps = hp->eps; P.flat_w = hp->flatten_weight;
  P.ibc1 = (float)(1.0 / (1.0 - pow((double)hp->beta1, (double)hp->step)));
  P.isbc2 = (float)(1.0 / sqrt(1.0 - pow((double)hp->beta2, (double)hp->step)));
  return P;
}

__device__ __forceinline__ float sqrt_approx(float v) {  // MUFU; sqrt(0) = 0
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}

// One element: (m, v) <- (b1 m + (1 - b1) g, b2 v + (1 - b2) g^2); returns
// raw - lr m / (1 - b1^t) / (sqrt(v / (1 - b2^t)) + eps).
__device__ __forceinline__ float adam_elem(const AdamP& P, float& m, float& v, float raw, float g, float lr) {
  m = __fmaf_rn(P.b1, m, __fmul_rn(1.f - P.b1, g));
  v = __fmaf_rn(P.b2, v, __fmul_rn(__fmul_rn(1.f - P.b2, g), g));
  return __fsub_rn(raw, __fdividef(__fmul_rn(__fmul_rn(lr, P.ibc1), m), __fmaf_rn(sqrt_approx(v), P.isbc2, P.eps)));
}

// The same on the moment arrays ([rows][n]) at row `row` of Gaussian i.
__device__ __forceinline__ float adam_at(const AdamP& P, float* __restrict__ M, float* __restrict__ V, int row,
                                         size_t n, size_t i, float raw, float g, float lr) {
  const size_t k = (size_t)row * n + i;
  float m = M[k], v = V[k];
  const float r = adam_elem(P, m, v, raw, g, lr);
  M[k] = m;
  V[k] = v;
  return r;
}

// L_s = mean_i min_k s_ik (ties -> lowest axis, R29): the minimum and its axis.
__device__ __forceinline__ float min_axis(float s0, float s1, float s2, int& kmin) {
  float smin = s0;
  kmin = 0;
  if (s1 < smin) { smin = s1; kmin = 1; }
  if (s2 < smin) { smin = s2; kmin = 2; }
  return smin;
}

// Raw-parameter gradients of the activated ones (R30): d/dlog s = s (dL/ds + [min axis] flat_w / n),
// d/dlogit o = o (1 - o) dL/do.
__device__ __forceinline__ float dlog_scale(float ds, bool is_min, float gflat, float s) {
  return __fmul_rn(__fadd_rn(ds, is_min ? gflat : 0.f), s);
}
__device__ __forceinline__ float dlogit_opacity(float dop, float o) {
  return __fmul_rn(__fmul_rn(dop, o), __fsub_rn(1.f, o));
}

}  // namespace pgsag
