// A8: per-Gaussian chain rule from A7's screen-space gradients to the 3D
// parameters (oracle O6), float64 arithmetic, one thread per Gaussian.
#include <cuda_runtime.h>
#include <stdint.h>

#include "adam.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kG2 = 14;

// --------------------------------------------------------------------- A8
// Per-Gaussian chain rule in float64 (FP64 on B200 is ample for ~600 ops per
// Gaussian; the conic -> covariance -> Sigma chain amplifies rounding, so it is
// done in double from A7's float32-accumulated 2D gradients, widened exactly).
struct CamB {
  double fx, fy, C[3], R[9], lx, ly;
};

#ifndef PGSAG_A8_MINB
#define PGSAG_A8_MINB 4
#endif

// Fused A8 + Adam (pgsag_render_bwd_adam): the optimiser state; the gradients are applied where
// A8 produces them (adam.cuh, bitwise the pgsag_adam_step update) instead of being written.
struct AdamFused {
  AdamP P;
  float *mean, *scale, *rot, *op, *sh, *log_scale, *logit_op, *m, *v;
  double* flat;  // L_s accumulator (zeroed by the launcher)
  const uint32_t* skip;  // optional device flag: nonzero = this view's sort overflowed, no update
};

// The Adam step of Gaussian i from its float32 gradients staged in shared memory by A8 (sg: this
// thread's column, row stride 128): rows in batches of 8, all loads of a batch before its stores.
// Same arithmetic as adam_kernel (adam.cuh).
template <int K3>
__device__ __forceinline__ void adam_rows(const AdamFused& F, size_t n, size_t i, const float* sg, float gflat) {
  constexpr int R = 11 + K3;
  const AdamP& P = F.P;
  int kmin;
  const float s3[3] = {__ldg(F.scale + i), __ldg(F.scale + n + i), __ldg(F.scale + 2 * n + i)};
  min_axis(s3[0], s3[1], s3[2], kmin);
  const float o = __ldg(F.op + i);
  auto raw_ptr = [&](int r) -> float* {
    return r < 3 ? F.mean + r * n : r < 6 ? F.log_scale + (r - 3) * n : r < 10 ? F.rot + (r - 6) * n
           : r == 10 ? F.logit_op : F.sh + (r - 11) * n;
  };
#pragma unroll
  for (int r0 = 0; r0 < R; r0 += 8) {
    float g[8], m[8], v[8], raw[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = r0 + q;
      if (r < R) {
        g[q] = sg[r * 128];
        m[q] = __ldg(F.m + r * n + i);
        v[q] = __ldg(F.v + r * n + i);
        raw[q] = __ldg(raw_ptr(r) + i);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int r = r0 + q;
      if (r < R) {
        float gr = g[q], lr;
        if (r < 3) lr = P.lr_mean;
        else if (r < 6) { gr = dlog_scale(gr, r - 3 == kmin, gflat, s3[r - 3]); lr = P.lr_scale; }
        else if (r < 10) lr = P.lr_rot;
        else if (r == 10) { gr = dlogit_opacity(gr, o); lr = P.lr_op; }
        else lr = r < 14 ? P.lr_dc : P.lr_rest;
        const float nr = adam_elem(P, m[q], v[q], raw[q], gr, lr);
        F.m[r * n + i] = m[q];
        F.v[r * n + i] = v[q];
        raw_ptr(r)[i] = nr;
        if (r >= 3 && r < 6) F.scale[(r - 3) * n + i] = expf(nr);
        if (r == 10) F.op[i] = 1.f / (1.f + expf(-nr));
      }
    }
  }
}

// A8 for one Gaussian.  kAdam: the float32 parameter gradients go to this thread's column of the
// block's shared staging area (sg, row stride 128) instead of global memory.
template <int DEG, bool kAdam>
__device__ __forceinline__ void a8_gaussian(
    int n, int i, const float* __restrict__ mean, const float* __restrict__ scale, const float* __restrict__ rot,
    const float* __restrict__ sh, const uint32_t* __restrict__ flags, const float4* __restrict__ g2d,
    const float4* __restrict__ conic_o, const CamB& cam,
    float* __restrict__ dmean, float* __restrict__ dscale, float* __restrict__ drot, float* __restrict__ dopac,
    float* __restrict__ dsh, float* __restrict__ absgrad, float* __restrict__ grad2d,
    const uint32_t* __restrict__ tiles_touched, float* __restrict__ daccum, float* __restrict__ dcount, double hw,
    double hh, float* gst) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  if (i >= n) return;
  const uint32_t fl = flags[i];
  // every per-Gaussian load issued before the liveness branch: one memory latency, not two
  float4 g2v[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) g2v[c] = g2d[(size_t)i * 4 + c];
  const float4 co = conic_o[i];
  const float mf[3] = {mean[i], mean[n + i], mean[2 * n + i]};
  const float rf[4] = {rot[i], rot[n + i], rot[2 * n + i], rot[3 * n + i]};
  const float sf[3] = {scale[i], scale[n + i], scale[2 * n + i]};
  if ((fl & PGSAG_F_LIVE) != PGSAG_F_LIVE) {
    if (kAdam) {
#pragma unroll
      for (int r = 0; r < 11 + 3 * K; ++r) gst[r * 128] = 0.f;
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) { dmean[(size_t)k * n + i] = 0.f; dscale[(size_t)k * n + i] = 0.f; }
#pragma unroll
      for (int k = 0; k < 4; ++k) drot[(size_t)k * n + i] = 0.f;
      dopac[i] = 0.f;
#pragma unroll
      for (int k = 0; k < 3 * K; ++k) dsh[(size_t)k * n + i] = 0.f;
    }
    if (absgrad) absgrad[i] = 0.f;
    if (grad2d)
      for (int c = 0; c < kG2; ++c) grad2d[(size_t)c * n + i] = 0.f;
    return;
  }
  double gg[16];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float4 q = g2v[c];
    gg[4 * c] = q.x; gg[4 * c + 1] = q.y; gg[4 * c + 2] = q.z; gg[4 * c + 3] = q.w;
  }
  {  // A7's moments of dpow = alpha dalpha -> the screen-space gradients, with the conic (ca, cb, cc) and
     // o the forward blended with (A1's float values): alpha = o 2^p, p = -log2(e)/2 (ca dx^2 + 2 cb dx dy
     // + cc dy^2), dx = px - u: du = ca S1 + cb Sy, dv = cb S1 + cc Sy, dca = -S2 / 2, dcb = -Sxy,
     // dcc = -Syy / 2, do = S0 / o
    const double S1 = gg[0], Sy = gg[1], S2 = gg[2], Sxy = gg[3], Syy = gg[4], S0 = gg[5];
    gg[0] = (double)co.x * S1 + (double)co.y * Sy;
    gg[1] = (double)co.y * S1 + (double)co.z * Sy;
    gg[2] = -0.5 * S2;
    gg[3] = -Sxy;
    gg[4] = -0.5 * Syy;
    gg[5] = S0 / (double)co.w;
  }
  if (grad2d) {
#pragma unroll
    for (int c = 0; c < kG2; ++c) grad2d[(size_t)c * n + i] = (float)gg[c];
  }
  const double* Rc = cam.R;
  const double t[3] = {(double)mf[0] - cam.C[0], (double)mf[1] - cam.C[1], (double)mf[2] - cam.C[2]};
  double pc[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) pc[r] = Rc[3 * r] * t[0] + Rc[3 * r + 1] * t[1] + Rc[3 * r + 2] * t[2];
  const double x = pc[0], y = pc[1], z = pc[2];
  const double q0[4] = {rf[0], rf[1], rf[2], rf[3]};
  const double qn = sqrt(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
  const double w = q0[0] / qn, X = q0[1] / qn, Y = q0[2] / qn, Z = q0[3] / qn;
  double Rg[3][3];
  Rg[0][0] = 1. - 2. * (Y * Y + Z * Z); Rg[0][1] = 2. * (X * Y - w * Z); Rg[0][2] = 2. * (X * Z + w * Y);
  Rg[1][0] = 2. * (X * Y + w * Z); Rg[1][1] = 1. - 2. * (X * X + Z * Z); Rg[1][2] = 2. * (Y * Z - w * X);
  Rg[2][0] = 2. * (X * Z - w * Y); Rg[2][1] = 2. * (Y * Z + w * X); Rg[2][2] = 1. - 2. * (X * X + Y * Y);
  const double s[3] = {sf[0], sf[1], sf[2]};
  double Mg[3][3], Sig[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Mg[r][c] = Rg[r][c] * s[c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Sig[r][c] = Mg[r][0] * Mg[c][0] + Mg[r][1] * Mg[c][1] + Mg[r][2] * Mg[c][2];
  const bool clx = fl & PGSAG_F_CLAMP_X, cly = fl & PGSAG_F_CLAMP_Y;
  const double xz = x / z, yz = y / z;
  const double cxz = clx ? fmin(fmax(xz, -cam.lx), cam.lx) : xz;
  const double cyz = cly ? fmin(fmax(yz, -cam.ly), cam.ly) : yz;
  const double J00 = cam.fx / z, J02 = -cam.fx * cxz / z, J11 = cam.fy / z, J12 = -cam.fy * cyz / z;
  double Tm[2][3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    Tm[0][b] = J00 * Rc[b] + J02 * Rc[6 + b];
    Tm[1][b] = J11 * Rc[3 + b] + J12 * Rc[6 + b];
  }
  double STm[2][3];  // Sig Tm_a^T
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) STm[a][k] = Sig[k][0] * Tm[a][0] + Sig[k][1] * Tm[a][1] + Sig[k][2] * Tm[a][2];
  const double A = Tm[0][0] * STm[0][0] + Tm[0][1] * STm[0][1] + Tm[0][2] * STm[0][2] + 0.3;
  const double B = Tm[0][0] * STm[1][0] + Tm[0][1] * STm[1][1] + Tm[0][2] * STm[1][2];
  const double Cc = Tm[1][0] * STm[1][0] + Tm[1][1] * STm[1][1] + Tm[1][2] * STm[1][2] + 0.3;
  const double det = A * Cc - B * B;
  const double id2 = 1.0 / (det * det);
  const double dca = gg[2], dcb = gg[3], dcc = gg[4];
  const double dA = (-Cc * Cc * dca + B * Cc * dcb - B * B * dcc) * id2;
  const double dC = (-B * B * dca + A * B * dcb - A * A * dcc) * id2;
  const double dB = (2. * B * Cc * dca - (A * Cc + B * B) * dcb + 2. * A * B * dcc) * id2;
  double dSig[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int l = 0; l < 3; ++l)
      dSig[k][l] = dA * Tm[0][k] * Tm[0][l] + dC * Tm[1][k] * Tm[1][l] + dB * Tm[0][k] * Tm[1][l];
  double dTm[2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dTm[0][k] = 2. * dA * STm[0][k] + dB * STm[1][k];
    dTm[1][k] = 2. * dC * STm[1][k] + dB * STm[0][k];
  }
  const double dJ00 = dTm[0][0] * Rc[0] + dTm[0][1] * Rc[1] + dTm[0][2] * Rc[2];
  const double dJ02 = dTm[0][0] * Rc[6] + dTm[0][1] * Rc[7] + dTm[0][2] * Rc[8];
  const double dJ11 = dTm[1][0] * Rc[3] + dTm[1][1] * Rc[4] + dTm[1][2] * Rc[5];
  const double dJ12 = dTm[1][0] * Rc[6] + dTm[1][1] * Rc[7] + dTm[1][2] * Rc[8];
  const double iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
  double dp0 = 0., dp1 = 0., dp2 = 0.;
  dp2 += -cam.fx * iz2 * dJ00 - cam.fy * iz2 * dJ11;
  if (!clx) { dp0 += -cam.fx * iz2 * dJ02; dp2 += 2. * cam.fx * x * iz3 * dJ02; }
  else { dp2 += cam.fx * cxz * iz2 * dJ02; }
  if (!cly) { dp1 += -cam.fy * iz2 * dJ12; dp2 += 2. * cam.fy * y * iz3 * dJ12; }
  else { dp2 += cam.fy * cyz * iz2 * dJ12; }
  const double du = gg[0], dv = gg[1];
  if (daccum && tiles_touched[i] > 0) {  // densification statistic (R31): |(du W/2, dv H/2)|
    daccum[i] += (float)sqrt((du * hw) * (du * hw) + (dv * hh) * (dv * hh));
    dcount[i] += 1.0f;
  }
  dp0 += cam.fx * iz * du;
  dp1 += cam.fy * iz * dv;
  dp2 += -(cam.fx * x * du + cam.fy * y * dv) * iz2;
  double dt[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) dt[k] = Rc[k] * dp0 + Rc[3 + k] * dp1 + Rc[6 + k] * dp2;
  double dRg[3][3], ds[3] = {0., 0., 0.};
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      double acc = 0.;
#pragma unroll
      for (int l = 0; l < 3; ++l) acc += (dSig[k][l] + dSig[l][k]) * Mg[l][m];
      ds[m] += acc * Rg[k][m];
      dRg[k][m] = acc * s[m];
    }
  const int ax = (fl >> PGSAG_F_AXIS_SHIFT) & 3;
  const double sg = (fl & PGSAG_F_NFLIP) ? -1. : 1.;
  const double ddist = gg[12];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double nk = sg * (ax == 0 ? Rg[k][0] : ax == 1 ? Rg[k][1] : Rg[k][2]);
    const double dn = Rc[k] * gg[9] + Rc[3 + k] * gg[10] + Rc[6 + k] * gg[11] + t[k] * ddist;
    dt[k] += nk * ddist;
    if (ax == 0) dRg[k][0] += sg * dn;
    else if (ax == 1) dRg[k][1] += sg * dn;
    else dRg[k][2] += sg * dn;
  }
  double dq[4] = {0., 0., 0., 0.};
  dq[2] += -4. * Y * dRg[0][0]; dq[3] += -4. * Z * dRg[0][0];
  dq[1] += 2. * Y * dRg[0][1]; dq[2] += 2. * X * dRg[0][1]; dq[0] += -2. * Z * dRg[0][1]; dq[3] += -2. * w * dRg[0][1];
  dq[1] += 2. * Z * dRg[0][2]; dq[3] += 2. * X * dRg[0][2]; dq[0] += 2. * Y * dRg[0][2]; dq[2] += 2. * w * dRg[0][2];
  dq[1] += 2. * Y * dRg[1][0]; dq[2] += 2. * X * dRg[1][0]; dq[0] += 2. * Z * dRg[1][0]; dq[3] += 2. * w * dRg[1][0];
  dq[1] += -4. * X * dRg[1][1]; dq[3] += -4. * Z * dRg[1][1];
  dq[2] += 2. * Z * dRg[1][2]; dq[3] += 2. * Y * dRg[1][2]; dq[0] += -2. * X * dRg[1][2]; dq[1] += -2. * w * dRg[1][2];
  dq[1] += 2. * Z * dRg[2][0]; dq[3] += 2. * X * dRg[2][0]; dq[0] += -2. * Y * dRg[2][0]; dq[2] += -2. * w * dRg[2][0];
  dq[2] += 2. * Z * dRg[2][1]; dq[3] += 2. * Y * dRg[2][1]; dq[0] += 2. * X * dRg[2][1]; dq[1] += 2. * w * dRg[2][1];
  dq[1] += -4. * X * dRg[2][2]; dq[2] += -4. * Y * dRg[2][2];
  const double qh[4] = {w, X, Y, Z};
  const double qdot = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float gq = (float)((dq[k] - qh[k] * qdot) / qn);
    if (kAdam) gst[(6 + k) * 128] = gq;
    else drot[(size_t)k * n + i] = gq;
  }
  // SH colour: rgb_c = max(0, sum_l Y_l(dir) sh_lc + 0.5)
  const double len = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  const double il = 1.0 / len;
  const double dx = t[0] * il, dy = t[1] * il, dz = t[2] * il;
  // SH part in float, one basis function at a time (value and gradient inline, streamed to dsh):
  // no per-thread arrays, so A8 stays in registers at a useful occupancy.
  float dd0 = 0.f, dd1 = 0.f, dd2 = 0.f;
  {
    const float x = (float)dx, y = (float)dy, z = (float)dz;
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    const float gcs[3] = {(fl & PGSAG_F_RGB_CLAMP0) ? 0.f : (float)gg[6],
                          (fl & (PGSAG_F_RGB_CLAMP0 << 1)) ? 0.f : (float)gg[7],
                          (fl & (PGSAG_F_RGB_CLAMP0 << 2)) ? 0.f : (float)gg[8]};
    auto term = [&](int l, float Yl, float gx, float gy, float gz) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const size_t k = (size_t)(l * 3 + c) * n + i;
        const float shv = __ldg(sh + k), gsh = Yl * gcs[c];
        if (kAdam) gst[(11 + l * 3 + c) * 128] = gsh;
        else dsh[k] = gsh;
        const float f = shv * gcs[c];
        dd0 += gx * f; dd1 += gy * f; dd2 += gz * f;
      }
    };
    term(0, 0.28209479177387814f, 0.f, 0.f, 0.f);
    if (DEG >= 1) {
      const float c1 = 0.4886025119029199f;
      term(1, -c1 * y, 0.f, -c1, 0.f);
      term(2, c1 * z, 0.f, 0.f, c1);
      term(3, -c1 * x, -c1, 0.f, 0.f);
    }
    if (DEG >= 2) {
      const float a = 1.0925484305920792f, b = 0.31539156525252005f, e = 0.5462742152960396f;
      term(4, a * xy, a * y, a * x, 0.f);
      term(5, -a * yz, 0.f, -a * z, -a * y);
      term(6, b * (2.f * zz - xx - yy), -2.f * b * x, -2.f * b * y, 4.f * b * z);
      term(7, -a * xz, -a * z, 0.f, -a * x);
      term(8, e * (xx - yy), 2.f * e * x, -2.f * e * y, 0.f);
    }
    if (DEG >= 3) {
      const float c0 = -0.5900435899266435f, cA = 2.890611442640554f, cB = -0.4570457994644658f,
                  cC = 0.3731763325901154f, cD = 1.445305721320277f;
      term(9, c0 * y * (3.f * xx - yy), 6.f * c0 * xy, c0 * (3.f * xx - 3.f * yy), 0.f);
      term(10, cA * xy * z, cA * yz, cA * xz, cA * xy);
      term(11, cB * y * (4.f * zz - xx - yy), -2.f * cB * xy, cB * (4.f * zz - xx - 3.f * yy), 8.f * cB * yz);
      term(12, cC * z * (2.f * zz - 3.f * xx - 3.f * yy), -6.f * cC * xz, -6.f * cC * yz,
           cC * (6.f * zz - 3.f * xx - 3.f * yy));
      term(13, cB * x * (4.f * zz - xx - yy), cB * (4.f * zz - 3.f * xx - yy), -2.f * cB * xy, 8.f * cB * xz);
      term(14, cD * z * (xx - yy), 2.f * cD * xz, -2.f * cD * yz, cD * (xx - yy));
      term(15, c0 * x * (xx - 3.f * yy), c0 * (3.f * xx - 3.f * yy), -6.f * c0 * xy, 0.f);
    }
  }
  const double ddot = dx * dd0 + dy * dd1 + dz * dd2;
  dt[0] += (dd0 - dx * ddot) * il;
  dt[1] += (dd1 - dy * ddot) * il;
  dt[2] += (dd2 - dz * ddot) * il;
  if (kAdam) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      gst[k * 128] = (float)dt[k];
      gst[(3 + k) * 128] = (float)ds[k];
    }
    gst[10 * 128] = (float)gg[5];
  } else {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      dmean[(size_t)k * n + i] = (float)dt[k];
      dscale[(size_t)k * n + i] = (float)ds[k];
    }
    dopac[i] = (float)gg[5];
  }
  if (absgrad) absgrad[i] = (float)gg[13];
}

template <int DEG, bool kAdam>
__global__ void __launch_bounds__(128, PGSAG_A8_MINB) preprocess_bwd_kernel(
    int n, const float* __restrict__ mean, const float* __restrict__ scale, const float* __restrict__ rot,
    const float* __restrict__ sh, const uint32_t* __restrict__ flags, const float4* __restrict__ g2d,
    const float4* __restrict__ conic_o, CamB cam,
    float* __restrict__ dmean, float* __restrict__ dscale, float* __restrict__ drot, float* __restrict__ dopac,
    float* __restrict__ dsh, float* __restrict__ absgrad, float* __restrict__ grad2d,
    const uint32_t* __restrict__ tiles_touched, float* __restrict__ daccum, float* __restrict__ dcount, double hw,
    double hh, AdamFused F) {
  constexpr int K3 = 3 * (DEG + 1) * (DEG + 1);
  __shared__ float s_g[kAdam ? (11 + K3) * 128 : 1];  // fused: the gradients, one column per thread
  if (kAdam && F.skip && *F.skip) return;  // overflowed view: its lists were empty, leave the state
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float gflat = kAdam ? F.P.flat_w / (float)n : 0.f;
  if (kAdam) {  // L_s = mean of min(scale) before the update: block sum, one atomic per block
    __shared__ float s_flat[4];
    float sm = 0.f;
    if (i < n) {
      int km;
      sm = min_axis(F.scale[i], F.scale[(size_t)n + i], F.scale[2 * (size_t)n + i], km);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sm += __shfl_xor_sync(0xffffffffu, sm, o);
    if ((threadIdx.x & 31) == 0) s_flat[threadIdx.x >> 5] = sm;
    __syncthreads();
    if (threadIdx.x == 0 && F.flat)
      atomicAdd(F.flat, ((double)s_flat[0] + s_flat[1] + s_flat[2] + s_flat[3]) / (double)n);
  }
  a8_gaussian<DEG, kAdam>(n, i, mean, scale, rot, sh, flags, g2d, conic_o, cam, dmean, dscale, drot, dopac, dsh, absgrad,
                          grad2d, tiles_touched, daccum, dcount, hw, hh, s_g + threadIdx.x);
  // each thread reads back only its own column: no barrier
  if (kAdam && i < n) adam_rows<K3>(F, n, i, s_g + threadIdx.x, gflat);
}

}  // namespace

cudaError_t launch_preprocess_bwd(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                                  pgsag_gaussian_grad* out, const float* g2d, cudaStream_t st,
                                  pgsag_adam_state* adam, const pgsag_adam_hparams* hp, double* flat,
                                  const uint32_t* skip) {
  const int n = g->n;
  AdamFused F{};
  F.skip = skip;
  if (adam) {
    F.P = adam_params(hp);
    F.mean = adam->mean; F.scale = adam->scale; F.rot = adam->rot; F.op = adam->opacity; F.sh = adam->sh;
    F.log_scale = adam->log_scale; F.logit_op = adam->logit_opacity; F.m = adam->m; F.v = adam->v;
    F.flat = flat;
    if (flat) {
      cudaError_t e = cudaMemsetAsync(flat, 0, sizeof(double), st);
      if (e != cudaSuccess) return e;
    }
  }
  CamB cb;
  cb.fx = cam->fx; cb.fy = cam->fy;
  for (int k = 0; k < 3; ++k) cb.C[k] = cam->C[k];
  for (int k = 0; k < 9; ++k) cb.R[k] = cam->R[k];
  cb.lx = (double)(1.3f * ((0.5f * (float)cam->width) / cam->fx));
  cb.ly = (double)(1.3f * ((0.5f * (float)cam->height) / cam->fy));
  {
    KTimer kt_(adam ? "A8_preprocess_bwd_adam" : "A8_preprocess_bwd", st);
    const int blocks = (n + 127) / 128;
    const float4* g2d4 = reinterpret_cast<const float4*>(g2d);
#define PGSAG_A8(DEG, AD)                                                                                    \
  preprocess_bwd_kernel<DEG, AD><<<blocks, 128, 0, st>>>(                                                  \
      n, g->mean, g->scale, g->rot, g->sh, p->flags, g2d4, reinterpret_cast<const float4*>(p->conic_o), cb,   \
      out->dmean, out->dscale, out->drot,         \
      out->dopacity, out->dsh, out->absgrad2d, out->grad2d, p->tiles_touched, out->densify_accum,          \
      out->densify_count, 0.5 * cam->width, 0.5 * cam->height, F)
    const int deg = g->sh_degree < 0 ? 0 : (g->sh_degree > 3 ? 3 : g->sh_degree);
    switch (deg * 2 + (adam ? 1 : 0)) {
      case 0: PGSAG_A8(0, false); break;
      case 1: PGSAG_A8(0, true); break;
      case 2: PGSAG_A8(1, false); break;
      case 3: PGSAG_A8(1, true); break;
      case 4: PGSAG_A8(2, false); break;
      case 5: PGSAG_A8(2, true); break;
      case 6: PGSAG_A8(3, false); break;
      default: PGSAG_A8(3, true); break;
    }
#undef PGSAG_A8
  }
  return cudaGetLastError();
}

}  // namespace pgsag
