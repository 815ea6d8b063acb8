// A8: per-Gaussian chain rule from A7's screen-space gradients to the 3D
// parameters (oracle O6), float64 arithmetic, one thread per Gaussian.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kG2 = 14;

// --------------------------------------------------------------------- A8
// Per-Gaussian chain rule in float64 (FP64 on B200 is ample for ~600 ops per
// Gaussian; the conic -> covariance -> Sigma chain amplifies rounding, so it is
// done in double from the double-accumulated 2D gradients).
struct CamB {
  double fx, fy, C[3], R[9], lx, ly;
};

template <int DEG>
__global__ void __launch_bounds__(256) preprocess_bwd_kernel(
    int n, const float* __restrict__ mean, const float* __restrict__ scale, const float* __restrict__ rot,
    const float* __restrict__ sh, const uint32_t* __restrict__ flags, const double* __restrict__ g2d, CamB cam,
    float* __restrict__ dmean, float* __restrict__ dscale, float* __restrict__ drot, float* __restrict__ dopac,
    float* __restrict__ dsh, float* __restrict__ absgrad, float* __restrict__ grad2d) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t fl = flags[i];
  if ((fl & PGSAG_F_LIVE) != PGSAG_F_LIVE) {
#pragma unroll
    for (int k = 0; k < 3; ++k) { dmean[(size_t)k * n + i] = 0.f; dscale[(size_t)k * n + i] = 0.f; }
#pragma unroll
    for (int k = 0; k < 4; ++k) drot[(size_t)k * n + i] = 0.f;
    dopac[i] = 0.f;
#pragma unroll
    for (int k = 0; k < 3 * K; ++k) dsh[(size_t)k * n + i] = 0.f;
    if (absgrad) absgrad[i] = 0.f;
    if (grad2d)
      for (int c = 0; c < kG2; ++c) grad2d[(size_t)c * n + i] = 0.f;
    return;
  }
  double gg[kG2];
#pragma unroll
  for (int c = 0; c < kG2; ++c) gg[c] = g2d[(size_t)c * n + i];
  if (grad2d) {
#pragma unroll
    for (int c = 0; c < kG2; ++c) grad2d[(size_t)c * n + i] = (float)gg[c];
  }
  const double* Rc = cam.R;
  const double t[3] = {(double)mean[i] - cam.C[0], (double)mean[n + i] - cam.C[1], (double)mean[2 * n + i] - cam.C[2]};
  double pc[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) pc[r] = Rc[3 * r] * t[0] + Rc[3 * r + 1] * t[1] + Rc[3 * r + 2] * t[2];
  const double x = pc[0], y = pc[1], z = pc[2];
  const double q0[4] = {rot[i], rot[n + i], rot[2 * n + i], rot[3 * n + i]};
  const double qn = sqrt(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
  const double w = q0[0] / qn, X = q0[1] / qn, Y = q0[2] / qn, Z = q0[3] / qn;
  double Rg[3][3];
  Rg[0][0] = 1. - 2. * (Y * Y + Z * Z); Rg[0][1] = 2. * (X * Y - w * Z); Rg[0][2] = 2. * (X * Z + w * Y);
  Rg[1][0] = 2. * (X * Y + w * Z); Rg[1][1] = 1. - 2. * (X * X + Z * Z); Rg[1][2] = 2. * (Y * Z - w * X);
  Rg[2][0] = 2. * (X * Z - w * Y); Rg[2][1] = 2. * (Y * Z + w * X); Rg[2][2] = 1. - 2. * (X * X + Y * Y);
  const double s[3] = {scale[i], scale[n + i], scale[2 * n + i]};
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
  for (int k = 0; k < 4; ++k) drot[(size_t)k * n + i] = (float)((dq[k] - qh[k] * qdot) / qn);
  // SH colour: rgb_c = max(0, sum_l Y_l(dir) sh_lc + 0.5)
  const double len = sqrt(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  const double il = 1.0 / len;
  const double dx = t[0] * il, dy = t[1] * il, dz = t[2] * il;
  const double xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yzp = dy * dz, xzp = dx * dz;
  const double c1 = 0.4886025119029199;
  const double c2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                        0.5462742152960396};
  const double c3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                        -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
  double Yb[16], GY[16][3];
  Yb[0] = 0.28209479177387814; GY[0][0] = 0.; GY[0][1] = 0.; GY[0][2] = 0.;
  Yb[1] = -c1 * dy; GY[1][0] = 0.; GY[1][1] = -c1; GY[1][2] = 0.;
  Yb[2] = c1 * dz; GY[2][0] = 0.; GY[2][1] = 0.; GY[2][2] = c1;
  Yb[3] = -c1 * dx; GY[3][0] = -c1; GY[3][1] = 0.; GY[3][2] = 0.;
  Yb[4] = c2[0] * xy; GY[4][0] = c2[0] * dy; GY[4][1] = c2[0] * dx; GY[4][2] = 0.;
  Yb[5] = c2[1] * yzp; GY[5][0] = 0.; GY[5][1] = c2[1] * dz; GY[5][2] = c2[1] * dy;
  Yb[6] = c2[2] * (2. * zz - xx - yy); GY[6][0] = -2. * c2[2] * dx; GY[6][1] = -2. * c2[2] * dy; GY[6][2] = 4. * c2[2] * dz;
  Yb[7] = c2[3] * xzp; GY[7][0] = c2[3] * dz; GY[7][1] = 0.; GY[7][2] = c2[3] * dx;
  Yb[8] = c2[4] * (xx - yy); GY[8][0] = 2. * c2[4] * dx; GY[8][1] = -2. * c2[4] * dy; GY[8][2] = 0.;
  Yb[9] = c3[0] * dy * (3. * xx - yy); GY[9][0] = 6. * c3[0] * xy; GY[9][1] = c3[0] * (3. * xx - 3. * yy); GY[9][2] = 0.;
  Yb[10] = c3[1] * xy * dz; GY[10][0] = c3[1] * yzp; GY[10][1] = c3[1] * xzp; GY[10][2] = c3[1] * xy;
  Yb[11] = c3[2] * dy * (4. * zz - xx - yy); GY[11][0] = -2. * c3[2] * xy; GY[11][1] = c3[2] * (4. * zz - xx - 3. * yy); GY[11][2] = 8. * c3[2] * yzp;
  Yb[12] = c3[3] * dz * (2. * zz - 3. * xx - 3. * yy); GY[12][0] = -6. * c3[3] * xzp; GY[12][1] = -6. * c3[3] * yzp; GY[12][2] = c3[3] * (6. * zz - 3. * xx - 3. * yy);
  Yb[13] = c3[4] * dx * (4. * zz - xx - yy); GY[13][0] = c3[4] * (4. * zz - 3. * xx - yy); GY[13][1] = -2. * c3[4] * xy; GY[13][2] = 8. * c3[4] * xzp;
  Yb[14] = c3[5] * dz * (xx - yy); GY[14][0] = 2. * c3[5] * xzp; GY[14][1] = -2. * c3[5] * yzp; GY[14][2] = c3[5] * (xx - yy);
  Yb[15] = c3[6] * dx * (xx - 3. * yy); GY[15][0] = c3[6] * (3. * xx - 3. * yy); GY[15][1] = -6. * c3[6] * xy; GY[15][2] = 0.;
  double dd0 = 0., dd1 = 0., dd2 = 0.;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double gc = (fl & (PGSAG_F_RGB_CLAMP0 << c)) ? 0. : gg[6 + c];
#pragma unroll
    for (int l = 0; l < K; ++l) {
      const double shv = sh[(size_t)(l * 3 + c) * n + i];
      dsh[(size_t)(l * 3 + c) * n + i] = (float)(Yb[l] * gc);
      const double f = shv * gc;
      dd0 += GY[l][0] * f; dd1 += GY[l][1] * f; dd2 += GY[l][2] * f;
    }
  }
  const double ddot = dx * dd0 + dy * dd1 + dz * dd2;
  dt[0] += (dd0 - dx * ddot) * il;
  dt[1] += (dd1 - dy * ddot) * il;
  dt[2] += (dd2 - dz * ddot) * il;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dmean[(size_t)k * n + i] = (float)dt[k];
    dscale[(size_t)k * n + i] = (float)ds[k];
  }
  dopac[i] = (float)gg[5];
  if (absgrad) absgrad[i] = (float)gg[13];
}

}  // namespace

cudaError_t launch_preprocess_bwd(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                                  pgsag_gaussian_grad* out, const double* g2d, cudaStream_t st) {
  const int n = g->n;
  CamB cb;
  cb.fx = cam->fx; cb.fy = cam->fy;
  for (int k = 0; k < 3; ++k) cb.C[k] = cam->C[k];
  for (int k = 0; k < 9; ++k) cb.R[k] = cam->R[k];
  cb.lx = (double)(1.3f * ((0.5f * (float)cam->width) / cam->fx));
  cb.ly = (double)(1.3f * ((0.5f * (float)cam->height) / cam->fy));
  {
    KTimer kt_("A8_preprocess_bwd", st);
    const int blocks = (n + 255) / 256;
#define PGSAG_A8(DEG)                                                                                         \
  preprocess_bwd_kernel<DEG><<<blocks, 256, 0, st>>>(n, g->mean, g->scale, g->rot, g->sh, p->flags, g2d, cb, \
                                                      out->dmean, out->dscale, out->drot, out->dopacity,      \
                                                      out->dsh, out->absgrad2d, out->grad2d)
    switch (g->sh_degree) {
      case 0: PGSAG_A8(0); break;
      case 1: PGSAG_A8(1); break;
      case 2: PGSAG_A8(2); break;
      default: PGSAG_A8(3); break;
    }
#undef PGSAG_A8
  }
  return cudaGetLastError();
}

}  // namespace pgsag
