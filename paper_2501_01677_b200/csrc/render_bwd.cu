// A7 (reverse-order backward compositor) and A8 (per-Gaussian chain rule) for sm_100a.
//
// P:82 "all the encoded parameters are optimized ... using differentiable
// rendering": the exact reverse mode of A6 (Eq. 1-4) with the forward's discrete
// decisions frozen (R16, R17).  Per pixel, walking the tile list backwards from
// the pixel's last blended entry:
//   T_i    = T_{i+1} / (1 - alpha_i)                       (recovered, T_end = A6's T)
//   dalpha = T_i (G . (F_i - S) - P (bg . gC))              F = (rgb, n_cam, d, 1)
//   dF_i   = alpha_i T_i G,   S <- alpha F + (1 - alpha) S,   P <- (1 - alpha) P
// then d(o, power) -> d(conic, mean2d).  Per entry, the warp's 14 partial
// gradients are butterfly-reduced and one lane issues the global atomics.
#include <cuda_runtime.h>
#include <stdint.h>

#include "alpha.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kG2 = 14;  // du dv dca dcb dcc dop drgb3 dncam3 ddist absgrad

struct BwdArgs {
  const float2* mean2d;
  const float4* conic_o;
  const float4* rgb_d;
  const float4* ncam;
  const uint32_t* vals;
  const uint32_t* ranges;
  const uint32_t* active;
  const uint32_t* n_active;
  const uint8_t* mask;
  Dims d;
  float fx, fy, cx, cy;
  float bg0, bg1, bg2;
  const float *N, *D, *T;
  const int32_t *g, *last;
  const float *dC, *dN, *dD, *dA, *dDep;
  float* g2d;  // [kG2][n]
  int n;
  unsigned long long* counters;
  uint32_t* work;
};

__device__ __forceinline__ float ld_or0(const float* p, size_t k) { return p ? __ldg(p + k) : 0.0f; }

template <bool kCount>
__global__ void __launch_bounds__(kTilePix) render_bwd_kernel(BwdArgs a) {
  __shared__ float2 s_xy[kTilePix];
  __shared__ float4 s_co[kTilePix];
  __shared__ float4 s_raw[kTilePix];  // (ca, cb, cc, o) unscaled
  __shared__ float4 s_cd[kTilePix];
  __shared__ float4 s_n[kTilePix];
  __shared__ uint32_t s_id[kTilePix];
  __shared__ uint32_t s_tile;
  __shared__ int s_maxlast;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t n_active = *a.n_active;
  const size_t HW = (size_t)a.d.W * a.d.H;
  unsigned long long cntV = 0;
  for (;;) {
    if (tid == 0) { s_tile = atomicAdd(a.work, 1u); s_maxlast = -1; }
    __syncthreads();
    const uint32_t widx = s_tile;
    if (widx >= n_active) break;
    const uint32_t tile = a.active[widx];
    const int ty = tile / a.d.TX, tx = tile - ty * a.d.TX;
    const int i = tx * kTile + (tid & (kTile - 1));
    const int j = ty * kTile + (tid >> 4);
    const bool inside = i < a.d.W && j < a.d.H;
    const size_t pix = (size_t)j * a.d.W + i;
    const bool masked = inside && a.mask[pix] != 0;
    const uint32_t rs = a.ranges[2 * tile];
    const float px = (float)i + 0.5f, py = (float)j + 0.5f;
    int mylast = -1;
    float Tcur = 1.0f;
    float G[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float bgdot = 0.f;
    if (masked) {
      mylast = a.last[pix];
      Tcur = a.T[pix];
      G[0] = ld_or0(a.dC, pix); G[1] = ld_or0(a.dC, HW + pix); G[2] = ld_or0(a.dC, 2 * HW + pix);
      G[3] = ld_or0(a.dN, pix); G[4] = ld_or0(a.dN, HW + pix); G[5] = ld_or0(a.dN, 2 * HW + pix);
      G[6] = ld_or0(a.dD, pix);
      G[7] = ld_or0(a.dA, pix);
      const float gDep = ld_or0(a.dDep, pix);
      // Eq. 4 prologue: Dep = D / (N . r), validity re-derived exactly as A6 did
      const float N0 = a.N[pix], N1 = a.N[HW + pix], N2 = a.N[2 * HW + pix];
      const float r0 = __fdiv_rn(__fsub_rn(px, a.cx), a.fx), r1 = __fdiv_rn(__fsub_rn(py, a.cy), a.fy);
      const float den = __fadd_rn(__fadd_rn(__fmul_rn(N0, r0), __fmul_rn(N1, r1)), N2);
      if (a.g[pix] > 0 && fabsf(den) > 1e-6f) {
        const float inv = 1.0f / den;
        G[6] += gDep * inv;
        const float c = gDep * a.D[pix] * inv * inv;
        G[3] -= c * r0; G[4] -= c * r1; G[5] -= c;
      }
      bgdot = a.bg0 * G[0] + a.bg1 * G[1] + a.bg2 * G[2];
      if (mylast >= 0) atomicMax(&s_maxlast, mylast);
    }
    __syncthreads();
    const int maxlast = s_maxlast;
    float S[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float P = 1.0f;
    for (int bhi = maxlast + 1; bhi > (int)rs; bhi -= kTilePix) {
      const int blo = max((int)rs, bhi - kTilePix);
      const int k = blo + tid;
      __syncthreads();  // previous batch fully consumed
      if (k < bhi) {
        const uint32_t id = a.vals[k];
        s_id[tid] = id;
        s_xy[tid] = a.mean2d[id];
        const float4 co = a.conic_o[id];
        s_raw[tid] = co;
        s_co[tid] = scaled_conic(co);
        s_cd[tid] = a.rgb_d[id];
        s_n[tid] = a.ncam[id];
      }
      __syncthreads();
      for (int q = bhi - blo - 1; q >= 0; --q) {
        const int kk = blo + q;
        bool contrib = kk <= mylast;  // false for masked-out pixels (mylast = -1)
        float alpha = 0.f, rho = 0.f, dx = 0.f, dy = 0.f;
        const float2 xy = s_xy[q];
        const float4 sc = s_co[q];
        if (contrib) {
          dx = px - xy.x; dy = py - xy.y;
          const float p2 = power2(sc, dx, dy);
          if (p2 > 0.0f) {
            contrib = false;
          } else {
            rho = ex2_approx(p2);
            alpha = fminf(kAlphaMax, __fmul_rn(sc.w, rho));
            if (alpha < kAlphaMin) contrib = false;
          }
          if (kCount) ++cntV;
        }
        if (!__any_sync(0xffffffffu, contrib)) continue;
        float v[kG2];
#pragma unroll
        for (int c = 0; c < kG2; ++c) v[c] = 0.f;
        if (contrib) {
          const float4 cd = s_cd[q];
          const float4 nn = s_n[q];
          const float4 raw = s_raw[q];
          const float om = 1.0f - alpha;
          const float Ti = Tcur / om;
          const float F[8] = {cd.x, cd.y, cd.z, nn.x, nn.y, nn.z, cd.w, 1.0f};
          float dot = 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) dot += G[c] * (F[c] - S[c]);
          const float dalpha = Ti * (dot - P * bgdot);
          const float w = alpha * Ti;
          v[6] = w * G[0]; v[7] = w * G[1]; v[8] = w * G[2];
          v[9] = w * G[3]; v[10] = w * G[4]; v[11] = w * G[5];
          v[12] = w * G[6];
#pragma unroll
          for (int c = 0; c < 8; ++c) S[c] = alpha * F[c] + om * S[c];
          P *= om;
          Tcur = Ti;
          float dpow = 0.f;
          if (__fmul_rn(raw.w, rho) <= kAlphaMax) {
            v[5] = rho * dalpha;
            dpow = alpha * dalpha;
          }
          v[2] = -0.5f * dx * dx * dpow;
          v[3] = -dx * dy * dpow;
          v[4] = -0.5f * dy * dy * dpow;
          v[0] = (raw.x * dx + raw.y * dy) * dpow;
          v[1] = (raw.y * dx + raw.z * dy) * dpow;
          v[13] = fabsf(v[0]) + fabsf(v[1]);
        }
#pragma unroll
        for (int c = 0; c < kG2; ++c) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
        }
        if (lane == 0) {
          const uint32_t id = s_id[q];
#pragma unroll
          for (int c = 0; c < kG2; ++c) atomicAdd(a.g2d + (size_t)c * a.n + id, v[c]);
        }
      }
    }
    __syncthreads();
  }
  if (kCount) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cntV += __shfl_xor_sync(0xffffffffu, cntV, o);
    if (lane == 0 && cntV) atomicAdd(a.counters + 2, cntV);
  }
}

// --------------------------------------------------------------------- A8
struct CamB {
  float fx, fy, C[3], R[9], lx, ly;
};

__constant__ float kC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                             -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                             0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                             -0.5900435899266435f};

__global__ void __launch_bounds__(256) preprocess_bwd_kernel(
    int n, int deg, const float* __restrict__ mean, const float* __restrict__ scale,
    const float* __restrict__ rot, const float* __restrict__ sh, const uint32_t* __restrict__ flags,
    const float* __restrict__ g2d, CamB cam, float* __restrict__ dmean, float* __restrict__ dscale,
    float* __restrict__ drot, float* __restrict__ dopac, float* __restrict__ dsh, float* __restrict__ absgrad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int K = (deg + 1) * (deg + 1);
  const uint32_t fl = flags[i];
  if ((fl & PGSAG_F_LIVE) != PGSAG_F_LIVE) {
    for (int k = 0; k < 3; ++k) { dmean[(size_t)k * n + i] = 0.f; dscale[(size_t)k * n + i] = 0.f; }
    for (int k = 0; k < 4; ++k) drot[(size_t)k * n + i] = 0.f;
    dopac[i] = 0.f;
    for (int k = 0; k < 3 * K; ++k) dsh[(size_t)k * n + i] = 0.f;
    if (absgrad) absgrad[i] = 0.f;
    return;
  }
  float gg[kG2];
#pragma unroll
  for (int c = 0; c < kG2; ++c) gg[c] = g2d[(size_t)c * n + i];
  const float* Rc = cam.R;
  const float t[3] = {mean[i] - cam.C[0], mean[n + i] - cam.C[1], mean[2 * n + i] - cam.C[2]};
  float pc[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) pc[r] = Rc[3 * r] * t[0] + Rc[3 * r + 1] * t[1] + Rc[3 * r + 2] * t[2];
  const float x = pc[0], y = pc[1], z = pc[2];
  const float q0[4] = {rot[i], rot[n + i], rot[2 * n + i], rot[3 * n + i]};
  const float qn = sqrtf(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
  const float w = q0[0] / qn, X = q0[1] / qn, Y = q0[2] / qn, Z = q0[3] / qn;
  float Rg[3][3];
  Rg[0][0] = 1.f - 2.f * (Y * Y + Z * Z); Rg[0][1] = 2.f * (X * Y - w * Z); Rg[0][2] = 2.f * (X * Z + w * Y);
  Rg[1][0] = 2.f * (X * Y + w * Z); Rg[1][1] = 1.f - 2.f * (X * X + Z * Z); Rg[1][2] = 2.f * (Y * Z - w * X);
  Rg[2][0] = 2.f * (X * Z - w * Y); Rg[2][1] = 2.f * (Y * Z + w * X); Rg[2][2] = 1.f - 2.f * (X * X + Y * Y);
  const float s[3] = {scale[i], scale[n + i], scale[2 * n + i]};
  float Mg[3][3], Sig[3][3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Mg[r][c] = Rg[r][c] * s[c];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) Sig[r][c] = Mg[r][0] * Mg[c][0] + Mg[r][1] * Mg[c][1] + Mg[r][2] * Mg[c][2];
  const bool clx = fl & PGSAG_F_CLAMP_X, cly = fl & PGSAG_F_CLAMP_Y;
  const float xz = x / z, yz = y / z;
  const float cxz = clx ? fminf(fmaxf(xz, -cam.lx), cam.lx) : xz;
  const float cyz = cly ? fminf(fmaxf(yz, -cam.ly), cam.ly) : yz;
  const float J00 = cam.fx / z, J02 = -cam.fx * cxz / z, J11 = cam.fy / z, J12 = -cam.fy * cyz / z;
  float Tm[2][3];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    Tm[0][b] = J00 * Rc[b] + J02 * Rc[6 + b];
    Tm[1][b] = J11 * Rc[3 + b] + J12 * Rc[6 + b];
  }
  float STm[2][3];  // Sig Tm_a^T
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int k = 0; k < 3; ++k) STm[a][k] = Sig[k][0] * Tm[a][0] + Sig[k][1] * Tm[a][1] + Sig[k][2] * Tm[a][2];
  const float A = Tm[0][0] * STm[0][0] + Tm[0][1] * STm[0][1] + Tm[0][2] * STm[0][2] + 0.3f;
  const float B = Tm[0][0] * STm[1][0] + Tm[0][1] * STm[1][1] + Tm[0][2] * STm[1][2];
  const float Cc = Tm[1][0] * STm[1][0] + Tm[1][1] * STm[1][1] + Tm[1][2] * STm[1][2] + 0.3f;
  const float det = A * Cc - B * B;
  const float id2 = 1.0f / (det * det);
  const float dca = gg[2], dcb = gg[3], dcc = gg[4];
  const float dA = (-Cc * Cc * dca + B * Cc * dcb - B * B * dcc) * id2;
  const float dC = (-B * B * dca + A * B * dcb - A * A * dcc) * id2;
  const float dB = (2.f * B * Cc * dca - (A * Cc + B * B) * dcb + 2.f * A * B * dcc) * id2;
  // cov_ab = Tm_a Sig Tm_b^T
  float dSig[3][3];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int l = 0; l < 3; ++l)
      dSig[k][l] = dA * Tm[0][k] * Tm[0][l] + dC * Tm[1][k] * Tm[1][l] + dB * Tm[0][k] * Tm[1][l];
  float dTm[2][3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dTm[0][k] = 2.f * dA * STm[0][k] + dB * STm[1][k];
    dTm[1][k] = 2.f * dC * STm[1][k] + dB * STm[0][k];
  }
  // Tm = J R_c -> dJ = dTm R_c^T (only J00, J02, J11, J12 are variables)
  const float dJ00 = dTm[0][0] * Rc[0] + dTm[0][1] * Rc[1] + dTm[0][2] * Rc[2];
  const float dJ02 = dTm[0][0] * Rc[6] + dTm[0][1] * Rc[7] + dTm[0][2] * Rc[8];
  const float dJ11 = dTm[1][0] * Rc[3] + dTm[1][1] * Rc[4] + dTm[1][2] * Rc[5];
  const float dJ12 = dTm[1][0] * Rc[6] + dTm[1][1] * Rc[7] + dTm[1][2] * Rc[8];
  const float iz = 1.0f / z, iz2 = iz * iz, iz3 = iz2 * iz;
  float dp0 = 0.f, dp1 = 0.f, dp2 = 0.f;
  dp2 += -cam.fx * iz2 * dJ00 - cam.fy * iz2 * dJ11;
  if (!clx) { dp0 += -cam.fx * iz2 * dJ02; dp2 += 2.f * cam.fx * x * iz3 * dJ02; }
  else { dp2 += cam.fx * cxz * iz2 * dJ02; }
  if (!cly) { dp1 += -cam.fy * iz2 * dJ12; dp2 += 2.f * cam.fy * y * iz3 * dJ12; }
  else { dp2 += cam.fy * cyz * iz2 * dJ12; }
  // mean2d (u = fx x/z + cx, v = fy y/z + cy)
  const float du = gg[0], dv = gg[1];
  dp0 += cam.fx * iz * du;
  dp1 += cam.fy * iz * dv;
  dp2 += -(cam.fx * x * du + cam.fy * y * dv) * iz2;
  float dt[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) dt[k] = Rc[k] * dp0 + Rc[3 + k] * dp1 + Rc[6 + k] * dp2;
  // Sigma = Mg Mg^T -> dMg = (dSig + dSig^T) Mg;  Mg = Rg diag(s)
  float dRg[3][3], ds[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      float acc = 0.f;
#pragma unroll
      for (int l = 0; l < 3; ++l) acc += (dSig[k][l] + dSig[l][k]) * Mg[l][m];
      ds[m] += acc * Rg[k][m];
      dRg[k][m] = acc * s[m];
    }
  // normal n = sg Rg[:,ax]; n_cam = R_c n; d = n . t
  const int ax = (fl >> PGSAG_F_AXIS_SHIFT) & 3;
  const float sg = (fl & PGSAG_F_NFLIP) ? -1.f : 1.f;
  const float nv[3] = {sg * Rg[0][ax], sg * Rg[1][ax], sg * Rg[2][ax]};
  const float ddist = gg[12];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float dn = Rc[k] * gg[9] + Rc[3 + k] * gg[10] + Rc[6 + k] * gg[11] + t[k] * ddist;
    dt[k] += nv[k] * ddist;
    dRg[k][ax] += sg * dn;
  }
  // Rg(q-hat) -> d q-hat
  float dq[4] = {0.f, 0.f, 0.f, 0.f};
  dq[2] += -4.f * Y * dRg[0][0]; dq[3] += -4.f * Z * dRg[0][0];
  dq[1] += 2.f * Y * dRg[0][1]; dq[2] += 2.f * X * dRg[0][1]; dq[0] += -2.f * Z * dRg[0][1]; dq[3] += -2.f * w * dRg[0][1];
  dq[1] += 2.f * Z * dRg[0][2]; dq[3] += 2.f * X * dRg[0][2]; dq[0] += 2.f * Y * dRg[0][2]; dq[2] += 2.f * w * dRg[0][2];
  dq[1] += 2.f * Y * dRg[1][0]; dq[2] += 2.f * X * dRg[1][0]; dq[0] += 2.f * Z * dRg[1][0]; dq[3] += 2.f * w * dRg[1][0];
  dq[1] += -4.f * X * dRg[1][1]; dq[3] += -4.f * Z * dRg[1][1];
  dq[2] += 2.f * Z * dRg[1][2]; dq[3] += 2.f * Y * dRg[1][2]; dq[0] += -2.f * X * dRg[1][2]; dq[1] += -2.f * w * dRg[1][2];
  dq[1] += 2.f * Z * dRg[2][0]; dq[3] += 2.f * X * dRg[2][0]; dq[0] += -2.f * Y * dRg[2][0]; dq[2] += -2.f * w * dRg[2][0];
  dq[2] += 2.f * Z * dRg[2][1]; dq[3] += 2.f * Y * dRg[2][1]; dq[0] += 2.f * X * dRg[2][1]; dq[1] += 2.f * w * dRg[2][1];
  dq[1] += -4.f * X * dRg[2][2]; dq[2] += -4.f * Y * dRg[2][2];
  const float qh[4] = {w, X, Y, Z};
  const float qdot = qh[0] * dq[0] + qh[1] * dq[1] + qh[2] * dq[2] + qh[3] * dq[3];
#pragma unroll
  for (int k = 0; k < 4; ++k) drot[(size_t)k * n + i] = (dq[k] - qh[k] * qdot) / qn;
  // SH colour: rgb_c = max(0, sum_l Y_l(dir) sh_lc + 0.5)
  const float len = sqrtf(t[0] * t[0] + t[1] * t[1] + t[2] * t[2]);
  const float il = 1.0f / len;
  const float dx = t[0] * il, dy = t[1] * il, dz = t[2] * il;
  const float xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yzp = dy * dz, xzp = dx * dz;
  float Yb[16];
  float GY[16][3];
  Yb[0] = 0.28209479177387814f; GY[0][0] = 0.f; GY[0][1] = 0.f; GY[0][2] = 0.f;
  const float c1 = 0.4886025119029199f;
  Yb[1] = -c1 * dy; GY[1][0] = 0.f; GY[1][1] = -c1; GY[1][2] = 0.f;
  Yb[2] = c1 * dz; GY[2][0] = 0.f; GY[2][1] = 0.f; GY[2][2] = c1;
  Yb[3] = -c1 * dx; GY[3][0] = -c1; GY[3][1] = 0.f; GY[3][2] = 0.f;
  Yb[4] = kC2[0] * xy; GY[4][0] = kC2[0] * dy; GY[4][1] = kC2[0] * dx; GY[4][2] = 0.f;
  Yb[5] = kC2[1] * yzp; GY[5][0] = 0.f; GY[5][1] = kC2[1] * dz; GY[5][2] = kC2[1] * dy;
  Yb[6] = kC2[2] * (2.f * zz - xx - yy); GY[6][0] = -2.f * kC2[2] * dx; GY[6][1] = -2.f * kC2[2] * dy; GY[6][2] = 4.f * kC2[2] * dz;
  Yb[7] = kC2[3] * xzp; GY[7][0] = kC2[3] * dz; GY[7][1] = 0.f; GY[7][2] = kC2[3] * dx;
  Yb[8] = kC2[4] * (xx - yy); GY[8][0] = 2.f * kC2[4] * dx; GY[8][1] = -2.f * kC2[4] * dy; GY[8][2] = 0.f;
  Yb[9] = kC3[0] * dy * (3.f * xx - yy); GY[9][0] = 6.f * kC3[0] * xy; GY[9][1] = kC3[0] * (3.f * xx - 3.f * yy); GY[9][2] = 0.f;
  Yb[10] = kC3[1] * xy * dz; GY[10][0] = kC3[1] * yzp; GY[10][1] = kC3[1] * xzp; GY[10][2] = kC3[1] * xy;
  Yb[11] = kC3[2] * dy * (4.f * zz - xx - yy); GY[11][0] = -2.f * kC3[2] * xy; GY[11][1] = kC3[2] * (4.f * zz - xx - 3.f * yy); GY[11][2] = 8.f * kC3[2] * yzp;
  Yb[12] = kC3[3] * dz * (2.f * zz - 3.f * xx - 3.f * yy); GY[12][0] = -6.f * kC3[3] * xzp; GY[12][1] = -6.f * kC3[3] * yzp; GY[12][2] = kC3[3] * (6.f * zz - 3.f * xx - 3.f * yy);
  Yb[13] = kC3[4] * dx * (4.f * zz - xx - yy); GY[13][0] = kC3[4] * (4.f * zz - 3.f * xx - yy); GY[13][1] = -2.f * kC3[4] * xy; GY[13][2] = 8.f * kC3[4] * xzp;
  Yb[14] = kC3[5] * dz * (xx - yy); GY[14][0] = 2.f * kC3[5] * xzp; GY[14][1] = -2.f * kC3[5] * yzp; GY[14][2] = kC3[5] * (xx - yy);
  Yb[15] = kC3[6] * dx * (xx - 3.f * yy); GY[15][0] = kC3[6] * (3.f * xx - 3.f * yy); GY[15][1] = -6.f * kC3[6] * xy; GY[15][2] = 0.f;
  float dd0 = 0.f, dd1 = 0.f, dd2 = 0.f;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const float gc = (fl & (PGSAG_F_RGB_CLAMP0 << c)) ? 0.f : gg[6 + c];
    for (int l = 0; l < K; ++l) {
      const float shv = sh[(size_t)(l * 3 + c) * n + i];
      dsh[(size_t)(l * 3 + c) * n + i] = Yb[l] * gc;
      const float f = shv * gc;
      dd0 += GY[l][0] * f; dd1 += GY[l][1] * f; dd2 += GY[l][2] * f;
    }
  }
  const float ddot = dx * dd0 + dy * dd1 + dz * dd2;
  dt[0] += (dd0 - dx * ddot) * il;
  dt[1] += (dd1 - dy * ddot) * il;
  dt[2] += (dd2 - dz * ddot) * il;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dmean[(size_t)k * n + i] = dt[k];
    dscale[(size_t)k * n + i] = ds[k];
  }
  dopac[i] = gg[5];
  if (absgrad) absgrad[i] = gg[13];
}

int bwd_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, render_bwd_kernel<false>, kTilePix, 0);
    grid = sms * (occ > 0 ? occ : 1);
  }
  return grid;
}

}  // namespace

cudaError_t launch_render_bwd(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                              const pgsag_bins* bins, const pgsag_tilemask* tm, const Dims& d,
                              const uint8_t* mask, const float bg[3], const pgsag_image* fwd,
                              const pgsag_image_grad* dL, pgsag_gaussian_grad* out, float* g2d,
                              uint32_t* work_counter, cudaStream_t st) {
  const int n = g->n;
  if (n == 0) return cudaSuccess;
  cudaMemsetAsync(g2d, 0, sizeof(float) * kG2 * (size_t)n, st);
  BwdArgs a;
  a.mean2d = reinterpret_cast<const float2*>(p->mean2d);
  a.conic_o = reinterpret_cast<const float4*>(p->conic_o);
  a.rgb_d = reinterpret_cast<const float4*>(p->rgb_d);
  a.ncam = reinterpret_cast<const float4*>(p->ncam);
  a.vals = bins->vals;
  a.ranges = bins->ranges;
  a.active = tm->active;
  a.n_active = tm->n_active;
  a.mask = mask;
  a.d = d;
  a.fx = cam->fx; a.fy = cam->fy; a.cx = cam->cx; a.cy = cam->cy;
  a.bg0 = bg[0]; a.bg1 = bg[1]; a.bg2 = bg[2];
  a.N = fwd->N; a.D = fwd->D; a.T = fwd->T; a.g = fwd->g; a.last = fwd->last;
  a.dC = dL->dC; a.dN = dL->dN; a.dD = dL->dD; a.dA = dL->dA; a.dDep = dL->dDep;
  a.g2d = g2d;
  a.n = n;
  a.counters = fwd->counters;
  a.work = work_counter;
  const int grid = min(bwd_grid(), d.TX * d.TY);
  if (fwd->counters)
    {
      KTimer kt_("A7_render_bwd", st);
      render_bwd_kernel<true><<<grid, kTilePix, 0, st>>>(a);
    }
  else
    {
      KTimer kt_("A7_render_bwd", st);
      render_bwd_kernel<false><<<grid, kTilePix, 0, st>>>(a);
    }
  CamB cb;
  cb.fx = cam->fx; cb.fy = cam->fy;
  for (int k = 0; k < 3; ++k) cb.C[k] = cam->C[k];
  for (int k = 0; k < 9; ++k) cb.R[k] = cam->R[k];
  cb.lx = 1.3f * ((0.5f * (float)cam->width) / cam->fx);
  cb.ly = 1.3f * ((0.5f * (float)cam->height) / cam->fy);
  {
    KTimer kt_("A8_preprocess_bwd", st);
    preprocess_bwd_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, g->sh_degree, g->mean, g->scale, g->rot, g->sh,
                                                           p->flags, g2d, cb, out->dmean, out->dscale, out->drot,
                                                           out->dopacity, out->dsh, out->absgrad2d);
  }
  return cudaGetLastError();
}

}  // namespace pgsag
