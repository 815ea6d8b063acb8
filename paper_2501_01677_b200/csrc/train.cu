// NEXT-3: the per-sub-region training step around the rasterizer (Eq. 10-11):
// the masked photometric loss L_rgb = 0.8 L1 + 0.2 (1 - SSIM) on the RBM pixels (R28),
// the flattening loss L_s = mean_i min(s_i) (R29) fused into an Adam update of the raw
// parameters (log-scale, logit-opacity; R30).  All HBM-bound stencils / elementwise.
//
// SSIM (Wang et al.): per channel, x = C m, y = I m (zero off the mask), 11x11 Gaussian
// window (sigma 1.5, zero padding), mu = G*x, sigma^2 = G*x^2 - mu^2, sigma_xy = G*(xy) - mu_x mu_y,
// S = (2 mu_x mu_y + C1)(2 sigma_xy + C2) / ((mu_x^2 + mu_y^2 + C1)(sigma_x^2 + sigma_y^2 + C2)).
// Backward: with A' = dS/dmu_x - 2 mu_x dS/dsigma_x^2 - mu_y dS/dsigma_xy, B = dS/dsigma_x^2,
// Cc = dS/dsigma_xy at every mask pixel (zero elsewhere), dS_mean/dx_q is
// k ((G*A')_q + 2 x_q (G*B)_q + y_q (G*Cc)_q) — three more separable blurs.
// Float32 throughout, with two shifts that keep the cancellations small (see the kernels):
// error bound and tolerance in DESIGN.md (R28).
// Tiles: forward 32 x 32 outputs per CTA (42 x 42 halo), backward 32 x 16 (42 x 26 halo), 256
// threads; separable passes (horizontal into shared memory, then vertical).
#include <cuda_runtime.h>
#include <stdint.h>

#include "adam.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kTW = 32, kTH = 16, kR = 5, kIW = kTW + 2 * kR, kIH = kTH + 2 * kR;
constexpr float kC1 = 0.01f * 0.01f, kC2 = 0.03f * 0.03f;

// Window weights g[k] = exp(-k^2 / 4.5) / sum (sigma 1.5), computed in double, rounded once.
__device__ __forceinline__ void window(float (&g)[2 * kR + 1]) {
  double w[2 * kR + 1], s = 0.0;
#pragma unroll
  for (int k = -kR; k <= kR; ++k) {
    w[k + kR] = exp(-(double)(k * k) / 4.5);
    s += w[k + kR];
  }
#pragma unroll
  for (int k = 0; k <= 2 * kR; ++k) g[k] = (float)(w[k] / s);
}

// Shift used by the backward combination: dS/dx_q = sum_p G [a_p + 2 b_p (x_q - mu_x,p) + c_p (y_q - mu_y,p)]
// holds with x_q - mu = (x_q - kShift) - (mu - kShift) for any constant, which keeps the float32
// cancellation between the two blurred terms small for images in [0, 1].
constexpr float kShift = 0.5f;

struct RgbArgs {
  const float* C;     // [3][H][W] rendered
  const float* I;     // [3][H][W] target
  const uint8_t* mask;
  int W, H;
  float weight;       // scale of dC
  float* abc;         // [3 ch][3][H][W] SSIM partials (A', B, Cc) at mask pixels
  double* loss;       // [6]: L, L1, S, sum|C-I|, sum S, mask pixels
  float* dC;
};

// true if any pixel of the CTA's 32x16 output tile is in the mask; also returns the mask bits
// of this thread's two output pixels (column tx, rows 2 ty and 2 ty + 1)
__device__ __forceinline__ bool tile_has_mask(const RgbArgs& A, int x, int y0, bool& m0, bool& m1) {
  m0 = x < A.W && y0 < A.H && __ldg(A.mask + (size_t)y0 * A.W + x);
  m1 = x < A.W && y0 + 1 < A.H && __ldg(A.mask + (size_t)(y0 + 1) * A.W + x);
  return __syncthreads_or(m0 || m1);
}

template <int K>
__device__ __forceinline__ void block_sum(float (&v)[K], float (*s_red)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) s_red[threadIdx.x >> 5][k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    v[k] = 0.f;
    for (int w = 0; w < 8; ++w) v[k] += s_red[w][k];
  }
}

// Shared-memory planes (row stride of the halo planes padded to 44 so that every row starts
// 16-byte aligned).  Pairs of quantities that are filtered identically are interleaved as
// float2 and filtered with packed FP32x2 instructions (FFMA2 / FMUL2 with a broadcast weight):
// forward (x, y) per channel and the horizontal-pass pairs (mu_x, mu_y), (E x^2, E y^2);
// backward (A', B).  Horizontal pass: one task = 4 adjacent output columns of one row
// (208 tasks, 14 samples from registers); vertical pass: each thread = 2 adjacent output rows
// of one column (12 samples).
constexpr int kIWp = 44;
constexpr int kPlane = kIH * kIWp, kHPlane = kIH * kTW;
constexpr int kBwdSmem = (3 * 3 * kPlane + 2 * kHPlane + kHPlane) * 4;

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ void load16x2(const float2* row, float2 (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 t = reinterpret_cast<const float4*>(row)[q];
    v[2 * q] = f2(t.x, t.y);
    v[2 * q + 1] = f2(t.z, t.w);
  }
}

__device__ __forceinline__ void load16(const float* row, float (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float4 t = reinterpret_cast<const float4*>(row)[q];
    v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
  }
}

__device__ __forceinline__ void store4x2(float2* row, const float2 (&v)[4]) {
  reinterpret_cast<float4*>(row)[0] = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
  reinterpret_cast<float4*>(row)[1] = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
}

__device__ __forceinline__ void store4(float* row, const float (&v)[4]) {
  *reinterpret_cast<float4*>(row) = make_float4(v[0], v[1], v[2], v[3]);
}

// Forward: window statistics in float32 on values shifted by the CTA's mean (every sample of the
// zero-padded, zero-masked input is shifted, so mu = c + G*(x - c) and the (co)variances are the
// shifted second moments minus the shifted means' products -- the cancellation in
// sigma^2 = E[x^2] - mu^2 is taken relative to the local mean instead of to 0).  One CTA = one 32x32
// output tile (the 42x42 halo: 1.72 input positions per output; a 32x16 tile measured 0.47 vs 0.44 ms
// on a C4 view), the channels one after the other, each loading its own halo (41.7 KB of shared
// memory); horizontal pass into shared memory, then a vertical pass of four output rows per thread
// from 14 rows.  The window weights come from the host (kernel parameters).
constexpr int kTW2 = 32, kTH2 = 32, kIW2 = kTW2 + 2 * kR, kIH2 = kTH2 + 2 * kR, kIWp2 = 44;
constexpr int kHalo2 = kIH2 * kIW2, kHIt2 = (kHalo2 + 255) / 256;
constexpr int kPlane2 = kIH2 * kIWp2, kHPlane2 = kIH2 * kTW2;
constexpr int kFwdSmem2 = (2 * kPlane2 + 2 * 2 * kHPlane2 + kHPlane2) * 4;

struct Win {
  float g[2 * kR + 1];
};

__global__ void __launch_bounds__(256, 4) rgb_fwd2_kernel(RgbArgs A, Win win) {
  extern __shared__ float4 smem_f4[];
  float2* s_in = reinterpret_cast<float2*>(smem_f4);            // (x, y) of the current channel
  float2* s_h2 = s_in + kPlane2;                                // [2]: (mu_x, mu_y), (E x^2, E y^2)
  float* s_h1 = reinterpret_cast<float*>(s_h2 + 2 * kHPlane2);  // E xy
  __shared__ float s_red[8][6];
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int bx = blockIdx.x * kTW2, by = blockIdx.y * kTH2;
  const int x = bx + tx, y0 = by + 4 * ty;
  bool m[4], any = false;
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    m[h] = x < A.W && y0 + h < A.H && __ldg(A.mask + (size_t)(y0 + h) * A.W + x);
    any = any || m[h];
  }
  if (!__syncthreads_or(any)) return;
  const size_t HW = (size_t)A.W * A.H;
  float g[2 * kR + 1];
#pragma unroll
  for (int k = 0; k <= 2 * kR; ++k) g[k] = win.g[k];
  float acc[3] = {0.f, 0.f, 0.f};  // sum |C - I|, sum S, count
#pragma unroll 1
  for (int ch = 0; ch < 3; ++ch) {
    // this channel's halo: every load first, then the shared stores and the sums for the shift
    float2 hv[kHIt2];
#pragma unroll
    for (int it = 0; it < kHIt2; ++it) {
      const int k = tid + 256 * it;
      const int r = k / kIW2, c = k - r * kIW2;
      const int gy = by - kR + r, gx = bx - kR + c;
      hv[it] = f2(0.f, 0.f);
      if (k < kHalo2 && gx >= 0 && gy >= 0 && gx < A.W && gy < A.H) {
        const size_t p = (size_t)gy * A.W + gx;
        const uint8_t mk = __ldg(A.mask + p);
        const float cv = __ldg(A.C + ch * HW + p), iv = __ldg(A.I + ch * HW + p);
        if (mk) hv[it] = f2(cv, iv);
      }
    }
    float sums[2] = {0.f, 0.f};
    if (ch) __syncthreads();  // the previous channel's passes are done with s_in / s_h
#pragma unroll
    for (int it = 0; it < kHIt2; ++it) {
      const int k = tid + 256 * it;
      if (k < kHalo2) {
        const int r = k / kIW2, c = k - r * kIW2;
        s_in[r * kIWp2 + c] = hv[it];
        sums[0] += hv[it].x;
        sums[1] += hv[it].y;
      }
    }
    block_sum<2>(sums, reinterpret_cast<float (*)[2]>(s_red));  // contains the barrier publishing s_in
    const float cx = sums[0] * (1.0f / (kIH2 * kIW2)), cy = sums[1] * (1.0f / (kIH2 * kIW2));
    // horizontal pass: 42 rows x 8 tasks of 4 adjacent output columns
    for (int t = tid; t < kIH2 * (kTW2 / 4); t += 256) {
      const int r = t >> 3, c0 = 4 * (t & 7);
      float2 v[16], sq[14];
      float pr[14];
      load16x2(s_in + r * kIWp2 + c0, v);
#pragma unroll
      for (int k = 0; k < 14; ++k) {
        v[k] = __fadd2_rn(v[k], f2(-cx, -cy));
        sq[k] = __fmul2_rn(v[k], v[k]);
        pr[k] = v[k].x * v[k].y;
      }
      float2 ab[4], q2[4];
      float xy[4];
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        ab[o] = q2[o] = f2(0.f, 0.f);
        xy[o] = 0.f;
#pragma unroll
        for (int k = 0; k <= 2 * kR; ++k) {
          ab[o] = __ffma2_rn(f2(g[k], g[k]), v[o + k], ab[o]);
          q2[o] = __ffma2_rn(f2(g[k], g[k]), sq[o + k], q2[o]);
          xy[o] = fmaf(g[k], pr[o + k], xy[o]);
        }
      }
      store4x2(s_h2 + r * kTW2 + c0, ab);
      store4x2(s_h2 + kHPlane2 + r * kTW2 + c0, q2);
      store4(s_h1 + r * kTW2 + c0, xy);
    }
    __syncthreads();
    // vertical pass: four output rows per thread from 14 rows, one quantity group at a time
    float2 ab[4], q2[4];
    float exy[4];
    {
      float2 col[14];
#pragma unroll
      for (int k = 0; k < 14; ++k) col[k] = s_h2[(4 * ty + k) * kTW2 + tx];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        ab[h] = f2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k <= 2 * kR; ++k) ab[h] = __ffma2_rn(f2(g[k], g[k]), col[k + h], ab[h]);
      }
#pragma unroll
      for (int k = 0; k < 14; ++k) col[k] = s_h2[kHPlane2 + (4 * ty + k) * kTW2 + tx];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        q2[h] = f2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k <= 2 * kR; ++k) q2[h] = __ffma2_rn(f2(g[k], g[k]), col[k + h], q2[h]);
      }
      float cxy[14];
#pragma unroll
      for (int k = 0; k < 14; ++k) cxy[k] = s_h1[(4 * ty + k) * kTW2 + tx];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        exy[h] = 0.f;
#pragma unroll
        for (int k = 0; k <= 2 * kR; ++k) exy[h] = fmaf(g[k], cxy[k + h], exy[h]);
      }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      if (!m[h]) continue;
      const float ax = ab[h].x, ay = ab[h].y;
      const float sxx = fmaf(-ax, ax, q2[h].x), syy = fmaf(-ay, ay, q2[h].y), sxy_ = fmaf(-ax, ay, exy[h]);
      const float mx = cx + ax, my = cy + ay;
      const float n1 = 2.f * mx * my + kC1, n2 = 2.f * sxy_ + kC2;
      const float d1 = mx * mx + my * my + kC1, d2 = sxx + syy + kC2;
      const float id = __fdividef(1.f, d1 * d2);
      const float s = n1 * n2 * id;
      const float dmx = 2.f * (my * n2 * id - __fdividef(mx * s, d1));
      const float dsxx = -__fdividef(s, d2), dsxy = 2.f * n1 * id;
      const size_t p = (size_t)(y0 + h) * A.W + x;
      float* abc = A.abc + (size_t)ch * 3 * HW;
      abc[p] = dmx - 2.f * dsxx * (mx - kShift) - dsxy * (my - kShift);
      abc[HW + p] = dsxx;
      abc[2 * HW + p] = dsxy;
      const float2 xy0 = s_in[(4 * ty + h + kR) * kIWp2 + tx + kR];
      acc[0] += fabsf(xy0.x - xy0.y);
      acc[1] += s;
      if (ch == 0) acc[2] += 1.f;
    }
  }
  block_sum<3>(acc, reinterpret_cast<float (*)[3]>(s_red));
  if (tid == 0) {
    atomicAdd(A.loss + 3, (double)acc[0]);
    atomicAdd(A.loss + 4, (double)acc[1]);
    atomicAdd(A.loss + 5, (double)acc[2]);
  }
}

__device__ __forceinline__ void rgb_finalize(double* loss) {
  const double n = loss[5];
  const double L1 = n > 0 ? loss[3] / (3.0 * n) : 0.0, S = n > 0 ? loss[4] / (3.0 * n) : 1.0;
  loss[0] = 0.8 * L1 + 0.2 * (1.0 - S);
  loss[1] = L1;
  loss[2] = S;
}

__global__ void rgb_finalize_kernel(double* loss) { rgb_finalize(loss); }

__global__ void __launch_bounds__(256) rgb_bwd_kernel(RgbArgs A) {
  extern __shared__ float4 smem_f4[];
  float2* s_ab = reinterpret_cast<float2*>(smem_f4);          // [3] planes of (A', B)
  float* s_c = reinterpret_cast<float*>(s_ab + 3 * kPlane);   // [3] planes of Cc
  float2* s_h2 = reinterpret_cast<float2*>(s_c + 3 * kPlane); // (G*A', G*B) horizontal
  float* s_h1 = reinterpret_cast<float*>(s_h2 + kHPlane);     // G*Cc horizontal
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int bx = blockIdx.x * kTW, by = blockIdx.y * kTH;
  const int x = bx + tx, y0 = by + 2 * ty;
  // the loss values (the sums are complete: rgb_fwd precedes on the stream); no separate
  // one-thread launch that would queue behind concurrent side-stream work
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) rgb_finalize(A.loss);
  bool m0, m1;
  if (!tile_has_mask(A, x, y0, m0, m1)) return;
  const double n = A.loss[5];
  const size_t HW = (size_t)A.W * A.H;
  for (int r = ty; r < kIH; r += 8) {
    const int gy = by - kR + r;
    for (int c = tx; c < kIW; c += 32) {
      const int gx = bx - kR + c;
      float v[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) v[k] = 0.f;
      if (gx >= 0 && gy >= 0 && gx < A.W && gy < A.H) {
        const size_t p = (size_t)gy * A.W + gx;
        const uint8_t mk = __ldg(A.mask + p);
#pragma unroll
        for (int k = 0; k < 9; ++k) v[k] = __ldg(A.abc + k * HW + p);
        if (!mk)  // partials exist only at mask pixels (elsewhere the buffer is stale)
#pragma unroll
          for (int k = 0; k < 9; ++k) v[k] = 0.f;
      }
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        s_ab[ch * kPlane + r * kIWp + c] = f2(v[3 * ch], v[3 * ch + 1]);
        s_c[ch * kPlane + r * kIWp + c] = v[3 * ch + 2];
      }
    }
  }
  float g[2 * kR + 1];
  window(g);
  const float kS = (float)(-0.2 / (3.0 * n) * A.weight);
  const float kL = (float)(0.8 / (3.0 * n) * A.weight);
  float xv[2][3], yv[2][3];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const size_t p = (size_t)(y0 + h) * A.W + x;
    const bool m = h ? m1 : m0;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      xv[h][ch] = m ? __ldg(A.C + ch * HW + p) : 0.f;
      yv[h][ch] = m ? __ldg(A.I + ch * HW + p) : 0.f;
    }
  }
#pragma unroll 1
  for (int ch = 0; ch < 3; ++ch) {
    __syncthreads();  // s_ab / s_c published (ch 0) / previous channel's vertical pass done
    if (tid < kIH * (kTW / 4)) {
      const int r = tid >> 3, c0 = 4 * (tid & 7);
      float2 v[16], o2[4];
      float w[16], o1[4];
      load16x2(s_ab + ch * kPlane + r * kIWp + c0, v);
      load16(s_c + ch * kPlane + r * kIWp + c0, w);
#pragma unroll
      for (int o = 0; o < 4; ++o) {
        o2[o] = f2(0.f, 0.f);
        o1[o] = 0.f;
#pragma unroll
        for (int k = 0; k <= 2 * kR; ++k) {
          o2[o] = __ffma2_rn(f2(g[k], g[k]), v[o + k], o2[o]);
          o1[o] = fmaf(g[k], w[o + k], o1[o]);
        }
      }
      store4x2(s_h2 + r * kTW + c0, o2);
      store4(s_h1 + r * kTW + c0, o1);
    }
    __syncthreads();
    float2 ab[2];
    float cc[2];
    {
      float2 ca[12];
      float cw[12];
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const int o = (2 * ty + k) * kTW + tx;
        ca[k] = s_h2[o];
        cw[k] = s_h1[o];
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ab[h] = f2(0.f, 0.f);
        cc[h] = 0.f;
#pragma unroll
        for (int k = 0; k <= 2 * kR; ++k) {
          ab[h] = __ffma2_rn(f2(g[k], g[k]), ca[k + h], ab[h]);
          cc[h] = fmaf(g[k], cw[k + h], cc[h]);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!(h ? m1 : m0)) continue;
      const float xq = ch == 0 ? xv[h][0] : (ch == 1 ? xv[h][1] : xv[h][2]);
      const float yq = ch == 0 ? yv[h][0] : (ch == 1 ? yv[h][1] : yv[h][2]);
      const float d = xq - yq;
      const float sg = d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f);
      A.dC[ch * HW + (size_t)(y0 + h) * A.W + x] =
          kS * (ab[h].x + 2.f * (xq - kShift) * ab[h].y + (yq - kShift) * cc[h]) + kL * sg;
    }
  }
}

// ------------------------------------------------------------------ Adam (+ L_s)
struct AdamArgs {
  int n, K3;
  const float *__restrict__ dmean, *__restrict__ dscale, *__restrict__ drot, *__restrict__ dop, *__restrict__ dsh;
  float *__restrict__ mean, *__restrict__ scale, *__restrict__ rot, *__restrict__ op, *__restrict__ sh;
  float *__restrict__ log_scale, *__restrict__ logit_op, *__restrict__ m, *__restrict__ v;
  AdamP P;  // adam.cuh: the update shared with the fused A8 + Adam
  double* flat;
};

__global__ void __launch_bounds__(256) adam_kernel(AdamArgs A) {
  __shared__ float s_red[8];
  const int i = blockIdx.x * 256 + threadIdx.x;
  float smin = 0.f;
  if (i < A.n) {
    const size_t n = A.n;
    const AdamP& P = A.P;
    // L_s = mean_i min_k s_ik: d/ds = flat_w / n on the minimum axis
    const float s0 = A.scale[i], s1 = A.scale[n + i], s2 = A.scale[2 * n + i];
    int kmin;
    smin = min_axis(s0, s1, s2, kmin);
    const float gflat = P.flat_w / (float)A.n;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      A.mean[c * n + i] = adam_at(P, A.m, A.v, c, n, i, A.mean[c * n + i], A.dmean[c * n + i], P.lr_mean);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float s = c == 0 ? s0 : (c == 1 ? s1 : s2);
      const float r = adam_at(P, A.m, A.v, 3 + c, n, i, A.log_scale[c * n + i],
                              dlog_scale(A.dscale[c * n + i], c == kmin, gflat, s), P.lr_scale);
      A.log_scale[c * n + i] = r;
      A.scale[c * n + i] = expf(r);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      A.rot[c * n + i] = adam_at(P, A.m, A.v, 6 + c, n, i, A.rot[c * n + i], A.drot[c * n + i], P.lr_rot);
    {
      const float o = A.op[i];
      const float r = adam_at(P, A.m, A.v, 10, n, i, A.logit_op[i], dlogit_opacity(A.dop[i], o), P.lr_op);
      A.logit_op[i] = r;
      A.op[i] = 1.f / (1.f + expf(-r));
    }
    // SH rows in batches of 4: all loads of a batch are issued before its stores (memory-level
    // parallelism; the arrays may alias as far as the compiler knows)
    int c = 0;
    for (; c + 4 <= A.K3; c += 4) {
      float gq[4], mq[4], vq[4], rq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const size_t k = (size_t)(11 + c + q) * n + i, e = (size_t)(c + q) * n + i;
        gq[q] = __ldg(A.dsh + e);
        mq[q] = A.m[k];
        vq[q] = A.v[k];
        rq[q] = A.sh[e];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const size_t k = (size_t)(11 + c + q) * n + i, e = (size_t)(c + q) * n + i;
        const float r = adam_elem(P, mq[q], vq[q], rq[q], gq[q], c + q < 3 ? P.lr_dc : P.lr_rest);
        A.m[k] = mq[q];
        A.v[k] = vq[q];
        A.sh[e] = r;
      }
    }
    for (; c < A.K3; ++c)
      A.sh[c * n + i] = adam_at(P, A.m, A.v, 11 + c, n, i, A.sh[c * n + i], A.dsh[c * n + i],
                                c < 3 ? P.lr_dc : P.lr_rest);
  }
  float v = smin;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0 && A.flat) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += s_red[k];
    atomicAdd(A.flat, s / (double)A.n);
  }
}

// 8-bit interleaved photo [H][W][3] -> planar float [3][H][W] in [0, 1] (b / 255, correctly
// rounded); 4 pixels (12 bytes, three aligned words) per thread when W allows.
__global__ void __launch_bounds__(256) unpack_rgb8_kernel(const uint8_t* __restrict__ rgb, size_t npix,
                                                          float* __restrict__ chw) {
  const size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // group of 4 pixels
  const size_t p0 = 4 * q;
  if (p0 >= npix) return;
  if (p0 + 4 <= npix) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(rgb + 3 * p0);
    const uint32_t a = __ldg(w), b = __ldg(w + 1), c = __ldg(w + 2);
    const uint32_t by[12] = {a & 255u, (a >> 8) & 255u, (a >> 16) & 255u, a >> 24, b & 255u, (b >> 8) & 255u,
                             (b >> 16) & 255u, b >> 24, c & 255u, (c >> 8) & 255u, (c >> 16) & 255u, c >> 24};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      float4 v;
      v.x = __fdiv_rn((float)by[ch], 255.0f);
      v.y = __fdiv_rn((float)by[3 + ch], 255.0f);
      v.z = __fdiv_rn((float)by[6 + ch], 255.0f);
      v.w = __fdiv_rn((float)by[9 + ch], 255.0f);
      *reinterpret_cast<float4*>(chw + ch * npix + p0) = v;
    }
  } else {
    for (size_t p = p0; p < npix; ++p)
      for (int ch = 0; ch < 3; ++ch) chw[ch * npix + p] = __fdiv_rn((float)rgb[3 * p + ch], 255.0f);
  }
}

}  // namespace

cudaError_t launch_unpack_rgb8(const uint8_t* rgb, int W, int H, float* chw, cudaStream_t st) {
  const size_t npix = (size_t)W * H;
  const size_t groups = (npix + 3) / 4;
  KTimer kt_("N3_unpack_rgb8", st);
  unpack_rgb8_kernel<<<(unsigned)((groups + 255) / 256), 256, 0, st>>>(rgb, npix, chw);
  return cudaGetLastError();
}

cudaError_t launch_rgb_loss(const float* image, const float* target, const uint8_t* mask, int W, int H, float weight,
                            double* loss, float* dC, float* abc, cudaStream_t st) {
  RgbArgs A;
  A.C = image; A.I = target; A.mask = mask; A.W = W; A.H = H; A.weight = weight;
  A.abc = abc; A.loss = loss; A.dC = dC;
  cudaError_t e = cudaMemsetAsync(loss, 0, 6 * sizeof(double), st);
  if (e != cudaSuccess) return e;
  static bool attr[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr[dev]) {
    cudaFuncSetAttribute(rgb_fwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem2);
    cudaFuncSetAttribute(rgb_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kBwdSmem);
    attr[dev] = true;
  }
  static const Win kWin = [] {  // g[k] = exp(-k^2 / 4.5) / sum in double, rounded once (as window())
    Win w;
    double v[2 * kR + 1], sum = 0.0;
    for (int k = -kR; k <= kR; ++k) {
      v[k + kR] = exp(-(double)(k * k) / 4.5);
      sum += v[k + kR];
    }
    for (int k = 0; k <= 2 * kR; ++k) w.g[k] = (float)(v[k] / sum);
    return w;
  }();
  const dim3 grid((W + kTW - 1) / kTW, (H + kTH - 1) / kTH);
  {
    KTimer kt_("N3_rgb_fwd", st);
    rgb_fwd2_kernel<<<dim3((W + kTW2 - 1) / kTW2, (H + kTH2 - 1) / kTH2), 256, kFwdSmem2, st>>>(A, kWin);
  }
  if (dC) {
    KTimer kt_("N3_rgb_bwd", st);
    rgb_bwd_kernel<<<grid, 256, kBwdSmem, st>>>(A);  // also finalises the loss values
  } else {
    KTimer kt_("N3_rgb_finalize", st);
    rgb_finalize_kernel<<<1, 1, 0, st>>>(loss);
  }
  return cudaGetLastError();
}

namespace {
// R30: the raw parameters of 3DGS's optimiser from the activated ones: log scale, logit opacity
// (the logit in double: o near 1 loses its low bits in float32's 1 - o).
__global__ void adam_init_kernel(int n, const float* __restrict__ scale, const float* __restrict__ op,
                                 float* __restrict__ log_scale, float* __restrict__ logit_op) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) log_scale[(size_t)k * n + i] = logf(scale[(size_t)k * n + i]);
  const double o = (double)op[i];
  logit_op[i] = (float)log(o / (1.0 - o));
}

// Eq. 10-11: L = (1 - lambda) (L_rgb + lambda3 L_s + lambda4 L_ban) + lambda L_GC-load.
__global__ void loss_total_kernel(const double* rgb, const double* flat, const double* ban, const double* gc,
                                  double lam, double lam3, double lam4, int ban_mean, double* out) {
  double Lban = 0.0;
  if (ban) Lban = ban_mean ? (ban[1] > 0.0 ? ban[0] / ban[1] : 0.0) : ban[0];
  const double Ls = flat ? flat[0] : 0.0;
  const double Lgc = gc ? gc[3] : 0.0;
  out[0] = (1.0 - lam) * (rgb[0] + lam3 * Ls + lam4 * Lban) + lam * Lgc;
}
}  // namespace

cudaError_t launch_adam_init(int n, pgsag_adam_state* s, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  adam_init_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, s->scale, s->opacity, s->log_scale, s->logit_opacity);
  return cudaGetLastError();
}

cudaError_t launch_loss_total(const double* rgb, const double* flat, const double* ban, const double* gc, double lam,
                              double lam3, double lam4, int ban_mean, double* out, cudaStream_t st) {
  loss_total_kernel<<<1, 1, 0, st>>>(rgb, flat, ban, gc, lam, lam3, lam4, ban_mean, out);
  return cudaGetLastError();
}

cudaError_t launch_adam(int n, int sh_degree, const pgsag_gaussian_grad* gr, pgsag_adam_state* s,
                        const pgsag_adam_hparams* hp, double* flat, cudaStream_t st) {
  AdamArgs A;
  A.n = n; A.K3 = (sh_degree + 1) * (sh_degree + 1) * 3;
  A.dmean = gr->dmean; A.dscale = gr->dscale; A.drot = gr->drot; A.dop = gr->dopacity; A.dsh = gr->dsh;
  A.mean = s->mean; A.scale = s->scale; A.rot = s->rot; A.op = s->opacity; A.sh = s->sh;
  A.log_scale = s->log_scale; A.logit_op = s->logit_opacity; A.m = s->m; A.v = s->v;
  A.P = adam_params(hp);
  A.flat = flat;
  if (flat) {
    cudaError_t e = cudaMemsetAsync(flat, 0, sizeof(double), st);
    if (e != cudaSuccess) return e;
  }
  if (n == 0) return cudaSuccess;
  KTimer kt_("N3_adam", st);
  adam_kernel<<<(n + 255) / 256, 256, 0, st>>>(A);
  return cudaGetLastError();
}

}  // namespace pgsag
