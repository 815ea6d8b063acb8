// NEXT-2: boundary band and the boundary-aware normal loss L_ban (Eq. 8),
// with the normal-from-depth of P:153 ("computed from the depth map using four
// neighboring points"); readings R25-R27.  Per-pixel stencils, HBM-bound:
//   band: MB = dilation(RBM, r) XOR erosion(RBM, r), square (2r+1)^2, zero outside.
//   loss: per mask pixel with valid depth at its four axis neighbours,
//         n_depth = +-normalize((P_r - P_l) x (P_d - P_u)) (camera-facing), n_r = N/|N|,
//         term = w |n_depth - n_r|^2, w = bw on the band, 1 elsewhere in the mask;
//         loss[0] += term, loss[1] += 1 (f64 atomics after a block reduction);
//   grad: dN += lambda s dL/dN at the pixel, dDep += lambda s dL/dDep at the four
//         neighbours (float atomics), s = 1 / loss[1] if mean else 1.
// The differences P_r - P_l = (Dep_r - Dep_l) r_l + Dep_r (2/fx, 0, 0) (same for the
// vertical pair) avoid the cancellation of subtracting nearly equal 3D points.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pgsag {
namespace {

__global__ void band_kernel(const uint8_t* __restrict__ mask, int W, int H, int r, uint8_t* __restrict__ band) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  if (x >= W) return;
  bool any = false, all = true;
  for (int dy = -r; dy <= r; ++dy) {
    const int yy = y + dy;
    for (int dx = -r; dx <= r; ++dx) {
      const int xx = x + dx;
      const bool v = xx >= 0 && yy >= 0 && xx < W && yy < H && __ldg(mask + (size_t)yy * W + xx) != 0;
      any |= v;
      all &= v;
    }
  }
  band[(size_t)y * W + x] = (uint8_t)(any != all);
}

// Tiled variant for radii up to kBandRmax: the (8 + 2r) x (128 + 2r) mask window of a 128 x 8
// output tile is staged in shared memory once (coalesced 32-bit loads of the interior), then the
// square structuring element is applied separably (row any / all, then column any / all).
constexpr int kBandTW = 128, kBandTH = 8, kBandRmax = 8;
__global__ void __launch_bounds__(256) band_tiled_kernel(const uint8_t* __restrict__ mask, int W, int H, int r,
                                                         uint8_t* __restrict__ band) {
  constexpr int SW = kBandTW + 2 * kBandRmax, SH = kBandTH + 2 * kBandRmax;
  __shared__ uint8_t s_m[SH][SW];
  __shared__ __align__(4) uint8_t s_any[SH][kBandTW], s_all[SH][kBandTW];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * kBandTW, y0 = blockIdx.y * kBandTH;
  const int rows = kBandTH + 2 * r, cols = kBandTW + 2 * r;
  for (int ry = ty; ry < rows; ry += 8) {  // window staging: a warp per row, 32 consecutive bytes
    const int gy = y0 - r + ry;
    const bool rin = gy >= 0 && gy < H;
    for (int rx = tx; rx < cols; rx += 32) {
      const int gx = x0 - r + rx;
      s_m[ry][rx] = (rin && gx >= 0 && gx < W && __ldg(mask + (size_t)gy * W + gx) != 0) ? 1 : 0;
    }
  }
  __syncthreads();
  for (int ry = ty; ry < rows; ry += 8) {  // horizontal any / all: 4 adjacent columns per thread
    const int x = 4 * tx;
    uint32_t an = 0, al = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t a = 0, b = 1;
      for (int d = 0; d <= 2 * r; ++d) {
        const uint32_t v = s_m[ry][x + q + d];
        a |= v;
        b &= v;
      }
      an |= a << (8 * q);
      al |= b << (8 * q);
    }
    *reinterpret_cast<uint32_t*>(&s_any[ry][x]) = an;
    *reinterpret_cast<uint32_t*>(&s_all[ry][x]) = al;
  }
  __syncthreads();
  {  // vertical any / all on 4 columns at once (bytes are 0 / 1), band = any xor all
    const int x = 4 * tx, y = ty;
    uint32_t an = 0, al = 0x01010101u;
    for (int d = 0; d <= 2 * r; ++d) {
      an |= *reinterpret_cast<const uint32_t*>(&s_any[y + d][x]);
      al &= *reinterpret_cast<const uint32_t*>(&s_all[y + d][x]);
    }
    const uint32_t out = an ^ al;
    const int gx = x0 + x, gy = y0 + y;
    if (gy < H) {
      uint8_t* dst = band + (size_t)gy * W + gx;
      if (gx + 3 < W && (((size_t)gy * W + gx) & 3) == 0) {
        *reinterpret_cast<uint32_t*>(dst) = out;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (gx + q < W) dst[q] = (uint8_t)((out >> (8 * q)) & 0xffu);
      }
    }
  }
}

struct BanArgs {
  const uint8_t* mask;
  const uint8_t* band;
  const float* N;
  const float* Dep;
  int W, H;
  float ifx, ify, cx, cy;
  float bw, lambda;
  int mean;
  double* loss;
  float* dN;
  float* dDep;
};

struct BanTerm {
  bool valid;
  float e[3], w, c[3], cn, s, nr[3], Nn;
  float a[3], b[3];
};

// (x, y) is a mask pixel.  All loads of the stencil are issued before any test (neighbour
// addresses clamped into the image; a clamped neighbour is rejected by its bounds flag), so the
// pixel waits on one memory latency instead of one per short-circuited test.
__device__ __forceinline__ void ban_term(const BanArgs& A, int x, int y, BanTerm& t) {
  t.valid = false;
  const size_t HW = (size_t)A.W * A.H, p = (size_t)y * A.W + x;
  const bool il = x > 0, ir = x + 1 < A.W, iu = y > 0, id = y + 1 < A.H;
  const size_t pl = il ? p - 1 : p, pr = ir ? p + 1 : p, pu = iu ? p - A.W : p, pd = id ? p + A.W : p;
  const uint8_t ml = __ldg(A.mask + pl), mr = __ldg(A.mask + pr), mu = __ldg(A.mask + pu), md = __ldg(A.mask + pd);
  const float Dl = __ldg(A.Dep + pl), Dr = __ldg(A.Dep + pr), Du = __ldg(A.Dep + pu), Dd = __ldg(A.Dep + pd);
  const float Dp = __ldg(A.Dep + p);
  const float N0 = __ldg(A.N + p), N1 = __ldg(A.N + HW + p), N2 = __ldg(A.N + 2 * HW + p);
  if (!(Dp != 0.0f && il && ml && Dl != 0.0f && ir && mr && Dr != 0.0f && iu && mu && Du != 0.0f && id && md &&
        Dd != 0.0f))
    return;
  t.Nn = sqrtf(N0 * N0 + N1 * N1 + N2 * N2);
  if (!(t.Nn > 0.f)) return;
  const float rlx = ((float)x - 0.5f - A.cx) * A.ifx, ry = ((float)y + 0.5f - A.cy) * A.ify;
  const float rx = ((float)x + 0.5f - A.cx) * A.ifx, ruy = ((float)y - 0.5f - A.cy) * A.ify;
  const float dh = Dr - Dl, dv = Dd - Du;
  t.a[0] = dh * rlx + Dr * 2.0f * A.ifx; t.a[1] = dh * ry; t.a[2] = dh;
  t.b[0] = dv * rx; t.b[1] = dv * ruy + Dd * 2.0f * A.ify; t.b[2] = dv;
  t.c[0] = t.a[1] * t.b[2] - t.a[2] * t.b[1];
  t.c[1] = t.a[2] * t.b[0] - t.a[0] * t.b[2];
  t.c[2] = t.a[0] * t.b[1] - t.a[1] * t.b[0];
  t.cn = sqrtf(t.c[0] * t.c[0] + t.c[1] * t.c[1] + t.c[2] * t.c[2]);
  if (!(t.cn > 0.f)) return;
  const float facing = (t.c[0] * rx + t.c[1] * ry + t.c[2]) * Dp;
  t.s = facing > 0.f ? -1.f : 1.f;
  const float ic = 1.0f / t.cn, iN = 1.0f / t.Nn;
  t.nr[0] = N0 * iN; t.nr[1] = N1 * iN; t.nr[2] = N2 * iN;
#pragma unroll
  for (int k = 0; k < 3; ++k) t.e[k] = t.s * t.c[k] * ic - t.nr[k];
  t.w = __ldg(A.band + p) ? A.bw : 1.0f;
  t.valid = true;
}

// kLoss: accumulate (sum of terms, count) into loss[0..1]; kGrad: scatter lambda s dL/d(N, Dep)
// with s = 1 / loss[1] (mean, needs a finished loss pass) or 1 (sum).  mean = 0 runs both in
// one pass.
template <bool kLoss, bool kGrad>
__global__ void __launch_bounds__(256) ban_kernel(BanArgs A) {
  __shared__ float s_r[8][2];
  const int x = blockIdx.x * 32 + (threadIdx.x & 31), y = blockIdx.y * 8 + (threadIdx.x >> 5);
  float sum = 0.f, cnt = 0.f;
  BanTerm t;
  t.valid = false;
  if (x < A.W && y < A.H && __ldg(A.mask + (size_t)y * A.W + x)) ban_term(A, x, y, t);
  if (kLoss) {
    if (t.valid) {
      sum = t.w * (t.e[0] * t.e[0] + t.e[1] * t.e[1] + t.e[2] * t.e[2]);
      cnt = 1.f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sum += __shfl_xor_sync(0xffffffffu, sum, o);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if ((threadIdx.x & 31) == 0) { s_r[threadIdx.x >> 5][0] = sum; s_r[threadIdx.x >> 5][1] = cnt; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0, c = 0.0;
      for (int k = 0; k < 8; ++k) { s += s_r[k][0]; c += s_r[k][1]; }
      if (c > 0.0) { atomicAdd(A.loss, s); atomicAdd(A.loss + 1, c); }
    }
  }
  if (!kGrad || !t.valid) return;
  float sc = A.lambda;
  if (A.mean) {
    const double c = A.loss[1];
    if (c <= 0.0) return;
    sc *= (float)(1.0 / c);
  }
  const size_t HW = (size_t)A.W * A.H, p = (size_t)y * A.W + x;
  float gnd[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) gnd[k] = 2.0f * sc * t.w * t.e[k];
  if (A.dN) {  // n_r = N/|N|, its gradient is -gnd
    const float d = -(gnd[0] * t.nr[0] + gnd[1] * t.nr[1] + gnd[2] * t.nr[2]);
    const float iN = 1.0f / t.Nn;
#pragma unroll
    for (int k = 0; k < 3; ++k) A.dN[k * HW + p] += (-gnd[k] - t.nr[k] * d) * iN;
  }
  if (A.dDep) {  // n_d = s c/|c|, c = a x b
    const float ic = 1.0f / t.cn;
    const float cu[3] = {t.c[0] * ic, t.c[1] * ic, t.c[2] * ic};
    const float d = gnd[0] * cu[0] + gnd[1] * cu[1] + gnd[2] * cu[2];
    float gc[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) gc[k] = t.s * (gnd[k] - cu[k] * d) * ic;
    const float ga[3] = {t.b[1] * gc[2] - t.b[2] * gc[1], t.b[2] * gc[0] - t.b[0] * gc[2],
                         t.b[0] * gc[1] - t.b[1] * gc[0]};
    const float gb[3] = {gc[1] * t.a[2] - gc[2] * t.a[1], gc[2] * t.a[0] - gc[0] * t.a[2],
                         gc[0] * t.a[1] - gc[1] * t.a[0]};
    const float ry = ((float)y + 0.5f - A.cy) * A.ify, rx = ((float)x + 0.5f - A.cx) * A.ifx;
    const float rrx = ((float)x + 1.5f - A.cx) * A.ifx, rlx = ((float)x - 0.5f - A.cx) * A.ifx;
    const float rdy = ((float)y + 1.5f - A.cy) * A.ify, ruy = ((float)y - 0.5f - A.cy) * A.ify;
    atomicAdd(A.dDep + p + 1, ga[0] * rrx + ga[1] * ry + ga[2]);
    atomicAdd(A.dDep + p - 1, -(ga[0] * rlx + ga[1] * ry + ga[2]));
    atomicAdd(A.dDep + p + A.W, gb[0] * rx + gb[1] * rdy + gb[2]);
    atomicAdd(A.dDep + p - A.W, -(gb[0] * rx + gb[1] * ruy + gb[2]));
  }
}

}  // namespace

cudaError_t launch_boundary_band(const uint8_t* mask, int W, int H, int r, uint8_t* band, cudaStream_t st) {
  KTimer kt_("N2_band", st);
  if (r <= kBandRmax)
    band_tiled_kernel<<<dim3((W + kBandTW - 1) / kBandTW, (H + kBandTH - 1) / kBandTH), 256, 0, st>>>(mask, W, H,
                                                                                                    r, band);
  else
    band_kernel<<<dim3((W + 127) / 128, H), 128, 0, st>>>(mask, W, H, r, band);
  return cudaGetLastError();
}

cudaError_t launch_ban_loss(const pgsag_camera* cam, const uint8_t* mask, const uint8_t* band, const float* N,
                            const float* Dep, float bw, float lambda, int mean, double* loss, float* dN, float* dDep,
                            cudaStream_t st) {
  BanArgs A;
  A.mask = mask; A.band = band; A.N = N; A.Dep = Dep;
  A.W = cam->width; A.H = cam->height;
  A.ifx = 1.0f / cam->fx; A.ify = 1.0f / cam->fy; A.cx = cam->cx; A.cy = cam->cy;
  A.bw = bw; A.lambda = lambda; A.mean = mean;
  A.loss = loss; A.dN = dN; A.dDep = dDep;
  cudaMemsetAsync(loss, 0, 2 * sizeof(double), st);
  const dim3 grid((A.W + 31) / 32, (A.H + 7) / 8);
  const bool grads = dN || dDep;
  if (grads && !mean) {  // sum: loss and gradients in one pass
    KTimer kt_("N2_ban_fused", st);
    ban_kernel<true, true><<<grid, 256, 0, st>>>(A);
    return cudaGetLastError();
  }
  {
    KTimer kt_("N2_ban_loss", st);
    ban_kernel<true, false><<<grid, 256, 0, st>>>(A);
  }
  if (grads) {  // mean: the gradient pass needs the finished count
    KTimer kt_("N2_ban_grad", st);
    ban_kernel<false, true><<<grid, 256, 0, st>>>(A);
  }
  return cudaGetLastError();
}

}  // namespace pgsag
