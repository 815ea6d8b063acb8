// A7: reverse-order backward compositor for sm_100a (then A8, preprocess_bwd.cu).
//
// P:82 "all the encoded parameters are optimized ... using differentiable
// rendering": the exact reverse mode of A6 (Eq. 1-4) with the forward's discrete
// decisions frozen (R16, R17).  Per pixel, walking the tile list backwards from
// the pixel's last blended entry, with F_i = (rgb, n_cam, d, 1) and the upstream
// gradient G (Eq. 4 prologue folded into G):
//   T_i    = T_{i+1} / (1 - alpha_i)                   (recovered; T_end = A6's T)
//   dalpha = T_i (G.F_i - G.S - P (bg.gC))
//   dF_i   = alpha_i T_i G
//   G.S   <- alpha (G.F_i) + (1 - alpha) G.S,   P (bg.gC) <- (1 - alpha) P (bg.gC)
// Only the projection G.S of the 8-channel suffix S is ever needed, so the
// suffix is carried as one scalar (mathematically identical to the 8-vector
// recurrence of the oracle).
//
// Work mapping is A6's: per active tile, 8 warps on 8x4 pixel blocks, batches of
// 256 entries staged with the same exact warp-block cull and compacted per-warp
// candidate lists, walked in reverse.  Reduction: per entry, the warp's 14
// per-lane partials are reduce-scattered (5 butterfly levels, 16 shuffles) so
// that 14 lanes each hold one warp sum; those lanes add into a padded shared
// accumulator of the batch (shared by the tile's 8 warps); after the batch the
// CTA flushes one double-precision global atomic per (entry, value).
#include <cuda_runtime.h>
#include <stdint.h>

#include "alpha.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kG2 = 14;  // du dv dca dcb dcc dop drgb3 dncam3 ddist absgrad
constexpr int kNW = kTilePix / 32;
constexpr float kLn2 = 0.6931471805599453f;

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
  double* g2d;  // [kG2][n]
  int n;
  unsigned long long* counters;
  uint32_t* work;
};

__device__ __forceinline__ float ld_or0(const float* p, size_t k) { return p ? __ldg(p + k) : 0.0f; }

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// one butterfly level: keep half of the values, exchange the other half with lane ^ m
template <int H>
__device__ __forceinline__ void rs_level(float (&v)[2 * H], float (&o)[H], bool upper, int m) {
#pragma unroll
  for (int k = 0; k < H; ++k) {
    const float send = upper ? v[k] : v[k + H];
    const float keep = upper ? v[k + H] : v[k];
    o[k] = keep + __shfl_xor_sync(0xffffffffu, send, m);
  }
}

template <bool kCount>
__global__ void __launch_bounds__(kTilePix) render_bwd_kernel(BwdArgs a) {
  constexpr int kAccStride = 15;  // padded row: the 14 values of an entry sit in 14 distinct banks
  __shared__ float4 s_a[kTilePix];   // (u, v, A', B')
  __shared__ float4 s_b[kTilePix];   // (C', o, skip threshold, 0)
  __shared__ float4 s_cd[kTilePix];
  __shared__ float4 s_n[kTilePix];
  __shared__ uint32_t s_id[kTilePix];
  __shared__ float s_acc[kTilePix * kAccStride];
  __shared__ uint8_t s_list[8 * kTilePix];
  __shared__ uint32_t s_wc[kNW * 8];
  __shared__ int s_nw[8];
  __shared__ uint32_t s_tile;
  __shared__ int s_maxlast;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t n_active = *a.n_active;
  const size_t HW = (size_t)a.d.W * a.d.H;
  const uint8_t* my_list = s_list + w * kTilePix;
  unsigned long long cntV = 0;
  // value index this lane owns after the reduce-scatter: bit-reversed lane bits 1..4
  const int my_c = (((lane >> 4) & 1) << 3) | (((lane >> 3) & 1) << 2) | (((lane >> 2) & 1) << 1) | ((lane >> 1) & 1);
  const bool writer = ((lane & 1) == 0) && my_c < kG2;
  for (int k = tid; k < kTilePix * kAccStride; k += kTilePix) s_acc[k] = 0.f;
  for (;;) {
    if (tid == 0) { s_tile = atomicAdd(a.work, 1u); s_maxlast = -1; }
    __syncthreads();
    const uint32_t widx = s_tile;
    if (widx >= n_active) break;
    const uint32_t tile = a.active[widx];
    const int ty = tile / a.d.TX, tx = tile - ty * a.d.TX;
    const int i = tx * kTile + warp_px(w, lane);
    const int j = ty * kTile + warp_py(w, lane);
    const bool inside = i < a.d.W && j < a.d.H;
    const size_t pix = (size_t)j * a.d.W + i;
    const bool masked = inside && a.mask[pix] != 0;
    const uint32_t rs = a.ranges[2 * tile];
    const float px = (float)i + 0.5f, py = (float)j + 0.5f;
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
    int mylast = -1;
    float Tcur = 1.0f;
    float G[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float Pb = 0.f;  // P * (bg . gC)
    if (masked) {
      mylast = a.last[pix];
      Tcur = a.T[pix];
      G[0] = ld_or0(a.dC, pix); G[1] = ld_or0(a.dC, HW + pix); G[2] = ld_or0(a.dC, 2 * HW + pix);
      G[3] = ld_or0(a.dN, pix); G[4] = ld_or0(a.dN, HW + pix); G[5] = ld_or0(a.dN, 2 * HW + pix);
      G[6] = ld_or0(a.dD, pix);
      G[7] = ld_or0(a.dA, pix);
      const float gDep = ld_or0(a.dDep, pix);
      // Eq. 4 prologue: Dep = D / (N . r); validity re-derived exactly as A6 did
      const float N0 = a.N[pix], N1 = a.N[HW + pix], N2 = a.N[2 * HW + pix];
      const float r0 = __fdiv_rn(__fsub_rn(px, a.cx), a.fx), r1 = __fdiv_rn(__fsub_rn(py, a.cy), a.fy);
      const float den = __fadd_rn(__fadd_rn(__fmul_rn(N0, r0), __fmul_rn(N1, r1)), N2);
      if (a.g[pix] > 0 && fabsf(den) > 1e-6f) {
        const float inv = 1.0f / den;
        G[6] += gDep * inv;
        const float c = gDep * a.D[pix] * inv * inv;
        G[3] -= c * r0; G[4] -= c * r1; G[5] -= c;
      }
      Pb = a.bg0 * G[0] + a.bg1 * G[1] + a.bg2 * G[2];
      if (mylast >= 0) atomicMax(&s_maxlast, mylast);
    }
    const int wlast = __reduce_max_sync(0xffffffffu, mylast);
    __syncthreads();
    const int maxlast = s_maxlast;
    float Sg = 0.f;  // G . S
    for (int bhi = maxlast + 1; bhi > (int)rs; bhi -= kTilePix) {
      const int blo = max((int)rs, bhi - kTilePix);
      const int cnt = bhi - blo;
      uint32_t m = 0u;
      if (tid < cnt) {
        const uint32_t id = a.vals[blo + tid];
        const Staged st = stage_gaussian(a.mean2d[id], a.conic_o[id], tx0, ty0);
        s_id[tid] = id;
        s_a[tid] = st.a;
        s_b[tid] = st.b;
        s_cd[tid] = a.rgb_d[id];
        s_n[tid] = a.ncam[id];
        m = st.wmask;
      }
      build_warp_lists<kNW>(m, s_list, s_wc, s_nw);
      const int qtop = wlast - blo;  // entries past the warp's last are never needed
      for (int t = s_nw[w] - 1; t >= 0; --t) {
        const int q = my_list[t];
        if (q > qtop) continue;  // warp-uniform
        const int kk = blo + q;
        const float4 ra = s_a[q];
        const float4 rb = s_b[q];
        bool contrib = kk <= mylast;  // false for masked-out pixels (mylast = -1)
        float alpha = 0.f, rho = 0.f, dx = 0.f, dy = 0.f;
        if (contrib) {
          dx = px - ra.x; dy = py - ra.y;
          const float p2 = power2r(ra, rb.x, dx, dy);
          if (kCount) ++cntV;
          if (p2 >= rb.z && p2 <= 0.0f) {
            rho = ex2_approx(p2);
            alpha = fminf(kAlphaMax, __fmul_rn(rb.y, rho));
            contrib = alpha >= kAlphaMin;
          } else {
            contrib = false;
          }
        }
        if (!__any_sync(0xffffffffu, contrib)) continue;
        float v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) v[c] = 0.f;
        if (contrib) {
          const float4 cd = s_cd[q];
          const float4 nn = s_n[q];
          const float om = 1.0f - alpha;
          const float Ti = Tcur * rcp_approx(om);
          const float GF = G[0] * cd.x + G[1] * cd.y + G[2] * cd.z + G[3] * nn.x + G[4] * nn.y + G[5] * nn.z +
                           G[6] * cd.w + G[7];
          const float dalpha = Ti * (GF - Sg - Pb);
          Sg = alpha * GF + om * Sg;
          Pb *= om;
          Tcur = Ti;
          const float wgt = alpha * Ti;
#pragma unroll
          for (int c = 0; c < 7; ++c) v[6 + c] = wgt * G[c];
          if (__fmul_rn(rb.y, rho) <= kAlphaMax) {
            v[5] = rho * dalpha;
            const float dpow = alpha * dalpha;
            const float kx = dx * dpow;
            v[2] = -0.5f * dx * kx;
            v[3] = -dy * kx;
            v[4] = -0.5f * dy * dy * dpow;
            const float kd = -kLn2 * dpow;  // (ca, cb, cc) = -ln2 (2A', B', 2C')
            v[0] = (2.0f * ra.z * dx + ra.w * dy) * kd;
            v[1] = (ra.w * dx + 2.0f * rb.x * dy) * kd;
            v[13] = fabsf(v[0]) + fabsf(v[1]);
          }
        }
        // reduce-scatter 16 -> 1 value per lane pair
        float v8[8], v4[4], v2[2], v1[1];
        rs_level<8>(v, v8, (lane & 16) != 0, 16);
        rs_level<4>(v8, v4, (lane & 8) != 0, 8);
        rs_level<2>(v4, v2, (lane & 4) != 0, 4);
        rs_level<1>(v2, v1, (lane & 2) != 0, 2);
        const float s = v1[0] + __shfl_xor_sync(0xffffffffu, v1[0], 1);
        if (writer && s != 0.0f) atomicAdd(&s_acc[q * kAccStride + my_c], s);
      }
      __syncthreads();
      // flush the batch: one f64 atomic per (entry, value), then re-zero
      if (tid < cnt) {
        const uint32_t id = s_id[tid];
#pragma unroll
        for (int c = 0; c < kG2; ++c) {
          const float x = s_acc[tid * kAccStride + c];
          if (x != 0.0f) {
            atomicAdd(a.g2d + (size_t)c * a.n + id, (double)x);
            s_acc[tid * kAccStride + c] = 0.f;
          }
        }
      }
      __syncthreads();
    }
  }
  if (kCount) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cntV += __shfl_xor_sync(0xffffffffu, cntV, o);
    if (lane == 0 && cntV) atomicAdd(a.counters + 2, cntV);
  }
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
                              const pgsag_image_grad* dL, pgsag_gaussian_grad* out, double* g2d,
                              uint32_t* work_counter, cudaStream_t st) {
  const int n = g->n;
  if (n == 0) return cudaSuccess;
  cudaMemsetAsync(g2d, 0, sizeof(double) * kG2 * (size_t)n, st);
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
  {
    KTimer kt_("A7_render_bwd", st);
    if (fwd->counters)
      render_bwd_kernel<true><<<grid, kTilePix, 0, st>>>(a);
    else
      render_bwd_kernel<false><<<grid, kTilePix, 0, st>>>(a);
  }
  return launch_preprocess_bwd(g, cam, p, out, g2d, st);
}

}  // namespace pgsag
