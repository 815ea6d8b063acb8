// A6: masked forward compositor for sm_100a.
//
// P:79-92 Eq. 1-3 (front-to-back alpha blending of colour, camera-frame normal
// and plane distance), Eq. 4 (unbiased depth epilogue), P:163 (one
// thread per pixel), P:243 (only building-mask pixels are computed).
//
// Mapping: a persistent grid pulls ACTIVE tiles (tiles with >= 1 mask pixel) from
// the A0 list through an atomic counter; masked-out tiles are never visited.  One
// 256-thread CTA per 16x16 tile; warp w owns an 8x4 pixel block, one thread per
// pixel; masked-out pixels start "done".  Each batch of 256 sorted entries is
// staged in shared memory (one 56-byte record gather per thread) together with an
// 8-bit warp-block mask (exact conservative cull, alpha.cuh), from which every
// warp gets a compacted, depth-ordered candidate list; a warp's loop then touches
// only entries that can reach its pixels.  The tile stops when every pixel is done.
#include <cuda_runtime.h>
#include <stdint.h>

#include "alpha.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kNW = kTilePix / 32;

struct FwdArgs {
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
  float *C, *N, *D, *A, *Dep, *T;
  int32_t *g, *last;
  unsigned long long* counters;
  uint32_t* work;
};

template <bool kCount>
__global__ void __launch_bounds__(kTilePix) render_fwd_kernel(FwdArgs a) {
  __shared__ float4 s_a[kTilePix];
  __shared__ float4 s_b[kTilePix];
  __shared__ float4 s_cd[kTilePix];
  __shared__ float4 s_n[kTilePix];
  __shared__ uint8_t s_list[8 * kTilePix];
  __shared__ uint32_t s_wc[kNW * 8];
  __shared__ int s_nw[8];
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t n_active = *a.n_active;
  const size_t HW = (size_t)a.d.W * a.d.H;
  const uint8_t* my_list = s_list + w * kTilePix;
  unsigned long long cntE = 0, cntB = 0;
  for (;;) {
    if (tid == 0) s_tile = atomicAdd(a.work, 1u);
    __syncthreads();
    const uint32_t widx = s_tile;
    __syncthreads();
    if (widx >= n_active) break;
    const uint32_t tile = a.active[widx];
    const int ty = tile / a.d.TX, tx = tile - ty * a.d.TX;
    const int i = tx * kTile + warp_px(w, lane);
    const int j = ty * kTile + warp_py(w, lane);
    const bool inside = i < a.d.W && j < a.d.H;
    const size_t pix = (size_t)j * a.d.W + i;
    const bool masked = inside && a.mask[pix] != 0;
    const uint32_t rs = a.ranges[2 * tile], re = a.ranges[2 * tile + 1];
    const float px = (float)i + 0.5f, py = (float)j + 0.5f;
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f, N0 = 0.f, N1 = 0.f, N2 = 0.f, D = 0.f;
    int g = 0, last = -1;
    bool done = !masked;
    for (uint32_t b = rs; b < re; b += kTilePix) {
      if (__syncthreads_count(done) == kTilePix) break;
      const uint32_t k = b + tid;
      uint32_t m = 0u;
      if (k < re) {
        const uint32_t id = a.vals[k];
        const Staged st = stage_gaussian(a.mean2d[id], a.conic_o[id], tx0, ty0);
        s_a[tid] = st.a;
        s_b[tid] = st.b;
        s_cd[tid] = a.rgb_d[id];
        s_n[tid] = a.ncam[id];
        m = st.wmask;
      }
      build_warp_lists<kNW>(m, s_list, s_wc, s_nw);
      const int nw = s_nw[w];
      for (int t = 0; t < nw; ++t) {
        if (__all_sync(0xffffffffu, done)) break;
        const int q = my_list[t];
        const float4 ra = s_a[q];
        const float4 rb = s_b[q];
        if (!done) {
          const float dx = px - ra.x, dy = py - ra.y;
          const float p2 = power2r(ra, rb.x, dx, dy);
          if (kCount) ++cntE;
          if (p2 >= rb.z && p2 <= 0.0f) {
            const float alpha = fminf(kAlphaMax, __fmul_rn(rb.y, ex2_approx(p2)));
            if (alpha >= kAlphaMin) {
              const float Tn = __fmul_rn(T, 1.0f - alpha);
              if (Tn < kTmin) {
                done = true;
              } else {
                const float wgt = alpha * T;
                const float4 cd = s_cd[q];
                const float4 nn = s_n[q];
                C0 += wgt * cd.x; C1 += wgt * cd.y; C2 += wgt * cd.z; D += wgt * cd.w;
                N0 += wgt * nn.x; N1 += wgt * nn.y; N2 += wgt * nn.z;
                ++g;
                last = (int)(b + q);
                T = Tn;
              }
            }
          }
        }
      }
    }
    if (masked) {
      a.C[pix] = C0 + T * a.bg0;
      a.C[HW + pix] = C1 + T * a.bg1;
      a.C[2 * HW + pix] = C2 + T * a.bg2;
      a.N[pix] = N0; a.N[HW + pix] = N1; a.N[2 * HW + pix] = N2;
      a.D[pix] = D;
      a.A[pix] = 1.0f - T;
      a.T[pix] = T;
      a.g[pix] = g;
      a.last[pix] = last;
      // Eq. 4: depth of the ray / blended-plane intersection, r = K^-1 (px, py, 1)
      // (explicit roundings: the backward re-derives this validity decision bit-exactly)
      const float r0 = __fdiv_rn(__fsub_rn(px, a.cx), a.fx), r1 = __fdiv_rn(__fsub_rn(py, a.cy), a.fy);
      const float den = __fadd_rn(__fadd_rn(__fmul_rn(N0, r0), __fmul_rn(N1, r1)), N2);
      a.Dep[pix] = (g > 0 && fabsf(den) > 1e-6f) ? D / den : 0.0f;
      if (kCount) cntB += (unsigned long long)g;
    }
  }
  if (kCount) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cntE += __shfl_xor_sync(0xffffffffu, cntE, o);
      cntB += __shfl_xor_sync(0xffffffffu, cntB, o);
    }
    if (lane == 0 && (cntE | cntB)) {
      atomicAdd(a.counters + 0, cntE);
      atomicAdd(a.counters + 1, cntB);
    }
  }
}

int fwd_grid() {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, render_fwd_kernel<false>, kTilePix, 0);
    grid = sms * (occ > 0 ? occ : 1);
  }
  return grid;
}

}  // namespace

cudaError_t launch_render_fwd(const pgsag_projected* p, const pgsag_bins* bins, const pgsag_tilemask* tm,
                              const Dims& d, const pgsag_camera* cam, const uint8_t* mask, const float bg[3],
                              pgsag_image* out, uint32_t* work_counter, cudaStream_t st) {
  FwdArgs a;
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
  a.C = out->C; a.N = out->N; a.D = out->D; a.A = out->A; a.Dep = out->Dep; a.T = out->T;
  a.g = out->g; a.last = out->last;
  a.counters = out->counters;
  a.work = work_counter;
  const int grid = min(fwd_grid(), d.TX * d.TY);
  {
    KTimer kt_("A6_render_fwd", st);
    if (out->counters)
      render_fwd_kernel<true><<<grid, kTilePix, 0, st>>>(a);
    else
      render_fwd_kernel<false><<<grid, kTilePix, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace pgsag
