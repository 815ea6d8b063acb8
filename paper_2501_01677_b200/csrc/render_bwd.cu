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
// Work mapping is A6's: per active tile, 4 warps on 8x8 pixel blocks, two pixels
// (x, y), (x, y + 4) per lane in packed FP32x2, batches of 256 entries staged with
// the same exact warp-block cull and compacted per-warp candidate lists, walked
// in reverse.  A pixel that does not contribute to an entry carries alpha = rho =
// 0, which zeroes all of its terms and leaves its state unchanged without
// branches.  Reduction: per entry, the lane's two pixels are summed, the warp's
// 14 partials are reduce-scattered (5 butterfly levels, 16 shuffles) so that 14
// lanes each hold one warp sum, those lanes add into a padded shared accumulator
// of the batch, and after the batch the CTA flushes one double-precision global
// atomic per (entry, value).
#include <cuda_runtime.h>
#include <stdint.h>

#include "alpha.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kG2 = 14;  // du dv dca dcb dcc dop drgb3 dncam3 ddist absgrad
constexpr int kBT = 128;
constexpr int kBEPT = 2;
constexpr int kBBatch = kBT * kBEPT;
constexpr int kBNB = 4;
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

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
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

// Per-pixel prologue: upstream G (Eq. 4 folded in), P*(bg.gC), last index, T.
struct PixState {
  float G[8];
  float Pb;
  float T;
  int last;
};

__device__ __forceinline__ void load_pixel(const BwdArgs& a, bool masked, size_t pix, size_t HW, float px, float py,
                                           PixState& s) {
#pragma unroll
  for (int c = 0; c < 8; ++c) s.G[c] = 0.f;
  s.Pb = 0.f;
  s.T = 1.f;
  s.last = -1;
  if (!masked) return;
  s.last = a.last[pix];
  s.T = a.T[pix];
  s.G[0] = ld_or0(a.dC, pix); s.G[1] = ld_or0(a.dC, HW + pix); s.G[2] = ld_or0(a.dC, 2 * HW + pix);
  s.G[3] = ld_or0(a.dN, pix); s.G[4] = ld_or0(a.dN, HW + pix); s.G[5] = ld_or0(a.dN, 2 * HW + pix);
  s.G[6] = ld_or0(a.dD, pix);
  s.G[7] = ld_or0(a.dA, pix);
  const float gDep = ld_or0(a.dDep, pix);
  // Eq. 4 prologue: Dep = D / (N . r); validity re-derived exactly as A6 did
  const float N0 = a.N[pix], N1 = a.N[HW + pix], N2 = a.N[2 * HW + pix];
  const float r0 = __fdiv_rn(__fsub_rn(px, a.cx), a.fx), r1 = __fdiv_rn(__fsub_rn(py, a.cy), a.fy);
  const float den = __fadd_rn(__fadd_rn(__fmul_rn(N0, r0), __fmul_rn(N1, r1)), N2);
  if (a.g[pix] > 0 && fabsf(den) > 1e-6f) {
    const float inv = 1.0f / den;
    s.G[6] += gDep * inv;
    const float c = gDep * a.D[pix] * inv * inv;
    s.G[3] -= c * r0; s.G[4] -= c * r1; s.G[5] -= c;
  }
  s.Pb = a.bg0 * s.G[0] + a.bg1 * s.G[1] + a.bg2 * s.G[2];
}

template <bool kCount>
__global__ void __launch_bounds__(kBT) render_bwd_kernel(BwdArgs a) {
  constexpr int kAccStride = 15;  // padded row: the 14 values of an entry sit in 14 distinct banks
  __shared__ Rec s_rec[kBBatch];
  __shared__ uint32_t s_id[kBBatch];
  __shared__ float s_acc[kBBatch * kAccStride];
  __shared__ uint8_t s_list[kBNB * kBBatch];
  __shared__ uint32_t s_wc[kBEPT * (kBT / 32) * kBNB];
  __shared__ int s_nw[kBNB];
  __shared__ uint32_t s_tile;
  __shared__ int s_maxlast;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t n_active = *a.n_active;
  const size_t HW = (size_t)a.d.W * a.d.H;
  const uint32_t rec_base = smem_u32(s_rec), list_base = smem_u32(s_list);
  unsigned long long cntV = 0;
  // value index this lane owns after the reduce-scatter: bit-reversed lane bits 1..4
  const int my_c = (((lane >> 4) & 1) << 3) | (((lane >> 3) & 1) << 2) | (((lane >> 2) & 1) << 1) | ((lane >> 1) & 1);
  const bool writer = ((lane & 1) == 0) && my_c < kG2;
  for (int k = tid; k < kBBatch * kAccStride; k += kBT) s_acc[k] = 0.f;
  for (;;) {
    if (tid == 0) { s_tile = atomicAdd(a.work, 1u); s_maxlast = -1; }
    __syncthreads();
    const uint32_t widx = s_tile;
    if (widx >= n_active) break;
    const uint32_t tile = a.active[widx];
    const int ty = tile / a.d.TX, tx = tile - ty * a.d.TX;
    const int i = tx * kTile + (w & 1) * 8 + (lane & 7);
    const int j0 = ty * kTile + (w >> 1) * 8 + (lane >> 3), j1 = j0 + 4;
    const size_t pix0 = (size_t)j0 * a.d.W + i, pix1 = (size_t)j1 * a.d.W + i;
    const bool m0 = i < a.d.W && j0 < a.d.H && a.mask[pix0] != 0;
    const bool m1 = i < a.d.W && j1 < a.d.H && a.mask[pix1] != 0;
    const uint32_t rs = a.ranges[2 * tile];
    const float px = (float)i + 0.5f;
    const float2 py = f2((float)j0 + 0.5f, (float)j1 + 0.5f);
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
    PixState s0, s1;
    load_pixel(a, m0, pix0, HW, px, py.x, s0);
    load_pixel(a, m1, pix1, HW, px, py.y, s1);
    float2 Gp[8];  // (pixel0, pixel1) per channel
#pragma unroll
    for (int c = 0; c < 8; ++c) Gp[c] = f2(s0.G[c], s1.G[c]);
    float2 Pb = f2(s0.Pb, s1.Pb), Tcur = f2(s0.T, s1.T), Sg = f2(0.f, 0.f);
    const int last0 = s0.last, last1 = s1.last;
    const int mylast = max(last0, last1);
    if (mylast >= 0) atomicMax(&s_maxlast, mylast);
    const int wlast = __reduce_max_sync(0xffffffffu, mylast);
    __syncthreads();
    const int maxlast = s_maxlast;
    for (int bhi = maxlast + 1; bhi > (int)rs; bhi -= kBBatch) {
      const int blo = max((int)rs, bhi - kBBatch);
      const int cnt = bhi - blo;
      uint32_t mk[kBEPT];
#pragma unroll
      for (int e = 0; e < kBEPT; ++e) {
        const int slot = e * kBT + tid;
        mk[e] = 0u;
        if (slot < cnt) {
          const uint32_t id = a.vals[blo + slot];
          Rec& r = s_rec[slot];
          mk[e] = stage_gaussian<8, 8>(a.mean2d[id], a.conic_o[id], tx0, ty0, r);
          r.cd = a.rgb_d[id];
          r.n = a.ncam[id];
          s_id[slot] = id;
        }
      }
      build_lists<kBT, kBEPT, kBNB>(mk, s_list, s_wc, s_nw);
      const int qtop = wlast - blo;  // entries past the warp's last are never needed
      const uint32_t lbase = list_base + (uint32_t)(w * kBBatch);
      for (int t = s_nw[w] - 1; t >= 0; --t) {
        const int q = (int)lds_u8(lbase + (uint32_t)t);
        if (q > qtop) continue;  // warp-uniform
        const int kk = blo + q;
        const uint32_t ra_addr = rec_base + (uint32_t)q * (uint32_t)sizeof(Rec);
        const float4 ra = lds128(ra_addr);
        const float4 rb = lds128(ra_addr + 16);
        const float dx = px - ra.x;
        const float2 dy = __fadd2_rn(py, f2(-ra.y, -ra.y));
        const float tA = __fmul_rn(ra.z, dx);
        const float2 u = __ffma2_rn(f2(ra.w, ra.w), dy, f2(tA, tA));
        const float2 cq = __fmul2_rn(__fmul2_rn(f2(rb.x, rb.x), dy), dy);
        const float2 p2 = __ffma2_rn(f2(dx, dx), u, cq);
        const float rh0 = ex2_approx(p2.x), rh1 = ex2_approx(p2.y);
        const float2 orho = __fmul2_rn(f2(rb.y, rb.y), f2(rh0, rh1));
        float al0 = fminf(kAlphaMax, orho.x), al1 = fminf(kAlphaMax, orho.y);
        // exactly A6's blend decision (R6); entries past the pixel's last were not blended
        const bool c0 = kk <= last0 && p2.x <= 0.0f && al0 >= kAlphaMin;
        const bool c1 = kk <= last1 && p2.y <= 0.0f && al1 >= kAlphaMin;
        if (kCount) cntV += (unsigned long long)(kk <= last0) + (unsigned long long)(kk <= last1);
        if (!__any_sync(0xffffffffu, c0 || c1)) continue;
        al0 = c0 ? al0 : 0.f;
        al1 = c1 ? al1 : 0.f;
        // rho and alpha as they enter d(opacity) and d(power): zero when clamped at 0.99 (R16)
        const bool u0 = c0 && orho.x <= kAlphaMax, u1 = c1 && orho.y <= kAlphaMax;
        const float rc0 = u0 ? rh0 : 0.f, rc1 = u1 ? rh1 : 0.f;
        const float2 al = f2(al0, al1);
        const float2 om = __fadd2_rn(f2(1.f, 1.f), f2(-al0, -al1));
        const float2 Ti = __fmul2_rn(Tcur, f2(rcp_approx(om.x), rcp_approx(om.y)));
        const float4 cd = lds128(ra_addr + 32);
        const float4 nn = lds128(ra_addr + 48);
        float2 GF = Gp[7];
        GF = __ffma2_rn(Gp[0], f2(cd.x, cd.x), GF);
        GF = __ffma2_rn(Gp[1], f2(cd.y, cd.y), GF);
        GF = __ffma2_rn(Gp[2], f2(cd.z, cd.z), GF);
        GF = __ffma2_rn(Gp[3], f2(nn.x, nn.x), GF);
        GF = __ffma2_rn(Gp[4], f2(nn.y, nn.y), GF);
        GF = __ffma2_rn(Gp[5], f2(nn.z, nn.z), GF);
        GF = __ffma2_rn(Gp[6], f2(cd.w, cd.w), GF);
        const float2 dal = __fmul2_rn(Ti, __fadd2_rn(GF, f2(-(Sg.x + Pb.x), -(Sg.y + Pb.y))));
        Sg = __ffma2_rn(al, GF, __fmul2_rn(om, Sg));
        Pb = __fmul2_rn(Pb, om);
        Tcur = Ti;
        const float2 wt = __fmul2_rn(al, Ti);
        float v[16];
#pragma unroll
        for (int c = 0; c < 7; ++c) {
          const float2 x = __fmul2_rn(wt, Gp[c]);
          v[6 + c] = x.x + x.y;
        }
        const float2 dpow = __fmul2_rn(f2(u0 ? al0 : 0.f, u1 ? al1 : 0.f), dal);
        const float2 dop = __fmul2_rn(f2(rc0, rc1), dal);
        v[5] = dop.x + dop.y;
        const float sdp = dpow.x + dpow.y;
        const float2 dydp = __fmul2_rn(dy, dpow);
        const float sdydp = dydp.x + dydp.y;
        const float2 dy2dp = __fmul2_rn(dy, dydp);
        v[2] = -0.5f * dx * dx * sdp;
        v[3] = -dx * sdydp;
        v[4] = -0.5f * (dy2dp.x + dy2dp.y);
        // per-pixel screen-space mean gradient: (ca, cb, cc) = -ln2 (2A', B', 2C')
        const float2 gu = __ffma2_rn(f2(ra.w, ra.w), dy, f2(2.0f * tA, 2.0f * tA));        // 2A'dx + B'dy
        const float2 gv = __ffma2_rn(f2(2.0f * rb.x, 2.0f * rb.x), dy, f2(ra.w * dx, ra.w * dx));  // B'dx + 2C'dy
        const float2 du = __fmul2_rn(gu, __fmul2_rn(f2(-kLn2, -kLn2), dpow));
        const float2 dv = __fmul2_rn(gv, __fmul2_rn(f2(-kLn2, -kLn2), dpow));
        v[0] = du.x + du.y;
        v[1] = dv.x + dv.y;
        v[13] = (fabsf(du.x) + fabsf(dv.x)) + (fabsf(du.y) + fabsf(dv.y));
        v[14] = 0.f;
        v[15] = 0.f;
        // reduce-scatter 16 -> 1 value per lane pair
        float v8[8], v4[4], v2[2], v1[1];
        rs_level<8>(v, v8, (lane & 16) != 0, 16);
        rs_level<4>(v8, v4, (lane & 8) != 0, 8);
        rs_level<2>(v4, v2, (lane & 4) != 0, 4);
        rs_level<1>(v2, v1, (lane & 2) != 0, 2);
        const float sum = v1[0] + __shfl_xor_sync(0xffffffffu, v1[0], 1);
        if (writer && sum != 0.0f) atomicAdd(&s_acc[q * kAccStride + my_c], sum);
      }
      __syncthreads();
      // flush the batch: one f64 atomic per (entry, value), then re-zero
#pragma unroll
      for (int e = 0; e < kBEPT; ++e) {
        const int slot = e * kBT + tid;
        if (slot < cnt) {
          const uint32_t id = s_id[slot];
#pragma unroll
          for (int c = 0; c < kG2; ++c) {
            const float x = s_acc[slot * kAccStride + c];
            if (x != 0.0f) {
              atomicAdd(a.g2d + (size_t)c * a.n + id, (double)x);
              s_acc[slot * kAccStride + c] = 0.f;
            }
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, render_bwd_kernel<false>, kBT, 0);
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
      render_bwd_kernel<true><<<grid, kBT, 0, st>>>(a);
    else
      render_bwd_kernel<false><<<grid, kBT, 0, st>>>(a);
  }
  return launch_preprocess_bwd(g, cam, p, out, g2d, st);
}

}  // namespace pgsag
