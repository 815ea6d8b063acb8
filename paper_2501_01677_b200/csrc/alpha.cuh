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

#include "dcheck.cuh"

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

// same, with the record layout of the staged batch: ra = (u, v, A', B'), C' separately
__device__ __forceinline__ float power2r(const float4& ra, float Cp, float dx, float dy) {
  const float t = __fmaf_rn(ra.w, dy, __fmul_rn(ra.z, dx));
  return __fmaf_rn(dx, t, __fmul_rn(__fmul_rn(Cp, dy), dy));
}

// ------------------------------------------------------------------ staging
// A tile CTA has NW warps; warp w owns the BW x BH pixel block (w % (16/BW),
// w / (16/BW)) of the 16x16 tile.  Each staged entry gets a bit mask of the
// warp blocks it can reach (exact conservative cull below).

// Staged batch record, 64 B: one LDS.128 per field.
struct __align__(16) Rec {
  float4 a;   // u, v, A', B'
  float4 b;   // C', o, skip threshold on p2, 0
  float4 cd;  // r, g, b, d_i
  float4 n;   // n_cam, 0
};

// Exact refinement of the block cull: does the ellipse {d : d^T Q d <= k2} (Q = the
// conic) meet the rectangle of pixel centres?  If the centre is outside, the minimum
// of the convex quadratic over the rectangle lies on an edge; on each edge it is a 1D
// quadratic minimised in closed form and clamped.  The rectangle is declared missed
// only if that minimum exceeds k2 by more than a bound on its float rounding error.
__device__ __forceinline__ float edge_min(float ca, float cb, float cc, float dfix, float lo, float hi,
                                          bool fix_is_x, float& err) {
  // q(t) = ca dx^2 + 2 cb dx dy + cc dy^2 along an edge: dx (or dy) fixed, the other in [lo, hi]
  // the minimiser only picks the evaluation point: an approximate quotient moves q(t) by O(eps^2)
  // of the quadratic, far inside the cull's margins (k2m = 1.05 k2 + 0.05)
  float t = __fdividef(-cb * dfix, fix_is_x ? cc : ca);
  t = fminf(fmaxf(t, lo), hi);
  const float dx = fix_is_x ? dfix : t, dy = fix_is_x ? t : dfix;
  const float a = ca * dx * dx, b = 2.0f * cb * dx * dy, c = cc * dy * dy;
  err = fabsf(a) + fabsf(b) + fabsf(c);
  return a + b + c;
}

// Only the two edges nearer the centre are evaluated: with the centre mu outside the rectangle the
// minimiser d* of the convex q lies on a face whose outer side contains mu (else q would decrease
// from d* towards mu, inside the rectangle), i.e. on the nearer x-edge or the nearer y-edge; an
// extra edge checked where mu is inside that coordinate's range only adds a valid upper bound.
__device__ __forceinline__ bool ellipse_meets_rect(float2 mu, float4 co, float k2, float xlo, float xhi, float ylo,
                                                   float yhi) {
  if (mu.x >= xlo && mu.x <= xhi && mu.y >= ylo && mu.y <= yhi) return true;
  const float ca = co.x, cb = co.y, cc = co.z;
  const float ex = (mu.x < xlo ? xlo : xhi) - mu.x, ey = (mu.y < ylo ? ylo : yhi) - mu.y;
  float e0, e2;
  const float q0 = edge_min(ca, cb, cc, ex, ylo - mu.y, yhi - mu.y, true, e0);
  const float q2 = edge_min(ca, cb, cc, ey, xlo - mu.x, xhi - mu.x, false, e2);
  return (q0 - 1e-5f * e0 <= k2) || (q2 - 1e-5f * e2 <= k2);
}

// Per staged Gaussian: the scaled conic, a p2 threshold below which alpha < 1/255
// for certain (the exact test still decides every pair above it), and an EXACT
// conservative cull of the warp blocks: every pixel with alpha >= 1/255 has
// d^T conic d <= 2 ln(255 o), hence |dx| <= sqrt(2 ln(255 o) cov_xx) (R8), here
// with a 5% + 0.5 px margin that dominates the float error of the conic inverse.
struct StageCull {
  float rx, ry, k2m;  // bounding half-extents and the (margined) ellipse level of the cull
};

// The record of one staged Gaussian and its cull parameters.
__device__ __forceinline__ StageCull stage_record(float2 xy, float4 co, Rec& r) {
  const float4 sc = scaled_conic(co);
  r.a = make_float4(xy.x, xy.y, sc.x, sc.y);
  const float o = co.w;
  const float l2o = __log2f(255.0f * o);  // >= ~0 since o >= 1/255 for listed Gaussians
  r.b = make_float4(sc.z, o, -l2o - 0.01f, 0.0f);
  // det(conic) = ca cc - cb^2 with Kahan's FMA compensation (accurate to a few ulp even
  // for strongly anisotropic conics), then cov_xx = cc / det, cov_yy = ca / det.
  const float bb = co.y * co.y;
  const float det = __fmaf_rn(co.x, co.z, -bb) - __fmaf_rn(co.y, co.y, -bb);
  const float k2 = 2.0f * (fmaxf(l2o, 0.0f) * 0.6931472f + 0.01f) * 1.05f;
  const float kd = __fdividef(k2, det);
  const float rx = sqrtf(kd * co.z) + 0.5f;
  const float ry = sqrtf(kd * co.x) + 0.5f;
  const float k2m = k2 + 0.05f;
  return StageCull{rx, ry, k2m};
}

// Can the Gaussian reach a pixel centre of the rectangle [xlo, xhi] x [ylo, yhi]?
__device__ __forceinline__ bool block_hit(float2 xy, float4 co, const StageCull& c, float xlo, float xhi, float ylo,
                                          float yhi) {
  bool hit = (xy.x + c.rx >= xlo) && (xy.x - c.rx <= xhi) && (xy.y + c.ry >= ylo) && (xy.y - c.ry <= yhi);
  if (hit) hit = ellipse_meets_rect(xy, co, c.k2m, xlo, xhi, ylo, yhi);
  return hit;
}

// Record + bit mask of the warp blocks of the tile the Gaussian can reach.
template <int BW, int BH>
__device__ __forceinline__ uint32_t stage_gaussian(float2 xy, float4 co, float tile_x0, float tile_y0, Rec& r) {
  constexpr int NBX = 16 / BW, NB = NBX * (16 / BH);
  const StageCull c = stage_record(xy, co, r);
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < NB; ++k) {
    const float xlo = tile_x0 + (float)((k % NBX) * BW) + 0.5f, xhi = xlo + (float)(BW - 1);
    const float ylo = tile_y0 + (float)((k / NBX) * BH) + 0.5f, yhi = ylo + (float)(BH - 1);
    m |= (block_hit(xy, co, c, xlo, xhi, ylo, yhi) ? 1u : 0u) << k;
  }
  return m;
}

// 32-bit shared-window loads (the base address is computed once per kernel, so the
// hot loops do not re-derive the generic->shared mapping every iteration).
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

// per-thread asynchronous global -> shared copies (LDGSTS), completed by cp_async_wait_all
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ uint32_t lanemask_lt_() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Per-warp candidate lists of a staged batch of NT*EPT slots (slot e*NT + tid is
// thread tid's e-th entry, mask mk[e]): s_list[b*NT*EPT + ..] = the shared addresses
// rec_base + 16 slot of the ascending slots whose mask has bit b (the record planes' first
// plane; the loop reads a candidate's record with no address arithmetic), s_nw[b] = their count.  s_wc is [EPT*NW*NB] scratch.
// Contains the barriers that publish the staged records and the lists.
template <int NT, int EPT, int NB>
__device__ __forceinline__ void build_lists(const uint32_t (&mk)[EPT], uint32_t* s_list, uint32_t* s_wc,
                                            int* s_nw, uint32_t rec_base) {
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, sw = tid >> 5;
  const uint32_t lt = lanemask_lt_();
  uint32_t pos[EPT][NB];
#pragma unroll
  for (int e = 0; e < EPT; ++e)
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (mk[e] >> b) & 1u);
      pos[e][b] = __popc(bal & lt);
      if (lane == b) s_wc[(e * NW + sw) * NB + b] = __popc(bal);
    }
  __syncthreads();
  if (tid < NB) {
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < EPT * NW; ++k) {
      const uint32_t c = s_wc[k * NB + tid];
      s_wc[k * NB + tid] = acc;
      acc += c;
    }
    s_nw[tid] = (int)acc;
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < EPT; ++e)
#pragma unroll
    for (int b = 0; b < NB; ++b)
      if ((mk[e] >> b) & 1u) {
        PGSAG_DCHECK(s_wc[(e * NW + sw) * NB + b] + pos[e][b] < (uint32_t)(NT * EPT));
        s_list[b * (NT * EPT) + s_wc[(e * NW + sw) * NB + b] + pos[e][b]] = rec_base + 16u * (uint32_t)(e * NT + tid);
      }
  __syncthreads();
}

}  // namespace pgsag
