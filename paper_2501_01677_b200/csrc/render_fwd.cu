// A6: masked forward compositor for sm_100a.
//
// P:79-92 Eq. 1-3 (front-to-back alpha blending of colour, camera-frame normal
// and plane distance), Eq. 4 (unbiased depth epilogue)
// (pixel-parallel rendering), P:243 (only building-mask pixels are computed).
//
// Mapping: a persistent grid pulls ACTIVE tiles (tiles with >= 1 mask pixel) from
// the A0 list through an atomic counter; masked-out tiles are never visited.  One
// 128-thread CTA per 16x16 tile: warp w owns an 8x8 pixel block, each lane the two
// pixels (x, y) and (x, y + 4) of its column, which share dx and every per-entry
// load; their arithmetic runs as packed FP32x2 (FFMA2/FMUL2/FADD2, one issue slot
// for both pixels).  Masked-out pixels start "done".  Each batch of 256 sorted
// entries is staged in shared memory (64-byte records, as four 16-byte planes) together with a 4-bit
// warp-block mask (exact conservative cull, alpha.cuh), from which every warp gets
// a compacted depth-ordered list of its candidates' record addresses (walked by pointer).
// Blending is branch-free (predicated weights); a warp stops when its pixels are done (tested
// every 16 candidates), the tile when every pixel is.
#include <cuda_runtime.h>
#include <stdint.h>

#include "alpha.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {


struct FwdArgs {
  const float2* mean2d;
  const float4* conic_o;
  const float4* rgb_d;
  const float4* ncam;
  const uint32_t* vals;
  const uint32_t* ranges;
  const uint32_t* active;
  const uint32_t* order;  // optional LPT work order (pgsag_bins.order)
  const uint32_t* n_active;
  const uint8_t* mask;
  Dims d;
  float fx, fy, cx, cy;
  float bg0, bg1, bg2;
  float *C, *N, *D, *A, *Dep, *T;
  int32_t *g, *last;
  unsigned long long* counters;
  uint32_t* work;
  const float* gc_w;   // optional L_GC-load weights (NEXT-1)
  double* gc_stats;    // N, sum r, sum r^2, L, mean (written by gc_finalize_kernel)
  double* gc_part;     // [kGcSlots][3] partial sums (workspace counter block)
  const uint32_t* n_dev;  // Gaussians of the sorted view (A3's CNT_NG; debug bounds checks)
};

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ __forceinline__ void write_pixel(const FwdArgs& a, size_t pix, size_t HW, float px, float py, float T,
                                            float C0, float C1, float C2, float N0, float N1, float N2, float D,
                                            int g, int last) {
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
}

// NP packed pixel pairs per lane: NP = 1 -> 8x8 warp blocks, 4 warps per tile (a lane owns
// rows y, y+4); NP = 2 -> 8x16 warp blocks, 2 warps per tile (rows y, y+4 | y+8, y+12), which
// amortises each candidate's list / record / address work over four pixels.
template <int NP>
struct FwdCfg {
  static constexpr int BH = 8 * NP;                // warp block height
  static constexpr int NT = 32 * 2 * (16 / BH);    // threads per tile CTA
  static constexpr int NB = NT / 32;               // warp blocks per tile
  static constexpr int EPT = 256 / NT;             // staged entries per thread (batch of 256)
  static constexpr int BATCH = NT * EPT;
};

#ifndef PGSAG_FWD_DONE_EVERY
#define PGSAG_FWD_DONE_EVERY 16  // candidates between two warp early-out tests (8: 0.7 % slower, 32: 0.2 %)
#endif
constexpr int kFwdDoneEvery = PGSAG_FWD_DONE_EVERY;
#ifndef PGSAG_FWD_MINB
#define PGSAG_FWD_MINB 8  // resident CTAs per SM the register budget is sized for (0: compiler choice; 7 CTAs at 72 regs measured 2 % slower)
#endif
#if PGSAG_FWD_MINB > 0
#define PGSAG_FWD_BOUNDS(NT) __launch_bounds__(NT, PGSAG_FWD_MINB)
#else
#define PGSAG_FWD_BOUNDS(NT) __launch_bounds__(NT)
#endif
template <bool kCount, int NP>
__global__ void PGSAG_FWD_BOUNDS(FwdCfg<NP>::NT) render_fwd_kernel(FwdArgs a) {
  using Cfg = FwdCfg<NP>;
  constexpr int NT = Cfg::NT, EPT = Cfg::EPT, NB = Cfg::NB, BATCH = Cfg::BATCH;
  __shared__ float4 s_rec[4 * BATCH];  // staged records as four float4 planes (conflict-free staging stores)
  __shared__ uint32_t s_list[NB * BATCH];  // candidate record addresses per warp block
  __shared__ uint32_t s_wc[EPT * (NT / 32) * NB];
  __shared__ int s_nw[NB];
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t n_active = *a.n_active;
  const size_t HW = (size_t)a.d.W * a.d.H;
  const uint32_t rec_base = smem_u32(s_rec), list_base = smem_u32(s_list);
  unsigned long long cntE = 0, cntB = 0;
  if (tid == 0) s_tile = atomicAdd(a.work, 1u);
  for (;;) {
    __syncthreads();  // s_tile published
    const uint32_t widx = s_tile;
    __syncthreads();  // read by every thread
    if (widx >= n_active) break;
    // claim the next tile now: the atomic's latency hides behind this tile's work
    if (tid == 0) s_tile = atomicAdd(a.work, 1u);
    const uint32_t tile = a.order ? a.order[widx] : a.active[widx];
    const int ty = tile / a.d.TX, tx = tile - ty * a.d.TX;
    const int i = tx * kTile + (w & 1) * 8 + (lane & 7);
    const int jb = ty * kTile + (w >> 1) * Cfg::BH + (lane >> 3);
    const uint32_t rs = a.ranges[2 * tile], re = a.ranges[2 * tile + 1];
    PGSAG_DCHECK(tile < (uint32_t)(a.d.TX * a.d.TY) && rs <= re);
    const float px = (float)i + 0.5f;
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
    // per pair p: rows jb + 8p and jb + 8p + 4.  T carries the pixel's "done" state in its
    // sign: T > 0 while compositing, T = -(final T) once stopped (-1 if not a mask pixel).
    bool m[NP][2];
    size_t pix[NP][2];
    float2 py[NP], T[NP], C0[NP], C1[NP], C2[NP], N0[NP], N1[NP], N2[NP], D[NP], gc[NP];
    int last[NP][2];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = jb + 8 * p + 4 * h;
        pix[p][h] = (size_t)j * a.d.W + i;
        m[p][h] = i < a.d.W && j < a.d.H && a.mask[pix[p][h]] != 0;
        last[p][h] = -1;
      }
      py[p] = f2((float)(jb + 8 * p) + 0.5f, (float)(jb + 8 * p + 4) + 0.5f);
      T[p] = f2(m[p][0] ? 1.f : -1.f, m[p][1] ? 1.f : -1.f);
      C0[p] = C1[p] = C2[p] = N0[p] = N1[p] = N2[p] = D[p] = gc[p] = f2(0.f, 0.f);
    }
    auto all_done = [&]() {
      bool d = true;
#pragma unroll
      for (int p = 0; p < NP; ++p) d = d && T[p].x < 0.f && T[p].y < 0.f;
      return d;
    };
    for (uint32_t b = rs; b < re; b += BATCH) {
      if (__syncthreads_count(all_done()) == NT) break;
      uint32_t mk[EPT];
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const uint32_t k = b + e * NT + tid;
        mk[e] = 0u;
        if (k < re) {
          const uint32_t id = a.vals[k];
          PGSAG_DCHECK(id < *a.n_dev);
          Rec r;
          mk[e] = stage_gaussian<8, Cfg::BH>(a.mean2d[id], a.conic_o[id], tx0, ty0, r);
          r.b.w = (float)(e * NT + tid);  // slot in the batch, for the blend's last index
          const int slot = e * NT + tid;
          s_rec[slot] = r.a;
          s_rec[BATCH + slot] = r.b;
          s_rec[2 * BATCH + slot] = a.rgb_d[id];
          s_rec[3 * BATCH + slot] = a.ncam[id];
        }
      }
      build_lists<NT, EPT, NB>(mk, s_list, s_wc, s_nw, rec_base);
      const int nw = s_nw[w];
      // batch slot of each pixel's last blend in this batch (-1: none), kept on the FMA pipe
      float2 lastf[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) lastf[p] = f2(-1.f, -1.f);
      const uint32_t lbase = list_base + (uint32_t)(4 * w * BATCH), lend = lbase + 4u * (uint32_t)nw;
      for (uint32_t l0 = lbase; l0 < lend; l0 += 4u * kFwdDoneEvery) {  // the warp's early-out test once per kFwdDoneEvery candidates
        if (__all_sync(0xffffffffu, all_done())) break;
        const uint32_t l1 = min(l0 + 4u * kFwdDoneEvery, lend);
        for (uint32_t la = l0; la < l1; la += 4u) {
          uint32_t ra_addr;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(ra_addr) : "r"(la));
          PGSAG_DCHECK(b + (ra_addr - rec_base) / 16u < re);
          const float4 ra = lds128(ra_addr);
          const float4 rb = lds128(ra_addr + 16 * BATCH);
          const float dx = px - ra.x;
          const float tA = __fmul_rn(ra.z, dx);
          const float4 cd = lds128(ra_addr + 32 * BATCH);
          const float4 nn = lds128(ra_addr + 48 * BATCH);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            // p2 for the pair (bit-identical to power2r per element)
            const float2 dy = __fadd2_rn(py[p], f2(-ra.y, -ra.y));
            const float2 u = __ffma2_rn(f2(ra.w, ra.w), dy, f2(tA, tA));
            const float2 cq = __fmul2_rn(__fmul2_rn(f2(rb.x, rb.x), dy), dy);
            const float2 p2 = __ffma2_rn(f2(dx, dx), u, cq);
            const float2 orho = __fmul2_rn(f2(rb.y, rb.y), f2(ex2_approx(p2.x), ex2_approx(p2.y)));
            const float al0 = fminf(kAlphaMax, orho.x), al1 = fminf(kAlphaMax, orho.y);
            if (kCount) cntE += (unsigned long long)(T[p].x > 0.f) + (unsigned long long)(T[p].y > 0.f);
            // e = alpha passes (R6); ok = blends (e and T stays >= 1e-4: a done pixel has T < 0, so
            // Tn < 0 and it never blends); e && !ok = terminates here, T <- -|T| (idempotent once done)
            const bool e0 = p2.x <= 0.0f && al0 >= kAlphaMin;
            const bool e1 = p2.y <= 0.0f && al1 >= kAlphaMin;
            const float2 Tn = __fmul2_rn(T[p], __fadd2_rn(f2(1.f, 1.f), f2(-al0, -al1)));
            const bool ok0 = e0 && Tn.x >= kTmin, ok1 = e1 && Tn.y >= kTmin;
            // branch-free blend (predicated weights): no loop-carried phi copies.  The blend
            // indicator (alpha >= 1/255 > 0 when blended) is formed by a saturating multiply on
            // the FMA pipe and drives the blend count and the last slot (the ALU pipe is the
            // limiter here)
            const float2 als = f2(ok0 ? al0 : 0.f, ok1 ? al1 : 0.f);
            const float2 okf = f2(__saturatef(als.x * 1e30f), __saturatef(als.y * 1e30f));
            const float2 wt = __fmul2_rn(als, T[p]);
            C0[p] = __ffma2_rn(wt, f2(cd.x, cd.x), C0[p]);
            C1[p] = __ffma2_rn(wt, f2(cd.y, cd.y), C1[p]);
            C2[p] = __ffma2_rn(wt, f2(cd.z, cd.z), C2[p]);
            D[p] = __ffma2_rn(wt, f2(cd.w, cd.w), D[p]);
            N0[p] = __ffma2_rn(wt, f2(nn.x, nn.x), N0[p]);
            N1[p] = __ffma2_rn(wt, f2(nn.y, nn.y), N1[p]);
            N2[p] = __ffma2_rn(wt, f2(nn.z, nn.z), N2[p]);
            T[p].x = ok0 ? Tn.x : (e0 ? -fabsf(T[p].x) : T[p].x);
            T[p].y = ok1 ? Tn.y : (e1 ? -fabsf(T[p].y) : T[p].y);
            gc[p] = __fadd2_rn(gc[p], okf);  // blend counts (exact below 2^24)
            // lastf <- okf ? slot : lastf, exactly (small integers)
            lastf[p] = __ffma2_rn(okf, __fadd2_rn(f2(rb.w, rb.w), f2(-lastf[p].x, -lastf[p].y)), lastf[p]);
          }
        }
      }
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        if (lastf[p].x >= 0.f) last[p][0] = (int)b + (int)lastf[p].x;
        if (lastf[p].y >= 0.f) last[p][1] = (int)b + (int)lastf[p].y;
      }
    }
    float n = 0.f, s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float Tf = fabsf(h ? T[p].y : T[p].x);
        const int g = (int)(h ? gc[p].y : gc[p].x);
        const float py_ = h ? py[p].y : py[p].x;
        if (m[p][h]) {
          write_pixel(a, pix[p][h], HW, px, py_, Tf, h ? C0[p].y : C0[p].x, h ? C1[p].y : C1[p].x,
                      h ? C2[p].y : C2[p].x, h ? N0[p].y : N0[p].x, h ? N1[p].y : N1[p].x, h ? N2[p].y : N2[p].x,
                      h ? D[p].y : D[p].x, g, last[p][h]);
          if (a.gc_w) {  // fused Eq. 9 statistics over the mask pixels of this tile (NEXT-1)
            const float r = (float)g / __ldg(a.gc_w + pix[p][h]);
            n += 1.f; s1 += r; s2 += r * r;
          }
          if (kCount) cntB += (unsigned long long)g;
        }
      }
    }
    if (a.gc_w) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        n += __shfl_xor_sync(0xffffffffu, n, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      if (lane == 0 && n > 0.f) {
        double* slot = a.gc_part + 3 * (blockIdx.x % kGcSlots);
        atomicAdd(slot, (double)n);
        atomicAdd(slot + 1, (double)s1);
        atomicAdd(slot + 2, (double)s2);
      }
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

#ifndef PGSAG_FWD_NP
#define PGSAG_FWD_NP 1
#endif
constexpr int kNP = PGSAG_FWD_NP;
constexpr int kFT = FwdCfg<kNP>::NT;

// Eq. 9 from the fused statistics: L_GC-load = population std of r = g / w over the mask pixels.
__global__ void gc_finalize_kernel(double* st, const double* part) {
  double acc[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < kGcSlots; ++k)
    for (int c = 0; c < 3; ++c) acc[c] += part[3 * k + c];
  st[0] = acc[0];
  st[1] = acc[1];
  st[2] = acc[2];
  const double n = st[0];
  const double mu = n > 0.0 ? st[1] / n : 0.0;
  st[3] = n > 0.0 ? sqrt(fmax(st[2] / n - mu * mu, 0.0)) : 0.0;
  st[4] = mu;
}

int fwd_grid() {
  static int grid[kMaxDevices] = {};
  const int dev = current_device();
  if (!grid[dev]) {
    int sms = 148, occ = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, render_fwd_kernel<false, kNP>, kFT, 0);
    grid[dev] = sms * (occ > 0 ? occ : 1);
  }
  return grid[dev];
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
  a.order = bins->order;
  a.n_active = tm->n_active;
  a.mask = mask;
  a.d = d;
  a.fx = cam->fx; a.fy = cam->fy; a.cx = cam->cx; a.cy = cam->cy;
  a.bg0 = bg[0]; a.bg1 = bg[1]; a.bg2 = bg[2];
  a.C = out->C; a.N = out->N; a.D = out->D; a.A = out->A; a.Dep = out->Dep; a.T = out->T;
  a.g = out->g; a.last = out->last;
  a.counters = out->counters;
  a.work = work_counter;
  a.gc_w = out->gc_w;
  a.gc_stats = out->gc_stats;
  a.n_dev = work_counter + (CNT_NG - CNT_FWD);
  a.gc_part = reinterpret_cast<double*>(work_counter + (CNT_GCF - CNT_FWD));
  if (a.gc_w) cudaMemsetAsync(a.gc_part, 0, 3 * kGcSlots * sizeof(double), st);
  const int grid = min(fwd_grid(), d.TX * d.TY);
  {
    KTimer kt_("A6_render_fwd", st);
    if (out->counters)
      render_fwd_kernel<true, kNP><<<grid, kFT, 0, st>>>(a);
    else
      render_fwd_kernel<false, kNP><<<grid, kFT, 0, st>>>(a);
  }
  if (a.gc_w) {
    KTimer kt_("N1_gc_finalize", st);
    gc_finalize_kernel<<<1, 1, 0, st>>>(a.gc_stats, a.gc_part);
  }
  return cudaGetLastError();
}

}  // namespace pgsag
