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
// recurrence of the oracle); the background term obeys the same
// recursion, so Sg = G.S + P (bg.gC) is one scalar started at bg.gC.
//
// Mapping: per active tile two single-warp CTAs, the one of half h
// owning the 8x16 pixel block of columns 8h..8h+7; a lane owns the FOUR pixels (x, y + 4k),
// k = 0..3, of its column, which share dx and every per-entry load and run as two packed FP32x2
// pairs.  Batches of 32 entries (one per lane; the next batch's inputs prefetched by cp.async)
// are staged with the exact block cull of A6 (per 8x8 block of the half: block p holds the
// lane's pair p; an entry past the block's deepest needed entry is culled for it too) and walked
// in reverse over the ballot of the culled slots; a pair whose block the entry misses, or none of
// whose 64 pixels blends it, is skipped by a warp-uniform branch.  A pixel that does not
// contribute to an entry carries alpha = rho = 0, which zeroes all of its terms and leaves its
// state unchanged without branches.  Reduction: per entry the
// lane sums its four pixels into 13 raw sums (the seven feature gradients sum alpha T G_c and the
// moments sum dpow {1, dx, dx^2, dy, dx dy, dy^2} of dpow = alpha dalpha; A8 turns the moments
// into the mean, conic and opacity gradients with the entry's conic and o), the warp transposes
// them through a 13 x 32 shared buffer and sums each row (lane r and r + 16 add half a row each,
// one shuffle joins the halves), and lane r stores row r's total in the batch accumulator.  After
// the batch the CTA flushes each entry's nonzero groups of four with one vector reduction
// (red.add.v4.f32) into the Gaussian's 64-byte line of the [n][16] accumulator.
#include <cuda_runtime.h>
#include <stdint.h>

#include "alpha.cuh"
#include "internal.cuh"

namespace pgsag {
namespace {

// One single-warp CTA per 8x16 half tile: the tile's entries are staged by both halves' CTAs,
// each culling against its own half, so there is no inter-warp barrier and no shared atomics, at
// twice the record loads (L2 hits).  (A two-warp CTA per tile sharing the staged batch measured
// slower in round 1: C4 A7 3.51 vs 3.41 ms.)
constexpr int kBT = 32;
constexpr int kBBatch = kBT;  // a batch is one entry per lane (64-entry batches measured 1.6 % slower)
#ifndef PGSAG_BWD_MINB
#define PGSAG_BWD_MINB 20  // resident CTAs per SM the register budget is sized for
#endif
constexpr float kLn2 = 0.6931471805599453f;


struct BwdArgs {
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
  const float *N, *D, *T;
  const int32_t *g, *last;
  const float *dC, *dN, *dD, *dA, *dDep;
  const double* nd_div;  // optional: dN, dDep divided by *nd_div
  float* g2d;  // [n][16] (kG2 used)
  int n;
  unsigned long long* counters;
  uint32_t* work;
  const float* gc_w;        // NEXT-1: L_GC-load weights, statistics and weight lambda
  const double* gc_stats;
  float gc_lambda;
};

constexpr float kGcK = 100.0f;  // soft-count sharpness (R24)

#ifdef PGSAG_A7_STATS
// diagnostic build only: per entry-warp work statistics of the candidate loop
__device__ unsigned long long g_a7_stats[32];
__device__ unsigned long long g_a7_t0 = ~0ull, g_a7_end[8192];  // kernel start, per-CTA end (globaltimer ns)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }
__device__ __forceinline__ float hsum(float2 a) { return a.x + a.y; }
__device__ __forceinline__ float ld_or0(const float* p, size_t k) { return p ? __ldg(p + k) : 0.0f; }

// Opaque copies: values the compiler would otherwise rematerialise inside the candidate loop
// (from S2R / integer-to-float sequences) under register pressure.
__device__ __forceinline__ float opaque(float x) {
  asm volatile("mov.b32 %0, %0;" : "+f"(x));
  return x;
}
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Per-pixel prologue: upstream G (Eq. 4 folded in), P*(bg.gC), last index, T.
struct PixState {
  float G[8];
  float Pb;
  float T;
  float gG;  // dL/d(soft count) of lambda * L_GC-load (R24)
  int last;
};

// inb: the pixel lies inside the image.  Every load is issued unconditionally (from pixel 0 when
// outside) and the mask applied by selection afterwards, so the loads of the lane's pixels overlap
// instead of waiting behind the mask test (one memory latency per tile).
__device__ __forceinline__ void load_pixel(const BwdArgs& a, bool inb, size_t pix, size_t HW, float px, float py,
                                           PixState& s) {
  const size_t q = inb ? pix : 0;
  const bool masked = inb && __ldg(a.mask + q) != 0;
  const int last = __ldg(a.last + q), gcount = __ldg(a.g + q);
  const float T = __ldg(a.T + q);
  float G[8];
  G[0] = ld_or0(a.dC, q); G[1] = ld_or0(a.dC, HW + q); G[2] = ld_or0(a.dC, 2 * HW + q);
  G[3] = ld_or0(a.dN, q); G[4] = ld_or0(a.dN, HW + q); G[5] = ld_or0(a.dN, 2 * HW + q);
  G[6] = ld_or0(a.dD, q);
  G[7] = ld_or0(a.dA, q);
  float gDep = ld_or0(a.dDep, q);
  const float N0 = __ldg(a.N + q), N1 = __ldg(a.N + HW + q), N2 = __ldg(a.N + 2 * HW + q), D = __ldg(a.D + q);
  const float w = a.gc_w ? __ldg(a.gc_w + q) : 1.0f;
  float gG = 0.f;
  if (a.gc_w) {  // Eq. 9: L = std(r), r = g / w  ->  dL/dg = (r - mean) / (N L w)
    const double Nn = a.gc_stats[0], L = a.gc_stats[3], mu = a.gc_stats[4];  // finalised after A6
    if (L > 0.0) gG = (float)((double)a.gc_lambda * ((double)gcount / w - mu) / (Nn * L * w));
  }
  if (a.nd_div) {  // sum-gradient of a mean loss: divide by its term count
    const double dv = *a.nd_div;
    const float sc = dv > 0.0 ? (float)(1.0 / dv) : 0.0f;
    G[3] *= sc; G[4] *= sc; G[5] *= sc;
    gDep *= sc;
  }
  // Eq. 4 prologue: Dep = D / (N . r); validity re-derived exactly as A6 did
  const float r0 = __fdiv_rn(__fsub_rn(px, a.cx), a.fx), r1 = __fdiv_rn(__fsub_rn(py, a.cy), a.fy);
  const float den = __fadd_rn(__fadd_rn(__fmul_rn(N0, r0), __fmul_rn(N1, r1)), N2);
  if (gcount > 0 && fabsf(den) > 1e-6f) {
    const float inv = 1.0f / den;
    G[6] += gDep * inv;
    const float c = gDep * D * inv * inv;
    G[3] -= c * r0; G[4] -= c * r1; G[5] -= c;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) s.G[c] = masked ? G[c] : 0.f;
  s.Pb = masked ? a.bg0 * G[0] + a.bg1 * G[1] + a.bg2 * G[2] : 0.f;
  s.T = masked ? T : 1.f;
  s.gG = masked ? gG : 0.f;
  s.last = masked ? last : -1;
}

// State of one packed pixel pair.
struct Pair {
  float2 G[8];
  float2 T, Sg, gGk;  // Sg = G.S + P (bg.gC) (one recursion for both, P' = (1 - alpha) P); gGk = k dL/d(soft count)
  int last0, last1;
};

__device__ __forceinline__ void make_pair(const PixState& a, const PixState& b, Pair& p) {
#pragma unroll
  for (int c = 0; c < 8; ++c) p.G[c] = f2(a.G[c], b.G[c]);
  p.gGk = f2(kGcK * a.gG, kGcK * b.gG);
  p.T = f2(a.T, b.T);
  p.Sg = f2(a.Pb, b.Pb);
  p.last0 = a.last;
  p.last1 = b.last;
}

// Per-entry per-pair partials: alpha T and dpow = alpha dalpha of the pair's two pixels.
struct PairOut {
  float2 wt, dpow;
};

template <bool kGC>
// al: the blended alphas (0 where the pixel does not blend the entry, which zeroes its d power
// too); u0 / u1: the pixel's alpha is not clamped (R16: d opacity and d power are zero through the
// clamp).  d opacity = rho dalpha = (alpha / o) dalpha is formed by A8 from sum dpow.
__device__ __forceinline__ void pair_grad(Pair& p, float2 al, bool u0, bool u1, const float4& cd, const float4& nn,
                                          PairOut& o) {
  const float2 om = __fadd2_rn(bc(1.f), f2(-al.x, -al.y));
  const float2 Ti = __fmul2_rn(p.T, f2(rcp_approx(om.x), rcp_approx(om.y)));
  float2 GF = p.G[7];
  GF = __ffma2_rn(p.G[0], bc(cd.x), GF);
  GF = __ffma2_rn(p.G[1], bc(cd.y), GF);
  GF = __ffma2_rn(p.G[2], bc(cd.z), GF);
  GF = __ffma2_rn(p.G[3], bc(nn.x), GF);
  GF = __ffma2_rn(p.G[4], bc(nn.y), GF);
  GF = __ffma2_rn(p.G[5], bc(nn.z), GF);
  GF = __ffma2_rn(p.G[6], bc(cd.w), GF);
  float2 dal = __fmul2_rn(Ti, __fadd2_rn(GF, f2(-p.Sg.x, -p.Sg.y)));
  if (kGC) {  // + gG * d(sigmoid(k (alpha - 1/255)))/d alpha; only reaches the outputs through ac / rc
    // z = -k log2(e) (alpha - 1/255), s = 1 / (1 + 2^z), 1 - s = 2^z s
    const float2 z = __ffma2_rn(al, bc(-kGcK * kLog2e), bc(kGcK * kLog2e * kAlphaMin));
    const float2 e = f2(ex2_approx(z.x), ex2_approx(z.y));
    const float2 s = f2(rcp_approx(1.0f + e.x), rcp_approx(1.0f + e.y));
    dal = __ffma2_rn(__fmul2_rn(p.gGk, s), __fmul2_rn(e, s), dal);
  }
  p.Sg = __ffma2_rn(al, GF, __fmul2_rn(om, p.Sg));
  p.T = Ti;
  o.wt = __fmul2_rn(al, Ti);
  const float2 dalu = f2(u0 ? dal.x : 0.f, u1 ? dal.y : 0.f);
  o.dpow = __fmul2_rn(al, dalu);
}

template <bool kCount, bool kGC, bool kAbs>
__global__ void __launch_bounds__(kBT, PGSAG_BWD_MINB) render_bwd_kernel(BwdArgs a) {
  constexpr int kNV = kAbs ? 14 : 13;  // raw sums per entry (g2d slots 0..kNV-1)
  constexpr int kAccStride = 16;       // one 64-byte row per entry: the flush's line
  constexpr int kRedStride = 36;       // transpose rows 4 banks apart: a lane's 128-bit loads of rows 0..7 do not collide
  // staged records as four float4 planes (SoA): the staging stores of consecutive slots are consecutive
  // 16-byte words (conflict-free), the candidate loop's broadcast loads take one address + offsets
  __shared__ float4 s_rec[4 * kBBatch];
  __shared__ uint32_t s_id[kBBatch];
  __shared__ __align__(16) float s_acc[(kBBatch + 1) * kAccStride];  // + a dummy row (no entry pending)
  __shared__ __align__(16) float s_red[14 * kRedStride];
  // the next batch's raw inputs (mean2d, conic_o, rgb_d, ncam), fetched by cp.async while this batch
  // runs; each lane writes and later reads only its own slot
  __shared__ float2 s_rxy[kBBatch];
  __shared__ float4 s_rco[kBBatch], s_rcd[kBBatch], s_rnn[kBBatch];
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t n_active = *a.n_active;
  const size_t HW = (size_t)a.d.W * a.d.H;
  const uint32_t rec_base = opaque(smem_u32(s_rec));
  unsigned long long cntV = 0;
#ifdef PGSAG_A7_STATS
  unsigned long long st[32] = {};
#endif
  // transpose: lane l writes column l of every row; lane l then sums half (l >> 4) of row l & 15
  // and, for l < kNV, stores the row's total
  const uint32_t red_w = opaque(smem_u32(s_red) + 4u * (uint32_t)lane);
  // (lanes past the last row re-read row kNV-1 with its lane: same address, no extra bank wavefront)
  const int my_row = (lane & 15) < kNV ? (lane & 15) : kNV - 1;
  const uint32_t red_r = opaque(smem_u32(s_red) + 4u * (uint32_t)(my_row * kRedStride + 16 * (lane >> 4)));
  const uint32_t acc_lane = opaque(smem_u32(s_acc) + 4u * (uint32_t)lane);
  const uint32_t wr = opaque((uint32_t)(lane < kNV));
  for (int k = tid; k < kBBatch * kAccStride; k += kBT) s_acc[k] = 0.f;
#ifdef PGSAG_A7_STATS
  if (tid == 0) atomicMin(&g_a7_t0, gtimer());
#endif
  if (tid == 0) s_tile = atomicAdd(a.work, 1u);
  for (;;) {
    __syncthreads();
    const uint32_t widx = s_tile;
    if (widx >= 2u * n_active) break;
    const uint32_t titem = widx >> 1;
    const int half = (int)(widx & 1u);  // which 8-column half of the tile
    const uint32_t tile = a.order ? a.order[titem] : a.active[titem];
    const int ty = tile / a.d.TX, tx = tile - ty * a.d.TX;
    const int i = tx * kTile + half * 8 + (lane & 7);
    const int jb = ty * kTile + (lane >> 3);
    const uint32_t rs = a.ranges[2 * tile];
    PGSAG_DCHECK(tile < (uint32_t)(a.d.TX * a.d.TY));
    const float px = opaque((float)i + 0.5f);
    const float2 py01 = f2(opaque((float)jb + 0.5f), opaque((float)(jb + 4) + 0.5f));
    const float2 py23 = f2(opaque((float)(jb + 8) + 0.5f), opaque((float)(jb + 12) + 0.5f));
    const float tx0 = (float)(tx * kTile), ty0 = (float)(ty * kTile);
    Pair P01, P23;
    {
      PixState s[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = jb + 4 * k;
        const size_t pix = (size_t)j * a.d.W + i;
        load_pixel(a, i < a.d.W && j < a.d.H, pix, HW, px, (float)j + 0.5f, s[k]);
      }
      make_pair(s[0], s[1], P01);
      make_pair(s[2], s[3], P23);
    }
    // the deepest entry each 8x8 block (pixel pair) needs: an entry past it skips the block's pair
    const int blast0 = __reduce_max_sync(0xffffffffu, max(P01.last0, P01.last1));
    const int blast1 = __reduce_max_sync(0xffffffffu, max(P23.last0, P23.last1));
    const int wlast = max(blast0, blast1);
    __syncthreads();
    const int maxlast = wlast;
    // every thread has read s_tile: claim the next tile now (latency hidden behind this one)
    if (tid == 0) s_tile = atomicAdd(a.work, 1u);
    // batches of 32 entries walked down from the deepest entry a pixel of the half needs.  Pipeline:
    // the raw inputs of batch k + 1 are in flight (cp.async) and the ids of batch k + 2 in a register
    // while batch k runs, so neither dependent global latency (vals -> records) stalls the warp.
    const auto fetch_raw = [&](uint32_t id) {
      cp_async8(smem_u32(s_rxy + tid), a.mean2d + id);
      cp_async16(smem_u32(s_rco + tid), a.conic_o + id);
      cp_async16(smem_u32(s_rcd + tid), a.rgb_d + id);
      cp_async16(smem_u32(s_rnn + tid), a.ncam + id);
    };
    const auto batch_lo = [&](int hi) { return max((int)rs, hi - kBBatch); };
    int bhi = maxlast + 1;
    uint32_t id_cur = 0u, id_n1 = 0u;
    if (bhi > (int)rs) {
      const int blo = batch_lo(bhi), blo1 = batch_lo(blo);
      if (tid < bhi - blo) {
        id_cur = a.vals[blo + tid];
        fetch_raw(id_cur);
      }
      cp_async_commit();
      if (tid < blo - blo1) id_n1 = a.vals[blo1 + tid];
    }
    for (; bhi > (int)rs; bhi -= kBBatch) {
      const int blo = batch_lo(bhi), cnt = bhi - blo;
      const int blo1 = batch_lo(blo), cnt1 = blo - blo1;
      const int blo2 = batch_lo(blo1), cnt2 = blo1 - blo2;
      uint32_t id_n2 = 0u;
      if (tid < cnt2) id_n2 = a.vals[blo2 + tid];  // consumed two batches from now
      cp_async_wait_all();
      uint32_t mk = 0u;
      if (tid < cnt) {
        const uint32_t id = id_cur;
        // the prefetched id is this batch's entry (the pipeline's bookkeeping) and a valid Gaussian
        PGSAG_DCHECK(id < (uint32_t)a.n && id == a.vals[blo + tid] && blo >= (int)rs && cnt <= kBBatch);
        Rec r;
        {  // this CTA's half only
          const float2 xy = s_rxy[tid];
          const float4 co = s_rco[tid];
          const StageCull c = stage_record(xy, co, r);
          const float xlo = tx0 + (float)(half * 8) + 0.5f, ylo = ty0 + 0.5f;
          // exact cull per 8x8 block of the half (block p = the rows of pixel pair p)
          const int kq = blo + tid;
          mk = (kq <= blast0 && block_hit(xy, co, c, xlo, xlo + 7.0f, ylo, ylo + 7.0f) ? 1u : 0u) |
               (kq <= blast1 && block_hit(xy, co, c, xlo, xlo + 7.0f, ylo + 8.0f, ylo + 15.0f) ? 2u : 0u);
          r.b.w = __uint_as_float(mk);
        }
        s_rec[tid] = r.a;
        s_rec[kBBatch + tid] = r.b;
        s_rec[2 * kBBatch + tid] = s_rcd[tid];
        s_rec[3 * kBBatch + tid] = s_rnn[tid];
        s_id[tid] = id;
      }
      // this lane's raw slot is consumed: fetch the next batch's into it
      if (tid < cnt1) fetch_raw(id_n1);
      cp_async_commit();
      id_cur = id_n1;
      id_n1 = id_n2;
      __syncwarp();  // the staged planes are visible to every lane
      // candidates: bit q = slot q reaches a block of the half; entries past the warp's last are
      // never needed.  Walked from the highest bit (back to front).
      uint32_t cm = __ballot_sync(0xffffffffu, mk != 0u);
      const int qtop = wlast - blo;
      if (qtop < 31) cm &= (2u << qtop) - 1u;
      // software pipeline over the candidates: the shuffle joining an entry's half-row sums is issued
      // at the top of the next candidate and its total stored after that candidate's alpha pass
      int pq = kBBatch;  // entry whose transposed rows await their sums (kBBatch: none, the dummy row)
      float hs = 0.f;  // this lane's half-row sum of entry pq
      while (cm != 0u) {
        const int q = 31 - __clz(cm);
        cm ^= 1u << q;
        const uint32_t ra_addr = rec_base + (uint32_t)q * 16u;
        const float4 ra = lds128(ra_addr);
        const float4 rb = lds128(ra_addr + 16 * kBBatch);
        PGSAG_DCHECK(q < cnt);
        const int kk = blo + q;
        // per 8x8 block (pixel pair) of the half: skipped when the splat misses it (staging cull)
        // or when none of its pixels blends the entry (a warp-uniform test after the alpha pass)
        const uint32_t smask = __float_as_uint(rb.w);
        const float dx = px - ra.x;
        const float tA = __fmul_rn(ra.z, dx);
        const float2 dy01 = __fadd2_rn(py01, bc(-ra.y));
        const float2 dy23 = __fadd2_rn(py23, bc(-ra.y));
        const float4 cd = lds128(ra_addr + 32 * kBBatch);
        const float4 nn = lds128(ra_addr + 48 * kBBatch);
        const float ho = __shfl_xor_sync(0xffffffffu, hs, 16);  // (unused when no entry is pending)
        PairOut o01, o23;  // zeroed where a pair is skipped (below)
#ifdef PGSAG_A7_STATS
        bool anyc = false;
        st[0]++;
        uint32_t stc = 0u;
        const uint32_t stb0 = st[4];
#endif
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          PairOut& OO = h ? o23 : o01;
          if (!((smask >> h) & 1u)) {
            OO.wt = OO.dpow = f2(0.f, 0.f);
            continue;
          }
          Pair& PP = h ? P23 : P01;
          const float2 dy = h ? dy23 : dy01;
          const float2 p2 = __ffma2_rn(bc(dx), __ffma2_rn(bc(ra.w), dy, bc(tA)), __fmul2_rn(__fmul2_rn(bc(rb.x), dy), dy));
          const float2 rh = f2(ex2_approx(p2.x), ex2_approx(p2.y));
          const float2 orh = __fmul2_rn(bc(rb.y), rh);
          float al0 = fminf(kAlphaMax, orh.x), al1 = fminf(kAlphaMax, orh.y);
          const bool c0 = kk <= PP.last0 && p2.x <= 0.0f && al0 >= kAlphaMin;
          const bool c1 = kk <= PP.last1 && p2.y <= 0.0f && al1 >= kAlphaMin;
          if (kCount) cntV += (unsigned long long)(kk <= PP.last0) + (kk <= PP.last1);
#ifdef PGSAG_A7_STATS
          st[2]++;
#endif
          if (!__any_sync(0xffffffffu, c0 || c1)) {
            OO.wt = OO.dpow = f2(0.f, 0.f);
            continue;
          }
#ifdef PGSAG_A7_STATS
          st[3]++;
          st[4] += __popc(__ballot_sync(0xffffffffu, c0)) + __popc(__ballot_sync(0xffffffffu, c1));
          stc |= __ballot_sync(0xffffffffu, c0 || c1);
          anyc = true;
#endif
          al0 = c0 ? al0 : 0.f;
          al1 = c1 ? al1 : 0.f;
          pair_grad<kGC>(PP, f2(al0, al1), orh.x <= kAlphaMax, orh.y <= kAlphaMax, cd, nn, OO);
        }
        PGSAG_DCHECK(pq <= kBBatch);
        if (wr) {  // one warp: (entry, row) has a single writer lane (none pending: the dummy row)
          const uint32_t addr = acc_lane + (uint32_t)pq * (uint32_t)(kAccStride * 4);
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(hs + ho) : "memory");
        }
        pq = kBBatch;
        // every candidate is summed (the ~7 % that no pixel blends transpose zeros): measured cheaper than
        // a branch on "any pair blended" per candidate
#ifdef PGSAG_A7_STATS
        if (anyc) {
          st[1]++;
          const int nl = __popc(stc), nb = (int)(st[4] - stb0);
          st[8 + (nl <= 1 ? 0 : nl <= 2 ? 1 : nl <= 4 ? 2 : nl <= 8 ? 3 : nl <= 16 ? 4 : 5)]++;
          st[16 + (nb <= 2 ? 0 : nb <= 4 ? 1 : nb <= 8 ? 2 : nb <= 16 ? 3 : nb <= 32 ? 4 : nb <= 64 ? 5 : 6)]++;
        }
#endif
        // the lane's raw sums (g2d slots): 0 S1 = sum dx dpow, 1 Sy = sum dy dpow, 2 S2 = sum dx^2 dpow,
        // 3 Sxy, 4 Syy, 5 S0 = sum dpow, 6..12 sum alpha T G_c, 13 (kAbs) sum |du| + |dv| per pixel;
        // dx is the lane's column offset, common to its four pixels
        float v[kNV];
#pragma unroll
        for (int c = 0; c < 7; ++c) v[6 + c] = hsum(__ffma2_rn(o23.wt, P23.G[c], __fmul2_rn(o01.wt, P01.G[c])));
        const float2 dydp01 = __fmul2_rn(dy01, o01.dpow), dydp23 = __fmul2_rn(dy23, o23.dpow);
        v[5] = hsum(__fadd2_rn(o01.dpow, o23.dpow));
        v[1] = hsum(__fadd2_rn(dydp01, dydp23));
        v[4] = hsum(__ffma2_rn(dy23, dydp23, __fmul2_rn(dy01, dydp01)));
        v[0] = dx * v[5];
        v[2] = dx * v[0];
        v[3] = dx * v[1];
        if (kAbs) {  // per-pixel du = -ln2 (B' dy + 2 A' dx) dpow, dv = -ln2 (2 C' dy + B' dx) dpow
          const float twoA = 2.0f * tA, bdx = ra.w * dx, twoC = 2.0f * rb.x;
          const float2 kd01 = __fmul2_rn(bc(-kLn2), o01.dpow), kd23 = __fmul2_rn(bc(-kLn2), o23.dpow);
          const float2 du01 = __fmul2_rn(__ffma2_rn(bc(ra.w), dy01, bc(twoA)), kd01);
          const float2 du23 = __fmul2_rn(__ffma2_rn(bc(ra.w), dy23, bc(twoA)), kd23);
          const float2 dv01 = __fmul2_rn(__ffma2_rn(bc(twoC), dy01, bc(bdx)), kd01);
          const float2 dv23 = __fmul2_rn(__ffma2_rn(bc(twoC), dy23, bc(bdx)), kd23);
          v[kNV - 1] = ((fabsf(du01.x) + fabsf(dv01.x)) + (fabsf(du01.y) + fabsf(dv01.y))) +
                       ((fabsf(du23.x) + fabsf(dv23.x)) + (fabsf(du23.y) + fabsf(dv23.y)));
        }
        // warp sums by a transpose through shared memory (single warp: __syncwarp orders it)
        __syncwarp();  // the previous entry's row reads are done
#pragma unroll
        for (int r = 0; r < kNV; ++r)
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(red_w + (uint32_t)(4 * r * kRedStride)), "f"(v[r]) : "memory");
        pq = q;
        __syncwarp();
        const float4 h0 = lds128(red_r), h1 = lds128(red_r + 16), h2 = lds128(red_r + 32), h3 = lds128(red_r + 48);
        const float2 t0 = __fadd2_rn(__fadd2_rn(f2(h0.x, h0.y), f2(h1.x, h1.y)), __fadd2_rn(f2(h0.z, h0.w), f2(h1.z, h1.w)));
        const float2 t1 = __fadd2_rn(__fadd2_rn(f2(h2.x, h2.y), f2(h3.x, h3.y)), __fadd2_rn(f2(h2.z, h2.w), f2(h3.z, h3.w)));
        hs = hsum(__fadd2_rn(t0, t1));
      }
      if (pq < kBBatch) {  // the batch's last transposed entry
        float sum = hs;
        sum += __shfl_xor_sync(0xffffffffu, sum, 16);
        if (wr) {
          const uint32_t addr = acc_lane + (uint32_t)pq * (uint32_t)(kAccStride * 4);
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(sum) : "memory");
        }
      }
      __syncwarp();
      // flush the batch: one vector reduction per nonzero group of four values, then re-zero
      if (tid < cnt) {
        float* dst = a.g2d + (size_t)s_id[tid] * 16;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float4* sp = reinterpret_cast<float4*>(s_acc + tid * kAccStride + 4 * c);
          const float4 x = *sp;
          if (x.x != 0.0f || x.y != 0.0f || x.z != 0.0f || x.w != 0.0f) {
            asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + 4 * c), "f"(x.x), "f"(x.y),
                         "f"(x.z), "f"(x.w)
                         : "memory");
            *sp = make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      }
      __syncwarp();
    }
  }
#ifdef PGSAG_A7_STATS
  if (lane == 0) {
    for (int k = 0; k < 32; ++k)
      if (st[k]) atomicAdd(&g_a7_stats[k], st[k]);
    if (blockIdx.x < 8192) g_a7_end[blockIdx.x] = gtimer();
  }
#endif
  if (kCount) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cntV += __shfl_xor_sync(0xffffffffu, cntV, o);
    if (lane == 0 && cntV) atomicAdd(a.counters + 2, cntV);
  }
}

int bwd_grid() {
  static int grid[kMaxDevices] = {};
  const int dev = current_device();
  if (!grid[dev]) {
    int sms = 148, occ = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, render_bwd_kernel<false, false, false>, kBT, 0);
    grid[dev] = sms * (occ > 0 ? occ : 1);
  }
  return grid[dev];
}

}  // namespace

cudaError_t launch_render_bwd(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                              const pgsag_bins* bins, const pgsag_tilemask* tm, const Dims& d,
                              const uint8_t* mask, const float bg[3], const pgsag_image* fwd,
                              const pgsag_image_grad* dL, pgsag_gaussian_grad* out, float* g2d,
                              uint32_t* work_counter, cudaStream_t st, pgsag_adam_state* adam,
                              const pgsag_adam_hparams* hp, double* flat, const uint32_t* skip) {
  const int n = g->n;
  if (n == 0) return cudaSuccess;
  cudaMemsetAsync(g2d, 0, sizeof(float) * 16 * (size_t)n, st);
  BwdArgs a;
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
  a.N = fwd->N; a.D = fwd->D; a.T = fwd->T; a.g = fwd->g; a.last = fwd->last;
  a.dC = dL->dC; a.dN = dL->dN; a.dD = dL->dD; a.dA = dL->dA; a.dDep = dL->dDep;
  a.nd_div = dL->nd_div;
  a.g2d = g2d;
  a.n = n;
  a.counters = fwd->counters;
  a.work = work_counter;
  const bool gc = dL->gc_lambda != 0.0f && fwd->gc_w && fwd->gc_stats;
  a.gc_w = gc ? fwd->gc_w : nullptr;
  a.gc_stats = fwd->gc_stats;
  a.gc_lambda = dL->gc_lambda;
  const int grid = min(bwd_grid(), d.TX * d.TY * 2);  // work items: half tiles
  {
    KTimer kt_("A7_render_bwd", st);
    const bool abs_ = out->absgrad2d || out->grad2d;
    const int variant = (fwd->counters ? 4 : 0) | (gc ? 2 : 0) | (abs_ ? 1 : 0);
    switch (variant) {
#define PGSAG_A7(V, C, G, A) \
  case V: render_bwd_kernel<C, G, A><<<grid, kBT, 0, st>>>(a); break;
      PGSAG_A7(0, false, false, false)
      PGSAG_A7(1, false, false, true)
      PGSAG_A7(2, false, true, false)
      PGSAG_A7(3, false, true, true)
      PGSAG_A7(4, true, false, false)
      PGSAG_A7(5, true, false, true)
      PGSAG_A7(6, true, true, false)
      PGSAG_A7(7, true, true, true)
#undef PGSAG_A7
    }
  }
  return launch_preprocess_bwd(g, cam, p, out, g2d, st, adam, hp, flat, skip);
}

}  // namespace pgsag

#ifdef PGSAG_A7_STATS
extern "C" int pgsag_debug_a7_times(unsigned long long* t0, unsigned long long* ends, int n) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(t0, pgsag::g_a7_t0, sizeof(unsigned long long));
  cudaMemcpyFromSymbol(ends, pgsag::g_a7_end, sizeof(unsigned long long) * (n < 8192 ? n : 8192));
  const unsigned long long big = ~0ull;
  cudaMemcpyToSymbol(pgsag::g_a7_t0, &big, sizeof(big));
  return 0;
}
extern "C" int pgsag_debug_a7_stats(unsigned long long* host, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, pgsag::g_a7_stats, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {};
    cudaMemcpyToSymbol(pgsag::g_a7_stats, z, sizeof(z));
  }
  return 0;
}
#endif
