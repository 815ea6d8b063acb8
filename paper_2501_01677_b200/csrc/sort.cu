// A2-A5 on sm_100a: depth sort, scan, key duplication, tile radix sort, ranges.
//
// P:78 "projected onto different image tiles. The 2D Gaussians are subsequently
// sorted" — realised as the TWO-STAGE equivalent of the 3DGS (tile|depth) 64-bit
// key sort: (1) stable LSD sort of the N Gaussians by depth bits
// (32 bits), (2) duplication in depth order into (tile, id) entries, (3) stable
// LSD sort of the M entries by tile id only (ceil(log2 #tiles) bits).  The result
// is exactly the (tile, depth bits, id) order with ~4x fewer bytes moved per entry
// than a 64-bit key sort.
//
// The radix sort is a hand-written onesweep (single read + single write per pass):
// each CTA ranks a 4096-key tile with warp match_any, publishes per-digit counts,
// and resolves its global digit offsets by decoupled look-back over predecessor
// CTAs (tile ids are taken from an atomic counter, so a CTA only ever waits on
// CTAs that started before it).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pgsag {
namespace {

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) { return *(const volatile uint32_t*)p; }
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) { *(volatile uint32_t*)p = v; }
__device__ __forceinline__ unsigned long long ld_volatile64(const unsigned long long* p) {
  return *(const volatile unsigned long long*)p;
}
__device__ __forceinline__ void st_volatile64(unsigned long long* p, unsigned long long v) {
  *(volatile unsigned long long*)p = v;
}

// exclusive scan of one value per thread across a 256-thread CTA; returns the CTA total
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& excl) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  uint32_t wbase = 0, total = 0;
#pragma unroll
  for (int k = 0; k < NT / 32; ++k) {
    const uint32_t t = s_warp[k];
    if (k < w) wbase += t;
    total += t;
  }
  excl = wbase + x - v;
  __syncthreads();
  return total;
}

// ------------------------------------------------------------ pass plan
// Digit widths of an LSD sort over `bits` key bits: 8-bit digits, or 9-bit ones
// where that saves a pass (17-18 bits: 2 passes instead of 3; 25-27: 3 instead of 4).  At 17 bits the
// 9-bit digit is the high one: its bins are the sparsely used ones (tile rows), which the pass skips.
struct PassPlan {
  int n;
  int shift[kMaxSortPasses];
  int width[kMaxSortPasses];
};

PassPlan make_plan(int bits) {
  PassPlan p;
  p.n = 0;
  int w[kMaxSortPasses];
  if (bits <= 0) return p;
  if (bits <= 9) { w[0] = bits; p.n = 1; }
  else if (bits <= 16) { w[0] = 8; w[1] = bits - 8; p.n = 2; }
  else if (bits <= 17) { w[0] = 8; w[1] = bits - 8; p.n = 2; }  // the wide digit on the sparse high bits
  else if (bits <= 18) { w[0] = 9; w[1] = bits - 9; p.n = 2; }
  else if (bits <= 24) { w[0] = 8; w[1] = 8; w[2] = bits - 16; p.n = 3; }
  else if (bits <= 27) { w[0] = 9; w[1] = 9; w[2] = bits - 18; p.n = 3; }
  else { w[0] = 8; w[1] = 8; w[2] = 8; w[3] = bits - 24; p.n = 4; }
  int s = 0;
  for (int k = 0; k < p.n; ++k) { p.shift[k] = s; p.width[k] = w[k]; s += w[k]; }
  return p;
}

// ------------------------------------------------------------ histogram
// Digit histograms of all passes at once (onesweep's upfront pass); ghist is
// [pass][kMaxRadix].  (Warp-aggregating the shared-memory counts with match_any was measured 4x
// slower.)  kFromDepth (stage 1): the keys are formed here from A1's outputs -- the depth bits of Gaussians
// that emit entries, all-ones (sorted last) otherwise; z > znear > 0, so bit order is value order
// -- and written out with the identity ids for the first pass.
template <bool kFromDepth>
__global__ void __launch_bounds__(256) radix_hist_kernel(const uint32_t* __restrict__ keys_in,
                                                          const uint32_t* __restrict__ n_ptr, uint32_t n_fixed,
                                                          PassPlan plan, uint32_t* __restrict__ ghist,
                                                          const float* __restrict__ depth,
                                                          const uint32_t* __restrict__ touched,
                                                          uint32_t* __restrict__ keys_out,
                                                          uint32_t* __restrict__ ids_out) {
  __shared__ uint32_t sh[kMaxSortPasses][kMaxRadix];
  const uint32_t n = n_ptr ? min(*n_ptr, n_fixed) : n_fixed;
  for (int k = threadIdx.x; k < kMaxSortPasses * kMaxRadix; k += blockDim.x) (&sh[0][0])[k] = 0;
  __syncthreads();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {  // warp-uniform trip count
    const uint32_t idx = base + threadIdx.x;
    const bool live = idx < n;
    uint32_t key = 0xFFFFFFFFu;
    if (live) {
      if (kFromDepth) {
        key = touched[idx] > 0 ? __float_as_uint(depth[idx]) : 0xFFFFFFFFu;
        keys_out[idx] = key;
        ids_out[idx] = idx;
      } else {
        key = keys_in[idx];
      }
    }
    if (live)
      for (int p = 0; p < plan.n; ++p) atomicAdd(&sh[p][(key >> plan.shift[p]) & ((1u << plan.width[p]) - 1u)], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < plan.n * kMaxRadix; k += blockDim.x) {
    const uint32_t v = (&sh[0][0])[k];
    if (v) atomicAdd(ghist + k, v);
  }
}

// Stage 2 (the tile keys of A3): a thread counts one contiguous span of the keys, run-length
// aggregated per pass in registers -- A3 emits each splat's tiles in row-major runs, so the high
// digit (the tile row) is constant over long runs that would otherwise hit one shared counter with
// 32-way conflicts (heavy-tailed C5 facades) -- and adds each run with one shared atomic.
__global__ void __launch_bounds__(256) radix_hist_runs_kernel(const uint32_t* __restrict__ keys,
                                                               const uint32_t* __restrict__ n_ptr, uint32_t n_fixed,
                                                               PassPlan plan, uint32_t* __restrict__ ghist) {
  __shared__ uint32_t sh[kMaxSortPasses][kMaxRadix];
  const uint32_t n = n_ptr ? min(*n_ptr, n_fixed) : n_fixed;
  for (int k = threadIdx.x; k < kMaxSortPasses * kMaxRadix; k += blockDim.x) (&sh[0][0])[k] = 0;
  __syncthreads();
  const uint32_t nt = gridDim.x * blockDim.x, t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t span = ((n + nt - 1) / nt + 3u) & ~3u;  // multiple of 4: aligned uint4 loads
  const uint32_t k0 = t * span, k1 = min(n, k0 + span);
  uint32_t cur[kMaxSortPasses], run[kMaxSortPasses];
#pragma unroll
  for (int p = 0; p < kMaxSortPasses; ++p) { cur[p] = 0xFFFFFFFFu; run[p] = 0u; }
  auto add = [&](uint32_t key) {
#pragma unroll
    for (int p = 0; p < kMaxSortPasses; ++p) {
      if (p >= plan.n) break;
      const uint32_t dg = (key >> plan.shift[p]) & ((1u << plan.width[p]) - 1u);
      if (dg != cur[p]) {
        if (run[p]) atomicAdd(&sh[p][cur[p]], run[p]);
        cur[p] = dg;
        run[p] = 0u;
      }
      ++run[p];
    }
  };
  uint32_t k = k0;
  for (; k + 4 <= k1; k += 4) {
    const uint4 v = *reinterpret_cast<const uint4*>(keys + k);
    add(v.x); add(v.y); add(v.z); add(v.w);
  }
  for (; k < k1; ++k) add(keys[k]);
#pragma unroll
  for (int p = 0; p < kMaxSortPasses; ++p)
    if (p < plan.n && run[p]) atomicAdd(&sh[p][cur[p]], run[p]);
  __syncthreads();
  for (int q = threadIdx.x; q < plan.n * kMaxRadix; q += blockDim.x) {
    const uint32_t v = (&sh[0][0])[q];
    if (v) atomicAdd(ghist + q, v);
  }
}

// ------------------------------------------------------------ onesweep pass
template <int RB>
constexpr size_t pass_smem() {
  return sizeof(uint32_t) * (2 * kSortTile + (kSortThreads / 32 + 2) * (1 << RB));
}

template <int RB>
#ifndef PGSAG_SORT_MINB
#define PGSAG_SORT_MINB 4  // 3 measured 1.4 % slower on the C4 sort chain
#endif
__global__ void __launch_bounds__(kSortThreads, PGSAG_SORT_MINB) radix_pass_kernel(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    uint32_t* __restrict__ vals_out, const uint32_t* __restrict__ n_ptr, uint32_t n_fixed, int shift, int nbits,
    const uint32_t* __restrict__ ghist, uint32_t* __restrict__ status, uint32_t* __restrict__ tile_counter) {
  constexpr int NW = kSortThreads / 32;
  constexpr int R = 1 << RB;
  constexpr int DPT = R / kSortThreads;  // digits per thread (1 or 2)
  extern __shared__ uint32_t sm[];
  uint32_t* s_keys = sm;
  uint32_t* s_vals = s_keys + kSortTile;
  uint32_t* s_whist = s_vals + kSortTile;  // [NW][R]
  uint32_t* s_cta_start = s_whist + NW * R;
  uint32_t* s_gbase = s_cta_start + R;
  __shared__ uint32_t s_warp[NW];
  __shared__ uint32_t s_tile;

  const uint32_t n = n_ptr ? min(*n_ptr, n_fixed) : n_fixed;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int k = tid; k < NW * R; k += kSortThreads) s_whist[k] = 0;
  for (int k = tid; k < R; k += kSortThreads) s_cta_start[k] = 0;  // the CTA's digit counts first
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * (uint32_t)kSortTile;
  if (base >= n) return;  // whole CTA: uniform
  const uint32_t mask = (1u << nbits) - 1u;

  uint32_t key[kSortItems], val[kSortItems], rank[kSortItems];
  const uint32_t wbase = base + (uint32_t)w * 32u * kSortItems;
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const uint32_t idx = wbase + (uint32_t)k * 32u + lane;
    if (idx < n) {
      key[k] = keys_in[idx];
      val[k] = vals_in[idx];
    } else {
      key[k] = 0xFFFFFFFFu;
      val[k] = 0u;
    }
  }
  // the CTA's digit counts (cheap shared atomics), published for the successors' look-back
  // BEFORE the expensive stable ranking: a CTA's successors then never wait on its ranking
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const uint32_t idx = wbase + (uint32_t)k * 32u + lane;
    if (idx < n) atomicAdd(&s_cta_start[(key[k] >> shift) & mask], 1u);
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int dgt = tid * DPT + j;
    if (ghist[dgt])  // a digit no key of the whole input has needs no look-back state
      st_volatile(status + (size_t)tile * R + dgt, (tile == 0 ? kLbPrefix : kLbAgg) | s_cta_start[dgt]);
  }
  const uint32_t lt = lanemask_lt();
  // stable warp-local ranking: item-major, lane-minor == input order
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const uint32_t idx = wbase + (uint32_t)k * 32u + lane;
    const uint32_t dg = idx < n ? ((key[k] >> shift) & mask) : (uint32_t)R;
    const uint32_t peers = __match_any_sync(0xffffffffu, dg);
    const uint32_t r = __popc(peers & lt);
    // the peers' leader takes the group's counts with one shared atomic (in item order: a warp's
    // shared-memory atomics on one address complete in issue order) and broadcasts the base
    const int leader = __ffs(peers) - 1;
    uint32_t prev = 0u;
    if (r == 0 && dg < (uint32_t)R) prev = atomicAdd(&s_whist[w * R + dg], (uint32_t)__popc(peers));
    prev = __shfl_sync(0xffffffffu, prev, leader);
    rank[k] = prev + r;
  }
  __syncthreads();
  // per digit (DPT consecutive digits per thread): exclusive offsets across warps,
  // CTA total, decoupled look-back over predecessor CTAs
  uint32_t tot[DPT], excl[DPT], gh[DPT];
  uint32_t tsum = 0, gsum = 0;
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int dgt = tid * DPT + j;
    uint32_t total = 0;
#pragma unroll
    for (int k = 0; k < NW; ++k) {
      const uint32_t t = s_whist[k * R + dgt];
      s_whist[k * R + dgt] = total;
      total += t;
    }
    tot[j] = total;
    tsum += total;
    gh[j] = ghist[dgt];
    gsum += gh[j];
  }
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int dgt = tid * DPT + j;
    uint32_t ex = 0;
    if (tile != 0 && gh[j] != 0) {
      int q = (int)tile - 1;
      while (q >= 0) {
        uint32_t s;
        do { s = ld_volatile(status + (size_t)q * R + dgt); } while ((s & ~kLbMask) == 0u);
        ex += s & kLbMask;
        if (s & kLbPrefix) break;
        --q;
      }
      st_volatile(status + (size_t)tile * R + dgt, kLbPrefix | (ex + tot[j]));
    }
    excl[j] = ex;
  }
  // global start of each digit = (exclusive scan of ghist) + excl; CTA-local starts
  uint32_t gex, cex;
  block_excl_scan<kSortThreads>(gsum, s_warp, gex);
  block_excl_scan<kSortThreads>(tsum, s_warp, cex);
#pragma unroll
  for (int j = 0; j < DPT; ++j) {
    const int dgt = tid * DPT + j;
    s_gbase[dgt] = gex + excl[j];
    s_cta_start[dgt] = cex;
    gex += gh[j];
    cex += tot[j];
  }
  __syncthreads();
  // scatter into shared memory in CTA-local sorted order
#pragma unroll
  for (int k = 0; k < kSortItems; ++k) {
    const uint32_t idx = wbase + (uint32_t)k * 32u + lane;
    if (idx < n) {
      const uint32_t dg = (key[k] >> shift) & mask;
      const uint32_t pos = s_cta_start[dg] + s_whist[w * R + dg] + rank[k];
      PGSAG_DCHECK(pos < (uint32_t)kSortTile);
      s_keys[pos] = key[k];
      s_vals[pos] = val[k];
    }
  }
  __syncthreads();
  const uint32_t cnt = min((uint32_t)kSortTile, n - base);
  for (uint32_t p = tid; p < cnt; p += kSortThreads) {
    const uint32_t k = s_keys[p];
    const uint32_t dg = (k >> shift) & mask;
    const uint32_t dst = s_gbase[dg] + (p - s_cta_start[dg]);
    PGSAG_DCHECK(dst < n);
    keys_out[dst] = k;
    vals_out[dst] = s_vals[p];
  }
}

// ---------------------------------------------------------------- A2 scan
// Single-pass decoupled-look-back exclusive scan of touched[ids[k]] (depth
// order).  Writes offsets[k] and the total M (u64) to *total.
__global__ void __launch_bounds__(256) scan_kernel(int n, const uint32_t* __restrict__ touched,
                                                    const uint32_t* __restrict__ ids,
                                                    uint32_t* __restrict__ offsets,
                                                    unsigned long long* __restrict__ status,
                                                    uint32_t* __restrict__ tile_counter,
                                                    unsigned long long* __restrict__ total) {
  constexpr int IT = kScanTile / 256;
  constexpr int PAD = IT + 1;  // padded rows: the blocked reads of the transpose are conflict-free
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_tile;
  __shared__ unsigned long long s_excl;
  __shared__ uint32_t s_v[256 * PAD];
  const int tid = threadIdx.x;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kScanTile;
  if (base >= (uint32_t)n) return;
  // striped (coalesced) loads of the ids and their counts, transposed through shared memory so
  // that each thread then owns IT consecutive items
#pragma unroll
  for (int k = 0; k < IT; ++k) {
    const uint32_t j = (uint32_t)(k * 256 + tid);
    const uint32_t idx = base + j;
    s_v[(j / IT) * PAD + j % IT] = idx < (uint32_t)n ? __ldg(touched + ids[idx]) : 0u;
  }
  __syncthreads();
  uint32_t v[IT];
  uint32_t sum = 0;
#pragma unroll
  for (int k = 0; k < IT; ++k) {
    v[k] = s_v[tid * PAD + k];
    sum += v[k];
  }
  uint32_t texcl;
  const uint32_t agg = block_excl_scan<256>(sum, s_warp, texcl);
  constexpr unsigned long long AGG = 1ull << 62, PRE = 2ull << 62, MASK = (1ull << 62) - 1;
  if (tid == 0) {
    unsigned long long ex = 0;
    if (tile == 0) {
      st_volatile64(status, PRE | agg);
    } else {
      st_volatile64(status + tile, AGG | agg);
      int j = (int)tile - 1;
      while (j >= 0) {
        unsigned long long s;
        do { s = ld_volatile64(status + j); } while ((s & ~MASK) == 0ull);
        ex += s & MASK;
        if (s & PRE) break;
        --j;
      }
      st_volatile64(status + tile, PRE | (ex + agg));
    }
    s_excl = ex;
    if (base + kScanTile >= (uint32_t)n) *total = ex + agg;
  }
  __syncthreads();
  uint32_t run = (uint32_t)s_excl + texcl;
#pragma unroll
  for (int k = 0; k < IT; ++k) {  // exclusive offsets back into the blocked slots
    s_v[tid * PAD + k] = run;
    run += v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < IT; ++k) {  // striped (coalesced) stores
    const uint32_t j = (uint32_t)(k * 256 + tid);
    const uint32_t idx = base + j;
    if (idx < (uint32_t)n) offsets[idx] = s_v[(j / IT) * PAD + j % IT];
  }
}

// ----------------------------------------------------------- A3 duplicate
// Thread per Gaussian in depth order; emits (tile, id) for every active tile of
// its rect in row-major order starting at offsets[k].
constexpr int kDupSmall = 16;  // rect tiles a lane emits on its own
constexpr int kDupStage = 512;  // entries of a warp's output range staged in shared memory

// Warp-cooperative for large splats: a warp takes 32 consecutive Gaussians (depth order) and emits them one
// after the other, its 32 lanes walking the Gaussian's rect in row-major chunks of 32 tiles and
// compacting the active ones with a ballot, so every entry run is written coalesced and a
// large splat is spread over 32 lanes instead of one thread.
// cap bounds the writes (sync-free path: M is not known on the host; if M > cap the
// output is incomplete and the caller retries).  Thread 0 also publishes the entry count the later
// stages use: M if it fits, else 0 (an overflowed view gets EMPTY lists, never a partially written
// prefix with stale entries), and the overflow flag.
__global__ void __launch_bounds__(256) duplicate_kernel(int n, const uint32_t* __restrict__ ids,
                                                         const uint32_t* __restrict__ offsets,
                                                         const uint32_t* __restrict__ touched,
                                                         const short4* __restrict__ rect,
                                                         const uint32_t* __restrict__ bitmap, Dims d,
                                                         uint32_t* __restrict__ tkeys, uint32_t* __restrict__ tvals,
                                                         uint32_t cap, const unsigned long long* __restrict__ M64,
                                                         uint32_t* __restrict__ m_clamped,
                                                         uint32_t* __restrict__ overflow,
                                                         uint32_t* __restrict__ n_out) {
  __shared__ uint32_t s_dk[8][kDupStage], s_dv[8][kDupStage];  // per-warp output staging
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  if (k == 0) {
    const unsigned long long M = *M64;
    *m_clamped = M <= (unsigned long long)cap ? (uint32_t)M : 0u;
    *overflow = M > (unsigned long long)cap ? 1u : 0u;
    *n_out = (uint32_t)n;
  }
  uint32_t id = 0, cnt = 0, o = 0;
  short4 r = make_short4(0, 0, -1, -1);
  if (k < n) {
    id = ids[k];
    cnt = touched[id];
    if (cnt) {
      o = offsets[k];
      if (o + cnt > cap) cnt = 0;  // would overflow: skip (the caller sees M > cap)
      else r = rect[id];
    }
  }
  // small rects (<= kDupSmall tiles): the lane emits its own entries.  The warp's 32 Gaussians are
  // consecutive in depth order, so their entries form ONE contiguous output range: if it fits the
  // warp's shared buffer the lanes stage their entries there and the warp writes the range out
  // coalesced (positions of the cooperative large splats stay untouched), else they write directly.
  const int area0 = (r.z - r.x + 1) * (r.w - r.y + 1);
  const bool big = cnt != 0 && area0 > kDupSmall;
  const int w = threadIdx.x >> 5;
  const uint32_t lo = __reduce_min_sync(0xffffffffu, cnt ? o : 0xFFFFFFFFu);
  const uint32_t hi = __reduce_max_sync(0xffffffffu, cnt ? o + cnt : 0u);
  const bool staged = hi > lo && hi - lo <= (uint32_t)kDupStage;  // warp-uniform
  if (staged) {
    for (uint32_t j = lane; j < hi - lo; j += 32) s_dk[w][j] = 0xFFFFFFFFu;
    __syncwarp();
  }
  if (cnt != 0 && !big) {
    // row by row, the rect's active tiles are the set bits of the row's bitmap words masked to
    // [x0, x1]: one load per word, one iteration per emitted entry (ascending tx, as the oracle)
    uint32_t oo = o;
    for (int ty = r.y; ty <= r.w; ++ty) {
      const uint32_t* row = bitmap + ty * d.WPR;
      for (int wx = r.x >> 5; wx <= (r.z >> 5); ++wx) {
        const int b0 = max(r.x - 32 * wx, 0), b1 = min(r.z - 32 * wx, 31);
        uint32_t bits = __ldg(row + wx) & (0xFFFFFFFFu << b0) & (0xFFFFFFFFu >> (31 - b1));
        while (bits) {
          const int tx = 32 * wx + __ffs(bits) - 1;
          bits &= bits - 1u;
          PGSAG_DCHECK(oo < o + cnt && oo < cap);
          if (staged) {
            s_dk[w][oo - lo] = (uint32_t)(ty * d.TX + tx);
            s_dv[w][oo - lo] = id;
          } else {
            tkeys[oo] = (uint32_t)(ty * d.TX + tx);
            tvals[oo] = id;
          }
          ++oo;
        }
      }
    }
  }
  if (staged) {
    __syncwarp();
    for (uint32_t j = lane; j < hi - lo; j += 32) {
      const uint32_t key = s_dk[w][j];
      if (key != 0xFFFFFFFFu) {
        tkeys[lo + j] = key;
        tvals[lo + j] = s_dv[w][j];
      }
    }
  }
  // large rects: the whole warp, one Gaussian at a time
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t todo = __ballot_sync(0xffffffffu, big);
  while (todo) {
    const int j = __ffs(todo) - 1;
    todo &= todo - 1;
    const uint32_t gid = __shfl_sync(0xffffffffu, id, j);
    const uint32_t go = __shfl_sync(0xffffffffu, o, j);
    const int x0 = __shfl_sync(0xffffffffu, (int)r.x, j), y0 = __shfl_sync(0xffffffffu, (int)r.y, j);
    const int x1 = __shfl_sync(0xffffffffu, (int)r.z, j), y1 = __shfl_sync(0xffffffffu, (int)r.w, j);
    const int w = x1 - x0 + 1, area = w * (y1 - y0 + 1);
    uint32_t written = 0;
    for (int t0 = 0; t0 < area; t0 += 32) {
      const int t = t0 + lane;
      bool act = false;
      uint32_t tile = 0;
      if (t < area) {
        const int ty = y0 + t / w, tx = x0 + (t - (t / w) * w);
        act = (__ldg(bitmap + ty * d.WPR + (tx >> 5)) >> (tx & 31)) & 1u;
        tile = (uint32_t)(ty * d.TX + tx);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, act);
      if (act) {
        const uint32_t pos = go + written + __popc(bal & lt);
        PGSAG_DCHECK(pos < cap);
        tkeys[pos] = tile;
        tvals[pos] = gid;
      }
      written += __popc(bal);
    }
  }
}

// -------------------------------------------------------------- A5 ranges
__global__ void ranges_kernel(const uint32_t* __restrict__ tkeys, const uint32_t* __restrict__ M_ptr,
                              uint32_t ntiles, uint32_t* __restrict__ ranges) {
  const uint32_t M = *M_ptr;  // the entry count published by A3 (0 after an overflow)
  // four consecutive keys per thread (one 128-bit load) and their two outer neighbours; keys past
  // M read as the all-ones sentinel (never a tile id), so the ends of the array close their ranges
  const uint32_t ng = (M + 3u) / 4u;
  const bool vec = (reinterpret_cast<uintptr_t>(tkeys) & 15u) == 0u;  // caller buffer: 16-byte aligned?
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ng; gi += gridDim.x * blockDim.x) {
    const uint32_t k0 = gi * 4u;
    uint32_t t[6];
    if (vec && k0 + 4u <= M) {
      const uint4 v = reinterpret_cast<const uint4*>(tkeys)[gi];
      t[1] = v.x; t[2] = v.y; t[3] = v.z; t[4] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) t[1 + j] = k0 + j < M ? tkeys[k0 + j] : 0xFFFFFFFFu;
    }
    t[0] = k0 > 0u ? tkeys[k0 - 1u] : 0xFFFFFFFFu;
    t[5] = k0 + 4u < M ? tkeys[k0 + 4u] : 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t c = t[1 + j], k = k0 + (uint32_t)j;
      if (k >= M || c >= ntiles) continue;  // (keys are tile ids < ntiles by construction)
      if (t[j] != c) ranges[2 * c] = k;
      if (t[j + 2] != c) ranges[2 * c + 1] = k + 1u;
    }
  }
}

// ------------------------------------------------------ A5b work order (LPT)
// The active tiles bucketed by floor(log2(list length)), emitted longest class first, so the
// persistent A6/A7 grids start the heaviest tiles first (longest-processing-time order; the order
// inside a class is arbitrary).  Two grid-wide kernels: (1) every active tile takes a slot in its
// class (warp-aggregated atomics on the 33 class counters), (2) every tile is written at its
// class's offset (classes longest first) + its slot.
__device__ __forceinline__ uint32_t lpt_class(const uint2* __restrict__ ranges, uint32_t tile) {
  const uint2 r = __ldg(ranges + tile);
  return 32u - (uint32_t)__clz(r.y - r.x);  // 0 for an empty list, 1..32 otherwise
}

__global__ void __launch_bounds__(256) lpt_class_kernel(const uint32_t* __restrict__ active,
                                                        const uint32_t* __restrict__ n_active,
                                                        const uint2* __restrict__ ranges,
                                                        uint32_t* __restrict__ cls_cnt, uint32_t* __restrict__ packed) {
  const uint32_t na = *n_active;
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = k < na;
  const uint32_t c = live ? lpt_class(ranges, __ldg(active + k)) : 63u;
  const uint32_t peers = __match_any_sync(0xffffffffu, c);
  const int leader = __ffs(peers) - 1, lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == leader && live) base = atomicAdd(cls_cnt + c, (uint32_t)__popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (live) packed[k] = (c << 26) | (base + (uint32_t)__popc(peers & ((1u << lane) - 1u)));
}

__global__ void __launch_bounds__(256) lpt_scatter_kernel(const uint32_t* __restrict__ active,
                                                          const uint32_t* __restrict__ n_active,
                                                          const uint32_t* __restrict__ cls_cnt,
                                                          const uint32_t* __restrict__ packed,
                                                          uint32_t* __restrict__ order) {
  __shared__ uint32_t s_pos[33];
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (int c = 32; c >= 0; --c) { s_pos[c] = run; run += cls_cnt[c]; }
  }
  __syncthreads();
  const uint32_t na = *n_active;
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= na) return;
  const uint32_t p = packed[k];
  order[s_pos[p >> 26] + (p & 0x3FFFFFFu)] = __ldg(active + k);
}

int num_sms() {
  static int sms[kMaxDevices] = {};
  const int dev = current_device();
  if (!sms[dev]) {
    int s = 0;
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = s > 0 ? s : 148;
  }
  return sms[dev];
}

// LSD radix sort of (keys, vals) on bits [0, end_bit).  Ping-pongs between (a)
// and (b); returns in *res_a whether the result ended in a.  n is a device
// pointer (n_dev) or a fixed count with a capacity bound for the grid size.
cudaError_t radix_sort(uint32_t* ka, uint32_t* va, uint32_t* kb, uint32_t* vb, const uint32_t* n_dev,
                       uint32_t n_fixed, uint32_t grid_bound, int end_bit, uint32_t* status, size_t status_stride,
                       uint32_t* ghist, uint32_t* counters, cudaStream_t st, bool* res_in_a,
                       const float* depth = nullptr, const uint32_t* touched = nullptr) {
  const PassPlan plan = make_plan(end_bit);
  const int npass = plan.n;
  *res_in_a = true;
  if (npass == 0 || grid_bound == 0) return cudaSuccess;
  static bool attr_set[kMaxDevices] = {};
  const int dev = current_device();
  if (!attr_set[dev]) {
    cudaFuncSetAttribute(radix_pass_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem<8>());
    cudaFuncSetAttribute(radix_pass_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem<9>());
    attr_set[dev] = true;
  }
  const int hist_grid = min((int)((grid_bound + 255) / 256), num_sms() * 4);
  {
    KTimer kt_(depth ? "A4_radix_hist_s1" : "A4_radix_hist_s2", st);
    if (depth)  // stage 1: the keys (and identity ids) are formed by the histogram pass itself
      radix_hist_kernel<true><<<hist_grid, 256, 0, st>>>(nullptr, n_dev, n_fixed, plan, ghist, depth, touched, ka, va);
    else
      radix_hist_runs_kernel<<<hist_grid, 256, 0, st>>>(ka, n_dev, n_fixed, plan, ghist);
  }
  const uint32_t tiles = (grid_bound + kSortTile - 1) / kSortTile;
  uint32_t *ki = ka, *vi = va, *ko = kb, *vo = vb;
  for (int p = 0; p < npass; ++p) {
    {
      KTimer kt_(depth ? "A4_radix_onesweep_s1" : "A4_radix_onesweep_s2", st);
      if (plan.width[p] <= 8)
        radix_pass_kernel<8><<<tiles, kSortThreads, pass_smem<8>(), st>>>(
            ki, vi, ko, vo, n_dev, n_fixed, plan.shift[p], plan.width[p], ghist + p * kMaxRadix,
            status + p * status_stride, counters + p);
      else
        radix_pass_kernel<9><<<tiles, kSortThreads, pass_smem<9>(), st>>>(
            ki, vi, ko, vo, n_dev, n_fixed, plan.shift[p], plan.width[p], ghist + p * kMaxRadix,
            status + p * status_stride, counters + p);
    }
    uint32_t* t;
    t = ki; ki = ko; ko = t;
    t = vi; vi = vo; vo = t;
  }
  *res_in_a = (npass % 2) == 0;
  return cudaGetLastError();
}

}  // namespace

WsLayout ws_layout(int32_t n, int32_t W, int32_t H, int64_t cap) {
  WsLayout L;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const size_t nn = (size_t)(n > 0 ? n : 0), cc = (size_t)(cap > 0 ? cap : 0);
  L.tiles1 = (int)((nn + kSortTile - 1) / kSortTile);
  L.tiles2 = (int)((cc + kSortTile - 1) / kSortTile);
  L.tilesN = (int)((nn + kScanTile - 1) / kScanTile);
  // counters first: their offset does not depend on n or the capacity, so a render call sees the
  // flags the sort of the same view published in the same workspace
  L.counters = take(4 * kCounters);
  L.a0 = take(4 * (size_t)(((H > 0 ? H : 0) + kTile - 1) / kTile) *
              (size_t)((((W > 0 ? W : 0) + kTile - 1) / kTile + 31) / 32));
  // the state a sort call zeroes, contiguous after the counters (one memset)
  L.hist = take(4 * 2 * kMaxSortPasses * kMaxRadix);
  L.scan_status = take(8 * (size_t)(L.tilesN > 0 ? L.tilesN : 1));
  L.status1 = take(4 * (size_t)kMaxSortPasses * L.tiles1 * kMaxRadix);
  L.zero_end = off;
  for (int k = 0; k < 2; ++k) { L.depth_keys[k] = take(4 * nn); L.ids[k] = take(4 * nn); }
  L.offsets = take(4 * nn);
  L.dup_keys = take(4 * cc);
  L.dup_vals = take(4 * cc);
  L.status2 = take(4 * (size_t)kMaxSortPasses * L.tiles2 * kMaxRadix);
  L.g2d = take(4 * 16 * nn);  // [n][16] f32 (14 used), one 64-byte line per Gaussian
  const size_t ntiles = (size_t)((W > 0 ? W : 0) + kTile - 1) / kTile * (size_t)(((H > 0 ? H : 0) + kTile - 1) / kTile);
  L.lpt = take(4 * ntiles);
  L.total = off;
  return L;
}

// Stage 1 (depth sort of Gaussians) + A2 scan.  The region [counters, zero_end) (counters,
// histograms, A2 and stage-1 look-back state) must have been cleared by the caller.
cudaError_t launch_bin_sort_stage1(const pgsag_projected* p, int n, const WsLayout& L, char* ws,
                                   cudaStream_t st, const uint32_t** ids_sorted) {
  uint32_t* k0 = reinterpret_cast<uint32_t*>(ws + L.depth_keys[0]);
  uint32_t* k1 = reinterpret_cast<uint32_t*>(ws + L.depth_keys[1]);
  uint32_t* i0 = reinterpret_cast<uint32_t*>(ws + L.ids[0]);
  uint32_t* i1 = reinterpret_cast<uint32_t*>(ws + L.ids[1]);
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + L.counters);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist);
  bool in_a = true;
  cudaError_t e = radix_sort(k0, i0, k1, i1, nullptr, (uint32_t)n, (uint32_t)n, 32,
                             reinterpret_cast<uint32_t*>(ws + L.status1), (size_t)L.tiles1 * kMaxRadix, hist,
                             counters + CNT_SORT1, st, &in_a, p->depth, p->tiles_touched);
  if (e != cudaSuccess) return e;
  const uint32_t* ids = in_a ? i0 : i1;
  *ids_sorted = ids;
  {
    KTimer kt_("A2_scan", st);
    scan_kernel<<<L.tilesN, 256, 0, st>>>(n, p->tiles_touched, ids, reinterpret_cast<uint32_t*>(ws + L.offsets),
                                          reinterpret_cast<unsigned long long*>(ws + L.scan_status),
                                          counters + CNT_SCAN, reinterpret_cast<unsigned long long*>(counters + CNT_M));
  }
  return cudaGetLastError();
}

// M_known: the host read M (sync path; grids sized by M).  Otherwise M is only on the device
// and every grid is bounded by the capacity (sync-free path).
cudaError_t launch_duplicate_and_sort(const pgsag_projected* p, const pgsag_tilemask* tm, const Dims& d, int n,
                                      uint32_t M, bool M_known, const uint32_t* ids_sorted, const WsLayout& L,
                                      char* ws, pgsag_bins* bins, cudaStream_t st) {
  uint32_t* counters = reinterpret_cast<uint32_t*>(ws + L.counters);
  uint32_t* hist = reinterpret_cast<uint32_t*>(ws + L.hist) + kMaxSortPasses * kMaxRadix;
  const int ntiles = d.TX * d.TY;
  int tile_bits = 0;
  while ((1 << tile_bits) < ntiles) ++tile_bits;
  const int npass = make_plan(tile_bits).n;
  // emit into the buffer that makes the last pass land in bins
  uint32_t *ek, *ev, *ok, *ov;
  if (npass % 2 == 0) {
    ek = bins->tile_keys; ev = bins->vals;
    ok = reinterpret_cast<uint32_t*>(ws + L.dup_keys); ov = reinterpret_cast<uint32_t*>(ws + L.dup_vals);
  } else {
    ek = reinterpret_cast<uint32_t*>(ws + L.dup_keys); ev = reinterpret_cast<uint32_t*>(ws + L.dup_vals);
    ok = bins->tile_keys; ov = bins->vals;
  }
  cudaMemsetAsync(bins->ranges, 0, sizeof(uint32_t) * 2 * (size_t)ntiles, st);
  auto order = [&]() {
    if (!bins->order || ntiles == 0) return;
    const int g = (ntiles + 255) / 256;
    uint32_t* packed = reinterpret_cast<uint32_t*>(ws + L.lpt);
    {
      KTimer kt_("A5_lpt_class", st);
      lpt_class_kernel<<<g, 256, 0, st>>>(tm->active, tm->n_active, reinterpret_cast<const uint2*>(bins->ranges),
                                          counters + CNT_LPT, packed);
    }
    KTimer kt_("A5_lpt_scatter", st);
    lpt_scatter_kernel<<<g, 256, 0, st>>>(tm->active, tm->n_active, counters + CNT_LPT, packed, bins->order);
  };
  const uint32_t bound = M_known ? M : (uint32_t)bins->capacity;  // grid bound
  if (bound == 0 || n == 0) {
    order();
    return cudaGetLastError();
  }
  uint32_t* m_clamped = counters + CNT_MC;
  {
    KTimer kt_("A3_duplicate", st);
    duplicate_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, ids_sorted, reinterpret_cast<uint32_t*>(ws + L.offsets),
                                                      p->tiles_touched, reinterpret_cast<const short4*>(p->rect),
                                                      tm->active_bits, d, ek, ev, (uint32_t)bins->capacity,
                                                      reinterpret_cast<const unsigned long long*>(counters + CNT_M),
                                                      m_clamped, counters + CNT_OVF, counters + CNT_NG);
  }
  bool in_a = true;
  // look-back state for exactly the tiles the bound needs
  const size_t stride = (size_t)((bound + kSortTile - 1) / kSortTile) * kMaxRadix;
  cudaMemsetAsync(ws + L.status2, 0, 4 * stride * (size_t)npass, st);
  cudaError_t e = radix_sort(ek, ev, ok, ov, m_clamped, bound, bound, tile_bits,
                             reinterpret_cast<uint32_t*>(ws + L.status2), stride, hist,
                             counters + CNT_SORT2, st, &in_a);
  if (e != cudaSuccess) return e;
  const int grid = min((int)(((bound + 3) / 4 + 255) / 256), num_sms() * 8);
  {
    KTimer kt_("A5_ranges", st);
    ranges_kernel<<<grid, 256, 0, st>>>(bins->tile_keys, m_clamped, (uint32_t)ntiles, bins->ranges);
  }
  order();
  return cudaGetLastError();
}

}  // namespace pgsag
