// A0 (building-mask tile occupancy) and A1 (per-Gaussian projection) for sm_100a.
//
// This translation unit is compiled with --fmad=false: A1's key path (camera z,
// the 2D covariance and the tile rect) is IEEE float32 with every product and sum
// rounded separately, in the order DESIGN.md §4 fixes, so the (tile, depth) keys
// are bit-exact with any other correct float32 evaluation of the same readings.
//
// P:78 "each 3D Gaussian sphere is transformed into a 2D Gaussian based on the
// viewing direction of each camera and then projected onto different image
// tiles"; Eq. 2-3 (n_i, R_c n_i, d_i); P:243 masked pixels only.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "internal.cuh"

namespace pgsag {
namespace {

// ------------------------------------------------------------------ A0 count
// One thread per tile; a warp covers 32 horizontally adjacent tiles, so each of
// its 16 row loads is 512 contiguous bytes (uint4 per lane) -> fully coalesced.
// The warp's ballot over "tile has a mask pixel" is exactly one bitmap word.
__global__ void __launch_bounds__(128) tilemask_count_kernel(const uint8_t* __restrict__ mask, Dims d,
                                                               uint32_t* __restrict__ tile_cnt,
                                                               uint32_t* __restrict__ bitmap, int vec16) {
  const int tx = blockIdx.x * blockDim.x + threadIdx.x;
  const int ty = blockIdx.y;
  uint32_t cnt = 0;
  if (tx < d.TX) {
    const int i0 = tx * kTile;
    const int i1 = min(i0 + kTile, d.W);
    const int j0 = ty * kTile;
    const int j1 = min(j0 + kTile, d.H);
    // bytes != 0 -> 0xFF per byte; popc / 8 = number of nonzero bytes
    const auto row16 = [&](int j) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(mask + (size_t)j * d.W + i0));
      return (uint32_t)(__popc(__vcmpne4(w.x, 0u)) + __popc(__vcmpne4(w.y, 0u)) + __popc(__vcmpne4(w.z, 0u)) +
                        __popc(__vcmpne4(w.w, 0u))) >> 3;
    };
    if (vec16 && i1 - i0 == kTile && j1 - j0 == kTile) {
      uint32_t c[kTile];  // the tile's 16 row loads all in flight
#pragma unroll
      for (int r = 0; r < kTile; ++r) c[r] = row16(j0 + r);
#pragma unroll
      for (int r = 0; r < kTile; ++r) cnt += c[r];
    } else if (vec16 && i1 - i0 == kTile) {
      for (int j = j0; j < j1; ++j) cnt += row16(j);
    } else {
      for (int j = j0; j < j1; ++j)
        for (int i = i0; i < i1; ++i) cnt += mask[(size_t)j * d.W + i] != 0;
    }
    tile_cnt[ty * d.TX + tx] = cnt;
  }
  const unsigned word = __ballot_sync(0xffffffffu, tx < d.TX && cnt > 0);
  const int lane = threadIdx.x & 31;
  const int wtx = tx - lane;  // first tile of this warp (multiple of 32 since blockDim % 32 == 0)
  if (lane == 0 && wtx < d.TX) bitmap[ty * d.WPR + wtx / 32] = word;
}

// ------------------------------------------------------------- A0 active list
// (1) one CTA: exclusive prefix of the active-tile counts of the bitmap words (TY x WPR words,
// row-major = tile order), 1024 threads with a few words each; (2) one warp per bitmap word, one
// lane per bit: every active tile is written at its word's prefix + the set bits below it, so the
// list is in ascending tile order.
__global__ void __launch_bounds__(1024) tilemask_prefix_kernel(Dims d, const uint32_t* __restrict__ bitmap,
                                                                 uint32_t* __restrict__ wpre,
                                                                 uint32_t* __restrict__ n_active) {
  constexpr int NT = 1024;
  __shared__ uint32_t s_warp[NT / 32];
  const int nw = d.TY * d.WPR, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int per = (nw + NT - 1) / NT;  // consecutive words per thread
  const int k0 = tid * per;
  uint32_t sum = 0;
  for (int j = 0; j < per; ++j)
    if (k0 + j < nw) sum += __popc(bitmap[k0 + j]);
  uint32_t x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  uint32_t wb = 0, tot = 0;
  for (int k = 0; k < NT / 32; ++k) {
    const uint32_t t = s_warp[k];
    if (k < w) wb += t;
    tot += t;
  }
  uint32_t run = wb + x - sum;
  for (int j = 0; j < per; ++j)
    if (k0 + j < nw) {
      wpre[k0 + j] = run;
      run += __popc(bitmap[k0 + j]);
    }
  if (tid == 0) *n_active = tot;
}

__global__ void __launch_bounds__(256) tilemask_list_kernel(Dims d, const uint32_t* __restrict__ bitmap,
                                                              const uint32_t* __restrict__ wpre,
                                                              uint32_t* __restrict__ active) {
  const int k = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (k >= d.TY * d.WPR) return;
  const uint32_t bits = bitmap[k];
  if (!((bits >> lane) & 1u)) return;
  const int y = k / d.WPR, x = (k - y * d.WPR) * 32 + lane;
  active[wpre[k] + __popc(bits & ((1u << lane) - 1u))] = (uint32_t)(y * d.TX + x);
}

// SAT of the active flags, SAT[y][x] = #active tiles with ty < y, tx < x: one warp per
// 32 columns; per-row word prefixes in shared memory, one running sum per lane.
__global__ void __launch_bounds__(32) tilemask_satcol_kernel(Dims d, const uint32_t* __restrict__ bitmap,
                                                              int32_t* __restrict__ sat) {
  extern __shared__ uint32_t pre[];  // [TY]: set bits in words < b of each row
  const int lane = threadIdx.x;
  const int b = blockIdx.x;  // word / 32-column block
  const int x = b * 32 + lane;
  const int S = d.TX + 1;
  for (int y = lane; y < d.TY; y += 32) {
    uint32_t c = 0;
    for (int w = 0; w < b && w < d.WPR; ++w) c += __popc(__ldg(bitmap + y * d.WPR + w));
    pre[y] = c;
  }
  __syncwarp();
  if (x > d.TX) return;
  sat[x] = 0;
  const uint32_t lowmask = lane ? ((1u << lane) - 1u) : 0u;
  uint32_t acc = 0;
#pragma unroll 4
  for (int y = 0; y < d.TY; ++y) {
    const uint32_t word = b < d.WPR ? __ldg(bitmap + y * d.WPR + b) : 0u;
    acc += pre[y] + __popc(word & lowmask);
    sat[(size_t)(y + 1) * S + x] = (int32_t)acc;
  }
}

// --------------------------------------------------------------- A1 project
struct CamK {
  float fx, fy, cx, cy;
  float R[9];
  float C[3];
  float znear;
  float lx, ly;  // 1.3 x half-FoV tangent (R9)
};

// real SH constants, degree <= 3 (R12)
__constant__ float kShC2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f,
                               -1.0925484305920792f, 0.5462742152960396f};
__constant__ float kShC3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f,
                               0.3731763325901154f, -0.4570457994644658f, 1.445305721320277f,
                               -0.5900435899266435f};

__device__ __forceinline__ int fdiv16(int a) { return a >> 4; }  // floor division (arithmetic shift)

// ln upper bound from y = m 2^ex, m in [0.5,1):  e ln2 + f(6+f)/(6+4f) + 2^-18 (R8)
__device__ __forceinline__ float lnup(float y) {
  const uint32_t b = __float_as_uint(y);
  const int ex = (int)((b >> 23) & 0xFFu) - 126;
  const float m = __uint_as_float((b & 0x807FFFFFu) | 0x3F000000u);
  const float e = (float)(ex - 1);
  const float f = 2.0f * m - 1.0f;
  return (e * 0.6931471805599453f + (f * (6.0f + f)) / (6.0f + 4.0f * f)) + 3.814697265625e-06f;
}

template <int DEG>
__global__ void __launch_bounds__(256) preprocess_kernel(
    int n, const float* __restrict__ mean, const float* __restrict__ scale,
    const float* __restrict__ rot, const float* __restrict__ opac, const float* __restrict__ sh, CamK cam,
    Dims d, const uint32_t* __restrict__ bits, float2* __restrict__ mean2d, float4* __restrict__ conic_o,
    float* __restrict__ depth, short4* __restrict__ rect, uint32_t* __restrict__ tiles_touched,
    float4* __restrict__ rgb_d, float4* __restrict__ ncam, uint32_t* __restrict__ flags) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float t0 = __ldg(mean + i) - cam.C[0];
  const float t1 = __ldg(mean + n + i) - cam.C[1];
  const float t2 = __ldg(mean + 2 * n + i) - cam.C[2];
  // the other per-Gaussian loads issued before the visibility branch (one memory latency)
  const float qw0 = __ldg(rot + i), qx0 = __ldg(rot + n + i), qy0 = __ldg(rot + 2 * n + i),
              qz0 = __ldg(rot + 3 * n + i);
  const float s[3] = {__ldg(scale + i), __ldg(scale + n + i), __ldg(scale + 2 * n + i)};
  const float opv = __ldg(opac + i);
  const float* Rc = cam.R;
  const float x = (Rc[0] * t0 + Rc[1] * t1) + Rc[2] * t2;
  const float y = (Rc[3] * t0 + Rc[4] * t1) + Rc[5] * t2;
  const float z = (Rc[6] * t0 + Rc[7] * t1) + Rc[8] * t2;

  uint32_t fl = 0;
  float2 uv = make_float2(0.f, 0.f);
  float4 co = make_float4(0.f, 0.f, 0.f, 0.f);
  short4 rc = make_short4(0, 0, -1, -1);
  uint32_t touched = 0;
  float4 cd = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 nc = make_float4(0.f, 0.f, 0.f, 0.f);
  float zout = 0.f;

  if (z > cam.znear) {
    fl |= PGSAG_F_VISIBLE;
    zout = z;
    const float xz = x / z, yz = y / z;
    uv.x = cam.fx * xz + cam.cx;
    uv.y = cam.fy * yz + cam.cy;

    // quaternion -> rotation (w,x,y,z), normalised
    const float qn = sqrtf(((qw0 * qw0 + qx0 * qx0) + qy0 * qy0) + qz0 * qz0);
    const float qw = qw0 / qn, qx = qx0 / qn, qy = qy0 / qn, qz = qz0 / qn;
    float Rg[3][3];
    Rg[0][0] = 1.0f - 2.0f * (qy * qy + qz * qz);
    Rg[0][1] = 2.0f * (qx * qy - qw * qz);
    Rg[0][2] = 2.0f * (qx * qz + qw * qy);
    Rg[1][0] = 2.0f * (qx * qy + qw * qz);
    Rg[1][1] = 1.0f - 2.0f * (qx * qx + qz * qz);
    Rg[1][2] = 2.0f * (qy * qz - qw * qx);
    Rg[2][0] = 2.0f * (qx * qz - qw * qy);
    Rg[2][1] = 2.0f * (qy * qz + qw * qx);
    Rg[2][2] = 1.0f - 2.0f * (qx * qx + qy * qy);
    float Mg[3][3], Sig[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) Mg[a][b] = Rg[a][b] * s[b];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) Sig[a][b] = (Mg[a][0] * Mg[b][0] + Mg[a][1] * Mg[b][1]) + Mg[a][2] * Mg[b][2];

    float cxz = xz, cyz = yz;
    if (xz < -cam.lx) { cxz = -cam.lx; fl |= PGSAG_F_CLAMP_X; }
    if (xz > cam.lx) { cxz = cam.lx; fl |= PGSAG_F_CLAMP_X; }
    if (yz < -cam.ly) { cyz = -cam.ly; fl |= PGSAG_F_CLAMP_Y; }
    if (yz > cam.ly) { cyz = cam.ly; fl |= PGSAG_F_CLAMP_Y; }
    const float J00 = cam.fx / z, J02 = -((cam.fx * cxz) / z);
    const float J11 = cam.fy / z, J12 = -((cam.fy * cyz) / z);
    // Tm = J R_c (J01 = J10 = 0: the omitted products are exact zeros)
    float Tm[2][3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      Tm[0][b] = J00 * Rc[b] + J02 * Rc[6 + b];
      Tm[1][b] = J11 * Rc[3 + b] + J12 * Rc[6 + b];
    }
    float Mt[2][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) Mt[a][b] = (Tm[a][0] * Sig[0][b] + Tm[a][1] * Sig[1][b]) + Tm[a][2] * Sig[2][b];
    const float c00 = (Mt[0][0] * Tm[0][0] + Mt[0][1] * Tm[0][1]) + Mt[0][2] * Tm[0][2];
    const float c01 = (Mt[0][0] * Tm[1][0] + Mt[0][1] * Tm[1][1]) + Mt[0][2] * Tm[1][2];
    const float c11 = (Mt[1][0] * Tm[1][0] + Mt[1][1] * Tm[1][1]) + Mt[1][2] * Tm[1][2];
    const float A = c00 + 0.3f, B = c01, Cc = c11 + 0.3f;  // low-pass (R10)
    const float det = A * Cc - B * B;
    if (det > 0.0f) {
      fl |= PGSAG_F_DET_OK;
      const float o = opv;
      co = make_float4(Cc / det, -B / det, A / det, o);
      if (!(o < 1.0f / 255.0f)) {
        fl |= PGSAG_F_OPAC_OK;
        // opacity-aware conservative ellipse AABB (R8)
        float k2 = (2.0f * lnup(255.0f * o)) * (1.0f + 0.0009765625f);
        if (k2 < 0.0f) k2 = 0.0f;
        const float rx = sqrtf(k2 * A) + 0.015625f, ry = sqrtf(k2 * Cc) + 0.015625f;
        const float lim = 1048576.0f;
        const int ix0 = (int)fminf(fmaxf(ceilf((uv.x - rx) - 0.5f), -lim), lim);
        const int ix1 = (int)fminf(fmaxf(floorf((uv.x + rx) - 0.5f), -lim), lim);
        const int iy0 = (int)fminf(fmaxf(ceilf((uv.y - ry) - 0.5f), -lim), lim);
        const int iy1 = (int)fminf(fmaxf(floorf((uv.y + ry) - 0.5f), -lim), lim);
        const int tx0 = max(0, fdiv16(ix0)), tx1 = min(d.TX - 1, fdiv16(ix1));
        const int ty0 = max(0, fdiv16(iy0)), ty1 = min(d.TY - 1, fdiv16(iy1));
        if (tx0 <= tx1 && ty0 <= ty1) {
          fl |= PGSAG_F_RECT;
          rc = make_short4((short)tx0, (short)ty0, (short)tx1, (short)ty1);
          // active tiles in the rect, straight from the A0 bitmap (rows of 32-tile words)
          const int w0 = tx0 >> 5, w1 = tx1 >> 5;
          const uint32_t m0 = ~0u << (tx0 & 31), m1 = ~0u >> (31 - (tx1 & 31));
          for (int y = ty0; y <= ty1; ++y) {
            const uint32_t* row = bits + y * d.WPR;
            if (w0 == w1) {
              touched += __popc(__ldg(row + w0) & m0 & m1);
            } else {
              touched += __popc(__ldg(row + w0) & m0) + __popc(__ldg(row + w1) & m1);
              for (int w = w0 + 1; w < w1; ++w) touched += __popc(__ldg(row + w));
            }
          }
        }
        // flattened-Gaussian normal (R4) and plane distance (Eq. 3, R2)
        int k = 0;
        float smin = s[0];
        if (s[1] < smin) { k = 1; smin = s[1]; }
        if (s[2] < smin) k = 2;
        fl |= (uint32_t)k << PGSAG_F_AXIS_SHIFT;
        // (selects, not a dynamic index: keeps Rg in registers)
        float n0 = k == 0 ? Rg[0][0] : (k == 1 ? Rg[0][1] : Rg[0][2]);
        float n1 = k == 0 ? Rg[1][0] : (k == 1 ? Rg[1][1] : Rg[1][2]);
        float n2 = k == 0 ? Rg[2][0] : (k == 1 ? Rg[2][1] : Rg[2][2]);
        const float dotv = (n0 * t0 + n1 * t1) + n2 * t2;
        if (dotv > 0.0f) { n0 = -n0; n1 = -n1; n2 = -n2; fl |= PGSAG_F_NFLIP; }
        nc.x = (Rc[0] * n0 + Rc[1] * n1) + Rc[2] * n2;
        nc.y = (Rc[3] * n0 + Rc[4] * n1) + Rc[5] * n2;
        nc.z = (Rc[6] * n0 + Rc[7] * n1) + Rc[8] * n2;
        cd.w = (n0 * t0 + n1 * t1) + n2 * t2;
        // SH colour (R12)
        const float len = sqrtf((t0 * t0 + t1 * t1) + t2 * t2);
        const float dx = t0 / len, dy = t1 / len, dz = t2 / len;
        float Y[16];
        const float xx = dx * dx, yy = dy * dy, zz = dz * dz, xy = dx * dy, yzp = dy * dz, xzp = dx * dz;
        Y[0] = 0.28209479177387814f;
        Y[1] = -0.4886025119029199f * dy;
        Y[2] = 0.4886025119029199f * dz;
        Y[3] = -0.4886025119029199f * dx;
        Y[4] = kShC2[0] * xy;
        Y[5] = kShC2[1] * yzp;
        Y[6] = kShC2[2] * ((2.0f * zz - xx) - yy);
        Y[7] = kShC2[3] * xzp;
        Y[8] = kShC2[4] * (xx - yy);
        Y[9] = (kShC3[0] * dy) * (3.0f * xx - yy);
        Y[10] = (kShC3[1] * xy) * dz;
        Y[11] = (kShC3[2] * dy) * ((4.0f * zz - xx) - yy);
        Y[12] = (kShC3[3] * dz) * ((2.0f * zz - 3.0f * xx) - 3.0f * yy);
        Y[13] = (kShC3[4] * dx) * ((4.0f * zz - xx) - yy);
        Y[14] = (kShC3[5] * dz) * (xx - yy);
        Y[15] = (kShC3[6] * dx) * (xx - 3.0f * yy);
        constexpr int K = (DEG + 1) * (DEG + 1);
        // SH coefficients: all loads issued up front (compile-time degree), then the same
        // left-to-right sums as the oracle
        float shv[3 * K];
#pragma unroll
        for (int q = 0; q < 3 * K; ++q) shv[q] = __ldg(sh + (size_t)q * n + i);
        float col[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          float acc = Y[0] * shv[c];
#pragma unroll
          for (int l = 1; l < K; ++l) acc = acc + Y[l] * shv[l * 3 + c];
          acc = acc + 0.5f;
          if (acc < 0.0f) { acc = 0.0f; fl |= PGSAG_F_RGB_CLAMP0 << c; }
          col[c] = acc;
        }
        cd.x = col[0]; cd.y = col[1]; cd.z = col[2];
      }
    }
  }
  mean2d[i] = uv;
  conic_o[i] = co;
  depth[i] = zout;
  rect[i] = rc;
  tiles_touched[i] = touched;
  rgb_d[i] = cd;
  ncam[i] = nc;
  flags[i] = fl;
}

}  // namespace

cudaError_t launch_tilemask(const uint8_t* mask, const Dims& d, pgsag_tilemask* tm, uint32_t* scratch,
                            cudaStream_t st) {
  uint32_t* bitmap = tm->active_bits;
  const int vec16 = (d.W % 16 == 0) && ((reinterpret_cast<uintptr_t>(mask) & 15u) == 0);
  dim3 grid((d.TX + 127) / 128, d.TY);
  {
    KTimer kt_("A0_tilemask_count", st);
    tilemask_count_kernel<<<grid, 128, 0, st>>>(mask, d, tm->tile_cnt, bitmap, vec16);
  }
  uint32_t* wpre = scratch;  // [TY*WPR] word prefixes (workspace)
  {
    KTimer kt_("A0_tilemask_prefix", st);
    tilemask_prefix_kernel<<<1, 1024, 0, st>>>(d, bitmap, wpre, tm->n_active);
  }
  {
    KTimer kt_("A0_tilemask_list", st);
    const int words = d.TY * d.WPR;
    tilemask_list_kernel<<<(words * 32 + 255) / 256, 256, 0, st>>>(d, bitmap, wpre, tm->active);
  }
  if (tm->sat) {  // optional output (not needed by the path: A1 counts from the bitmap)
    KTimer kt_("A0_tilemask_sat", st);
    tilemask_satcol_kernel<<<(d.TX + 1 + 31) / 32, 32, sizeof(uint32_t) * d.TY, st>>>(d, bitmap, tm->sat);
  }
  return cudaGetLastError();
}

namespace {
// Debug check (pgsag_set_checks): count non-finite Gaussian parameters (S:289 precondition).
__global__ void finite_check_kernel(const float* __restrict__ a, size_t count, unsigned int* __restrict__ bad) {
  unsigned int b = 0;
  for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < count; k += (size_t)gridDim.x * blockDim.x)
    b += !isfinite(a[k]);
  b = __reduce_add_sync(0xffffffffu, b);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
}
}  // namespace

cudaError_t launch_finite_check(const pgsag_gaussians* g, unsigned int* bad, cudaStream_t st) {
  const size_t n = (size_t)g->n, K3 = (size_t)(g->sh_degree + 1) * (g->sh_degree + 1) * 3;
  const float* arr[5] = {g->mean, g->scale, g->rot, g->opacity, g->sh};
  const size_t cnt[5] = {3 * n, 3 * n, 4 * n, n, K3 * n};
  for (int k = 0; k < 5; ++k) {
    if (!cnt[k]) continue;
    finite_check_kernel<<<(unsigned)std::min<size_t>((cnt[k] + 255) / 256, 1184), 256, 0, st>>>(arr[k], cnt[k], bad);
  }
  return cudaGetLastError();
}

cudaError_t launch_preprocess(const pgsag_gaussians* g, const pgsag_camera* c, const Dims& d,
                              const pgsag_tilemask* tm, pgsag_projected* out, cudaStream_t st) {
  if (g->n == 0) return cudaSuccess;
  CamK k;
  k.fx = c->fx; k.fy = c->fy; k.cx = c->cx; k.cy = c->cy;
  for (int a = 0; a < 9; ++a) k.R[a] = c->R[a];
  for (int a = 0; a < 3; ++a) k.C[a] = c->C[a];
  k.znear = c->znear;
  // evaluated on the host with the same IEEE ops: 1.3 * ((0.5 * W) / fx)
  volatile float hw = 0.5f * (float)c->width, hh = 0.5f * (float)c->height;
  volatile float qx = hw / c->fx, qy = hh / c->fy;
  k.lx = 1.3f * qx;
  k.ly = 1.3f * qy;
  const int threads = 256;
  {
    KTimer kt_("A1_preprocess", st);
#define PGSAG_A1(DEG)                                                                                      \
  preprocess_kernel<DEG><<<(g->n + threads - 1) / threads, threads, 0, st>>>(                              \
      g->n, g->mean, g->scale, g->rot, g->opacity, g->sh, k, d, tm->active_bits,                           \
      reinterpret_cast<float2*>(out->mean2d), reinterpret_cast<float4*>(out->conic_o), out->depth,         \
      reinterpret_cast<short4*>(out->rect), out->tiles_touched, reinterpret_cast<float4*>(out->rgb_d),     \
      reinterpret_cast<float4*>(out->ncam), out->flags)
    switch (g->sh_degree) {
      case 0: PGSAG_A1(0); break;
      case 1: PGSAG_A1(1); break;
      case 2: PGSAG_A1(2); break;
      default: PGSAG_A1(3); break;
    }
#undef PGSAG_A1
  }
  return cudaGetLastError();
}

}  // namespace pgsag
