// NEXT-3: 3DGS adaptive density control (clone / split / prune) and the opacity reset,
// over the optimiser state of pgsag_adam_state (reading R31).
//
// The view-space gradient statistic is accumulated by A8 (preprocess_bwd.cu).  Here:
//   plan  : per Gaussian an action (0 drop, 1 keep, 2 keep + clone, 3 split), decided in
//           float32 exactly as the oracle does, plus per-1024-block counts of
//           (kept, cloned, split) and one single-CTA scan of the block counts;
//   apply : per block the intra-block prefix of the three flags (ballots), then every
//           source writes its kept copy, its clone and / or its two split children into
//           the output regions [kept | clones | split children] (source order inside each).
// Split children: mu + R(q) (s * z) with z from a counter-based SplitMix64 + Box-Muller
// generator (both sides implement it), scale s / 1.6, other parameters copied; clones and
// children start with zero Adam moments.  HBM-bound row copies.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.cuh"

namespace pgsag {
namespace {

constexpr int kDB = 1024;  // sources per block

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// three N(0, 1) samples of split child `child` of source i (oracle.split_normals)
__device__ __forceinline__ void split_normals(uint64_t seed, uint32_t i, int child, float (&z)[3]) {
  double out[4];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint64_t h = splitmix64(seed ^ (4ull * i + 2ull * child + (uint64_t)k));
    const double ua = ((double)(h >> 40) + 0.5) / 16777216.0;
    const double ub = ((double)(h & 0xFFFFFFull) + 0.5) / 16777216.0;
    const double r = sqrt(-2.0 * log(ua));
    double sn, cs;
    sincospi(2.0 * ub, &sn, &cs);
    out[2 * k] = r * cs;
    out[2 * k + 1] = r * sn;
  }
  z[0] = (float)out[0]; z[1] = (float)out[1]; z[2] = (float)out[2];
}

__device__ __forceinline__ int classify(int i, int n, const float* __restrict__ scale, const float* __restrict__ op,
                                        const float* __restrict__ accum, const float* __restrict__ count,
                                        pgsag_densify_params dp) {
  if (op[i] < dp.min_opacity) return 0;
  const float c = count[i];
  const float avg = c > 0.f ? __fdiv_rn(accum[i], c) : 0.f;
  if (!(avg >= dp.grad_threshold)) return 1;
  const float s = fmaxf(fmaxf(scale[i], scale[n + i]), scale[2 * n + i]);
  return s > dp.dense_limit ? 3 : 2;
}

__global__ void __launch_bounds__(kDB) densify_classify_kernel(int n, const float* __restrict__ scale,
                                                               const float* __restrict__ op,
                                                               const float* __restrict__ accum,
                                                               const float* __restrict__ count,
                                                               pgsag_densify_params dp, uint8_t* __restrict__ action,
                                                               uint32_t* __restrict__ block_cnt) {
  __shared__ uint32_t s_c[3];
  if (threadIdx.x < 3) s_c[threadIdx.x] = 0;
  __syncthreads();
  const int i = blockIdx.x * kDB + threadIdx.x;
  int a = -1;
  if (i < n) {
    a = classify(i, n, scale, op, accum, count, dp);
    action[i] = (uint8_t)a;
  }
  const uint32_t kb = __ballot_sync(0xffffffffu, a == 1 || a == 2);
  const uint32_t cb = __ballot_sync(0xffffffffu, a == 2);
  const uint32_t sb = __ballot_sync(0xffffffffu, a == 3);
  if ((threadIdx.x & 31) == 0) {
    if (kb) atomicAdd(&s_c[0], __popc(kb));
    if (cb) atomicAdd(&s_c[1], __popc(cb));
    if (sb) atomicAdd(&s_c[2], __popc(sb));
  }
  __syncthreads();
  if (threadIdx.x < 3) block_cnt[3 * blockIdx.x + threadIdx.x] = s_c[threadIdx.x];
}

// exclusive scan of the block counts (one CTA, sequential chunks of 1024) + totals
__global__ void __launch_bounds__(kDB) densify_scan_kernel(int nb, uint32_t* __restrict__ block_cnt,
                                                           unsigned long long* __restrict__ totals) {
  __shared__ uint32_t s_w[32][3];
  __shared__ uint32_t s_carry[3];
  const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
  if (tid < 3) s_carry[tid] = 0;
  __syncthreads();
  for (int base = 0; base < nb; base += kDB) {
    const int b = base + tid;
    uint32_t v[3] = {0, 0, 0};
    if (b < nb)
#pragma unroll
      for (int f = 0; f < 3; ++f) v[f] = block_cnt[3 * b + f];
    uint32_t inc[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      inc[f] = v[f];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc[f], o);
        if (lane >= o) inc[f] += t;
      }
      if (lane == 31) s_w[wi][f] = inc[f];
    }
    __syncthreads();
    if (wi == 0) {
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        uint32_t x = s_w[lane][f];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += t;
        }
        s_w[lane][f] = x;  // inclusive over warps
      }
    }
    __syncthreads();
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const uint32_t ex = s_carry[f] + (wi ? s_w[wi - 1][f] : 0u) + inc[f] - v[f];
      if (b < nb) block_cnt[3 * b + f] = ex;
    }
    __syncthreads();
    if (tid < 3) s_carry[tid] += s_w[31][tid];
    __syncthreads();
  }
  if (tid < 3) totals[tid] = s_carry[tid];
}

struct ApplyArgs {
  int n, K3;
  pgsag_adam_state src, dst;
  const uint8_t* action;
  const uint32_t* block_off;
  uint32_t K, C;  // kept count, clone count
  int n_out;
  uint64_t seed;
};

__device__ __forceinline__ void copy_params(const ApplyArgs& A, int i, int j, bool moments) {
  const size_t n = A.n, m = A.n_out;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    A.dst.mean[c * m + j] = A.src.mean[c * n + i];
    A.dst.scale[c * m + j] = A.src.scale[c * n + i];
    A.dst.log_scale[c * m + j] = A.src.log_scale[c * n + i];
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) A.dst.rot[c * m + j] = A.src.rot[c * n + i];
  A.dst.opacity[j] = A.src.opacity[i];
  A.dst.logit_opacity[j] = A.src.logit_opacity[i];
  for (int c = 0; c < A.K3; ++c) A.dst.sh[c * m + j] = A.src.sh[c * n + i];
  for (int r = 0; r < 11 + A.K3; ++r) {
    A.dst.m[r * m + j] = moments ? A.src.m[r * n + i] : 0.f;
    A.dst.v[r * m + j] = moments ? A.src.v[r * n + i] : 0.f;
  }
}

__global__ void __launch_bounds__(kDB) densify_apply_kernel(ApplyArgs A) {
  __shared__ uint32_t s_w[32][3];
  const int tid = threadIdx.x, lane = tid & 31, wi = tid >> 5;
  const int i = blockIdx.x * kDB + tid;
  const int a = i < A.n ? (int)A.action[i] : 0;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t bal[3], pre[3];
  bal[0] = __ballot_sync(0xffffffffu, a == 1 || a == 2);
  bal[1] = __ballot_sync(0xffffffffu, a == 2);
  bal[2] = __ballot_sync(0xffffffffu, a == 3);
  if (lane == 0)
#pragma unroll
    for (int f = 0; f < 3; ++f) s_w[wi][f] = __popc(bal[f]);
  __syncthreads();
  if (wi == 0) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const uint32_t v = s_w[lane][f];
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += t;
      }
      s_w[lane][f] = x - v;  // exclusive over warps
    }
  }
  __syncthreads();
#pragma unroll
  for (int f = 0; f < 3; ++f) pre[f] = A.block_off[3 * blockIdx.x + f] + s_w[wi][f] + __popc(bal[f] & lt);
  if (i >= A.n || a == 0) return;
  if (a == 1 || a == 2) copy_params(A, i, (int)pre[0], true);
  if (a == 2) copy_params(A, i, (int)(A.K + pre[1]), false);
  if (a == 3) {
    const size_t n = A.n, m = A.n_out;
    // R(q) of the normalised source quaternion (w, x, y, z)
    const float q0 = A.src.rot[i], q1 = A.src.rot[n + i], q2 = A.src.rot[2 * n + i], q3 = A.src.rot[3 * n + i];
    const float qn = rsqrtf(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);
    const float w = q0 * qn, x = q1 * qn, y = q2 * qn, z = q3 * qn;
    const float R[3][3] = {{1.f - 2.f * (y * y + z * z), 2.f * (x * y - w * z), 2.f * (x * z + w * y)},
                           {2.f * (x * y + w * z), 1.f - 2.f * (x * x + z * z), 2.f * (y * z - w * x)},
                           {2.f * (x * z - w * y), 2.f * (y * z + w * x), 1.f - 2.f * (x * x + y * y)}};
    const float s[3] = {A.src.scale[i], A.src.scale[n + i], A.src.scale[2 * n + i]};
#pragma unroll
    for (int ch = 0; ch < 2; ++ch) {
      const int j = (int)(A.K + A.C + 2 * pre[2] + ch);
      copy_params(A, i, j, false);
      float zz[3];
      split_normals(A.seed, (uint32_t)i, ch, zz);
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const float d = R[r][0] * (s[0] * zz[0]) + R[r][1] * (s[1] * zz[1]) + R[r][2] * (s[2] * zz[2]);
        A.dst.mean[r * m + j] = A.src.mean[r * n + i] + d;
        const float sc = s[r] / 1.6f;
        A.dst.scale[r * m + j] = sc;
        A.dst.log_scale[r * m + j] = logf(sc);
      }
    }
  }
}

__global__ void opacity_reset_kernel(int n, float* __restrict__ op, float* __restrict__ logit, float* __restrict__ m,
                                     float* __restrict__ v, float cap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float o = op[i];
  if (o > cap) {
    op[i] = cap;
    logit[i] = logf(cap / (1.0f - cap));
  }
  m[10 * (size_t)n + i] = 0.f;
  v[10 * (size_t)n + i] = 0.f;
}

}  // namespace

size_t densify_ws_bytes(int n) {
  const int nb = (n + kDB - 1) / kDB;
  return 256 + (size_t)(3 * nb + 1) * sizeof(uint32_t) + 64;
}

cudaError_t launch_densify_plan(int n, const float* scale, const float* op, const float* accum, const float* count,
                                const pgsag_densify_params* dp, uint8_t* action, void* ws, cudaStream_t st,
                                unsigned long long* totals_host) {
  const int nb = (n + kDB - 1) / kDB;
  unsigned long long* totals = reinterpret_cast<unsigned long long*>(ws);
  uint32_t* block_cnt = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + 256);
  cudaError_t e = cudaMemsetAsync(totals, 0, 3 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (n > 0) {
    {
      KTimer kt_("N3_densify_classify", st);
      densify_classify_kernel<<<nb, kDB, 0, st>>>(n, scale, op, accum, count, *dp, action, block_cnt);
    }
    {
      KTimer kt_("N3_densify_scan", st);
      densify_scan_kernel<<<1, kDB, 0, st>>>(nb, block_cnt, totals);
    }
  }
  e = cudaMemcpyAsync(totals_host, totals, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

cudaError_t launch_densify_apply(int n, int sh_degree, const pgsag_adam_state* src, const uint8_t* action,
                                 const pgsag_densify_params* dp, pgsag_adam_state* dst, int n_out, uint32_t K,
                                 uint32_t Cn, const void* ws, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  ApplyArgs A;
  A.n = n; A.K3 = (sh_degree + 1) * (sh_degree + 1) * 3;
  A.src = *src; A.dst = *dst;
  A.action = action;
  A.block_off = reinterpret_cast<const uint32_t*>(static_cast<const char*>(ws) + 256);
  A.K = K; A.C = Cn; A.n_out = n_out;
  A.seed = dp->seed;
  KTimer kt_("N3_densify_apply", st);
  densify_apply_kernel<<<(n + kDB - 1) / kDB, kDB, 0, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_opacity_reset(int n, pgsag_adam_state* s, float cap, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  KTimer kt_("N3_opacity_reset", st);
  opacity_reset_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, s->opacity, s->logit_opacity, s->m, s->v, cap);
  return cudaGetLastError();
}

}  // namespace pgsag
