// Internal declarations shared by the libpgsag.so translation units.
// Product code only: nothing here is shared with oracle/ (DESIGN.md §1).
#pragma once
#include "dcheck.cuh"
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pgsag.h"

namespace pgsag {

constexpr int kTile = PGSAG_TILE;        // 16x16 pixel tiles
constexpr int kTilePix = kTile * kTile;  // 256 pixels -> 256 threads per compositing CTA

// ---- sort configuration (A4) ----
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kMaxRadix = 512;  // 9-bit digits where they save a pass
constexpr int kSortThreads = 256;
#ifndef PGSAG_SORT_ITEMS
#define PGSAG_SORT_ITEMS 16
#endif
constexpr int kSortItems = PGSAG_SORT_ITEMS;
constexpr int kSortTile = kSortThreads * kSortItems;  // 4096 keys per CTA
constexpr uint32_t kLbAgg = 1u << 30;                 // look-back flags (top 2 bits)
constexpr uint32_t kLbPrefix = 2u << 30;
constexpr uint32_t kLbMask = (1u << 30) - 1;
constexpr int kScanTile = 4096;                       // A2 scan items per CTA
constexpr int kMaxSortPasses = 4;

struct Dims {
  int W, H, TX, TY, WPR;  // WPR = 32-bit words per bitmap row
};

inline Dims make_dims(int W, int H) {
  Dims d;
  d.W = W; d.H = H;
  d.TX = (W + kTile - 1) / kTile;
  d.TY = (H + kTile - 1) / kTile;
  d.WPR = (d.TX + 31) / 32;
  return d;
}

// Launch-configuration caches are kept per device (a process may drive several GPUs).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}

// Workspace carve-up, identical for every call with the same sizes.
struct WsLayout {
  size_t depth_keys[2], ids[2];  // stage-1 sort ping-pong [n]
  size_t offsets;                // [n] exclusive scan of tiles_touched in depth order
  size_t dup_keys, dup_vals;     // stage-2 sort scratch [capacity]
  size_t status1;                // stage-1 look-back [passes][tiles1][256] u32
  size_t status2;                // stage-2 look-back [passes][tiles2][256] u32
  size_t scan_status;            // A2 look-back [tilesN] u64
  size_t hist;                   // [2][kMaxSortPasses][256] u32
  size_t counters;               // [64] u32 (tile counters, M, misc); first: offset 0 for every size
  size_t zero_end;               // end of the state a sort call zeroes: [counters, zero_end)
  size_t a0;                     // [TY*WPR] u32 A0 scratch (bitmap word prefixes); offset depends on W, H only
  size_t g2d;                    // [n][16] f32 per-Gaussian 2D gradients (A7 -> A8; 14 used)
  size_t lpt;                    // [TY*TX] u32 (length class, slot) of each active tile (A5b)
  size_t total;
  int tiles1, tiles2, tilesN;
};

WsLayout ws_layout(int32_t n, int32_t W, int32_t H, int64_t cap);

// counters[] slots
enum : int {
  CNT_SORT1 = 0,   // 4 slots: stage-1 pass tile counters
  CNT_SORT2 = 4,   // 4 slots: stage-2 pass tile counters
  CNT_SCAN = 8,    // A2 tile counter
  CNT_FWD = 9,     // A6 work counter
  CNT_BWD = 10,    // A7 work counter
  CNT_M = 12,      // 2 slots: M as u64 (A2 total)
  CNT_MC = 14,     // M as u32 if M <= capacity, else 0 (published by A3: an overflowed view has empty lists)
  CNT_OVF = 15,    // 1 if M > capacity (published by A3; the fused A8 + Adam step is then skipped)
  CNT_NG = 16,     // n of the sorted view (published by A3; read by the debug bounds checks of A6)
  CNT_LPT = 24,    // 33 slots: active tiles per LPT length class (A5b)
  CNT_N = 57
};

// ------------------------------------------------------------- kernel timing
// RAII scope recording a CUDA event pair around one kernel launch when
// pgsag_timing_enable(1) is on (api.cu).
struct KTimer {
  int slot;
  cudaStream_t st;
  KTimer(const char* name, cudaStream_t s);
  ~KTimer();
};

// ---------------------------------------------------------------- launchers
cudaError_t launch_tilemask(const uint8_t* mask, const Dims& d, pgsag_tilemask* tm, uint32_t* scratch,
                            cudaStream_t st);
cudaError_t launch_preprocess(const pgsag_gaussians* g, const pgsag_camera* cam, const Dims& d,
                              const pgsag_tilemask* tm, pgsag_projected* out, cudaStream_t st);
cudaError_t launch_bin_sort_stage1(const pgsag_projected* p, int n, const WsLayout& L, char* ws,
                                   cudaStream_t st, const uint32_t** ids_sorted);
cudaError_t launch_duplicate_and_sort(const pgsag_projected* p, const pgsag_tilemask* tm, const Dims& d, int n,
                                      uint32_t M, bool M_known, const uint32_t* ids_sorted, const WsLayout& L,
                                      char* ws, pgsag_bins* bins, cudaStream_t st);
cudaError_t launch_render_fwd(const pgsag_projected* p, const pgsag_bins* bins, const pgsag_tilemask* tm,
                              const Dims& d, const pgsag_camera* cam, const uint8_t* mask, const float bg[3],
                              pgsag_image* out, uint32_t* work_counter, cudaStream_t st);
cudaError_t launch_render_bwd(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                              const pgsag_bins* bins, const pgsag_tilemask* tm, const Dims& d,
                              const uint8_t* mask, const float bg[3], const pgsag_image* fwd,
                              const pgsag_image_grad* dL, pgsag_gaussian_grad* out, float* g2d,
                              uint32_t* work_counter, cudaStream_t st, pgsag_adam_state* adam = nullptr,
                              const pgsag_adam_hparams* hp = nullptr, double* flat = nullptr,
                              const uint32_t* skip = nullptr);
// adam != NULL: A8 applies the Adam step (hp, L_s into *flat) instead of writing the gradients,
// unless the device flag *skip (the sort's overflow flag) is set
cudaError_t launch_preprocess_bwd(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                                  pgsag_gaussian_grad* out, const float* g2d, cudaStream_t st,
                                  pgsag_adam_state* adam = nullptr, const pgsag_adam_hparams* hp = nullptr,
                                  double* flat = nullptr, const uint32_t* skip = nullptr);
cudaError_t launch_gc_weights(const float* image, const uint8_t* mask, int W, int H, float* w, double* acc,
                              cudaStream_t st);

cudaError_t launch_boundary_band(const uint8_t* mask, int W, int H, int r, uint8_t* band, cudaStream_t st);
cudaError_t launch_ban_loss(const pgsag_camera* cam, const uint8_t* mask, const uint8_t* band, const float* N,
                            const float* Dep, float bw, float lambda, int mean, double* loss, float* dN, float* dDep,
                            cudaStream_t st);

cudaError_t launch_rgb_loss(const float* image, const float* target, const uint8_t* mask, int W, int H, float weight,
                            double* loss, float* dC, float* abc, cudaStream_t st);
cudaError_t launch_unpack_rgb8(const uint8_t* rgb, int W, int H, float* chw, cudaStream_t st);
cudaError_t launch_adam(int n, int sh_degree, const pgsag_gaussian_grad* gr, pgsag_adam_state* s,
                        const pgsag_adam_hparams* hp, double* flat, cudaStream_t st);
cudaError_t launch_adam_init(int n, pgsag_adam_state* s, cudaStream_t st);
cudaError_t launch_loss_total(const double* rgb, const double* flat, const double* ban, const double* gc, double lam,
                              double lam3, double lam4, int ban_mean, double* out, cudaStream_t st);
cudaError_t launch_finite_check(const pgsag_gaussians* g, unsigned int* bad, cudaStream_t st);

size_t densify_ws_bytes(int n);
cudaError_t launch_densify_plan(int n, const float* scale, const float* op, const float* accum, const float* count,
                                const pgsag_densify_params* dp, uint8_t* action, void* ws, cudaStream_t st,
                                unsigned long long* totals_host);
cudaError_t launch_densify_apply(int n, int sh_degree, const pgsag_adam_state* src, const uint8_t* action,
                                 const pgsag_densify_params* dp, pgsag_adam_state* dst, int n_out, uint32_t K,
                                 uint32_t Cn, const void* ws, cudaStream_t st);
cudaError_t launch_opacity_reset(int n, pgsag_adam_state* s, float cap, cudaStream_t st);

cudaError_t launch_fp32_microbench(int mode, int iters, float* scratch, float* ms, double* flops, cudaStream_t st);

// counters[] slots for pgsag_gc_weights: 8 (sum, count) double pairs at bytes 4*CNT_GC .. 4*CNT_GC + 127
constexpr int CNT_GC = 64;
constexpr int kCounters = 256;  // u32 slots of the workspace counter block
// A6's fused Eq. 9 statistics: kGcSlots (N, sum r, sum r^2) double triples at bytes 4*CNT_GCF.. (the
// warps of CTA b add into slot b % kGcSlots: 16x less contention than three global addresses)
constexpr int CNT_GCF = 128;
constexpr int kGcSlots = 16;

}  // namespace pgsag
