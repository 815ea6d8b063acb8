/*
 * pgsag.h — C ABI of libpgsag.so, the B200 (sm_100a) masked tile rasterizer of
 * PG-SAG (arXiv 2501.01677), forward and backward.
 *
 * Citations: P:n = PAPER.md line n (/root/reference, §3.1 "3DGS and Unbiased
 * Depth Rendering", Eq. 1-4, lines 76-96; §4.3 masked, pixel-parallel rendering,
 * line 163; masked pixels only, line 243).  Rk = reading k of DESIGN.md §3.
 *
 * General rules (all calls):
 *   - Every pointer is a DEVICE pointer unless marked (host).  The caller owns and
 *     allocates every buffer; the library never allocates device memory.  Scratch
 *     comes from the caller's workspace `ws` (>= pgsag_workspace_size bytes,
 *     256-byte aligned).
 *   - All work is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream) in call order.  The only host synchronisations are the
 *     read-back of M (the number of (tile, Gaussian) entries) in pgsag_bin_sort (not in
 *     pgsag_bin_sort_async) and of the output counts in pgsag_densify_plan.
 *   - Return value: PGSAG_OK (0) or a negative PGSAG_E* code; the message is in
 *     pgsag_last_error() (thread-local).  No exception crosses the ABI.  On error
 *     nothing is guaranteed about the output buffers.
 *   - Calls with distinct workspaces and outputs may run concurrently on
 *     different streams.
 *   - Image planes are planar row-major [H][W] (channel planes [c][H][W]); pixel
 *     (i, j) = column i, row j, centre (i + 0.5, j + 0.5) (R5).  Tiles are 16x16,
 *     TX = ceil(W/16), TY = ceil(H/16), tile id = ty*TX + tx.
 */
#ifndef PGSAG_H
#define PGSAG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGSAG_TILE 16

enum {
  PGSAG_OK = 0,
  PGSAG_EINVAL = -1,    /* null pointer, n < 0, sh_degree > 3, width/height <= 0, misaligned buffer */
  PGSAG_ECAPACITY = -2, /* bins->capacity < M; bins->n_dup holds M, nothing else written */
  PGSAG_ECUDA = -3,     /* a CUDA launch/copy failed; message in pgsag_last_error() */
  PGSAG_ENONFINITE = -4, /* a Gaussian parameter is NaN / inf (checked only with pgsag_set_checks(1):
                            finiteness is a precondition; the check costs a host sync) */
  PGSAG_EWORKSPACE = -5  /* ws_bytes < pgsag_workspace_size(...) */
};

/* Per-Gaussian flag bits written by pgsag_preprocess (A1). */
enum {
  PGSAG_F_VISIBLE = 1u << 0,    /* camera z > znear (R9)                               */
  PGSAG_F_DET_OK = 1u << 1,     /* det(cov2d + 0.3 I) > 0 (R10)                        */
  PGSAG_F_OPAC_OK = 1u << 2,    /* opacity >= 1/255 (R6)                               */
  PGSAG_F_RECT = 1u << 3,       /* conservative tile rect non-empty (R8)               */
  PGSAG_F_CLAMP_X = 1u << 4,    /* x/z clamped to 1.3 half-FoV inside J (R9)           */
  PGSAG_F_CLAMP_Y = 1u << 5,
  PGSAG_F_RGB_CLAMP0 = 1u << 6, /* colour channel c clamped at 0: bit 6 + c (R12)      */
  PGSAG_F_AXIS_SHIFT = 9,       /* bits 9-10: index of the minimum-scale axis (R4)     */
  PGSAG_F_NFLIP = 1u << 11,     /* normal flipped to face the camera (R4)              */
  PGSAG_F_LIVE = 15u            /* VISIBLE|DET_OK|OPAC_OK|RECT: Gaussian can emit keys */
};

/* Camera (host struct, by pointer).  x_cam = R (x_world - C) (P:88 R_c, P:92 T_C);
 * pinhole u = fx x/z + cx, v = fy y/z + cy (P:96 K).  znear default 0.01 (R9). */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
  float R[9]; /* world -> camera rotation, row-major */
  float C[3]; /* camera centre in world coordinates  */
  float znear;
} pgsag_camera;

/* Gaussians (host struct holding device pointers), structure-of-arrays, float32.
 * position, anisotropic scale, rotation, opacity, SH colour.  Values are
 * ACTIVATED (R13): scale > 0 linear, opacity in (0,1).  rot = (w,x,y,z), any
 * non-zero norm (normalised inside).  sh row (l*3 + c), l < (sh_degree+1)^2. */
typedef struct {
  int32_t n, sh_degree;      /* n >= 0, 0 <= sh_degree <= 3              */
  const float *mean;         /* [3][n]                                    */
  const float *scale;        /* [3][n]                                    */
  const float *rot;          /* [4][n]                                    */
  const float *opacity;      /* [n]                                       */
  const float *sh;           /* [(sh_degree+1)^2 * 3][n]                  */
} pgsag_gaussians;

/* A1 output: projected Gaussians (caller-allocated, n entries each, 16-B aligned). */
typedef struct {
  float *mean2d;          /* [n][2]  (u, v) pixel coordinates                          */
  float *conic_o;         /* [n][4]  (ca, cb, cc, o): power = -0.5(ca dx^2 + cc dy^2) - cb dx dy */
  float *depth;           /* [n]     camera z (sort key, R11)                          */
  int16_t *rect;          /* [n][4]  tile rect tx0, ty0, tx1, ty1 inclusive; empty = (0,0,-1,-1) */
  uint32_t *tiles_touched;/* [n]     active tiles inside rect (0 unless LIVE)          */
  float *rgb_d;           /* [n][4]  (r, g, b, d_i): SH colour (R12) and plane distance d_i (Eq. 3, R2) */
  float *ncam;            /* [n][4]  (R_c n_i, 0): camera-frame normal (Eq. 2, R4)     */
  uint32_t *flags;        /* [n]     PGSAG_F_* bits                                    */
} pgsag_projected;

/* A0 output: building-mask tile occupancy (R14). */
typedef struct {
  uint32_t *tile_cnt; /* [TY*TX]        number of mask pixels per tile                  */
  int32_t *sat;       /* [(TY+1)*(TX+1)] summed-area table of active (cnt > 0) tiles;
                         OPTIONAL (NULL = not computed; the path itself uses active_bits) */
  uint32_t *active;   /* [TY*TX]        active tile ids ascending; first *n_active valid  */
  uint32_t *n_active; /* [1]            device scalar                                     */
  uint32_t *active_bits; /* [TY*ceil(TX/32)] bitmap of active tiles, row-major, bit tx%32 */
} pgsag_tilemask;

/* A2-A5 output: per-tile sorted lists ("projected onto different image tiles ...
 * sorted"; R11).  Entry k: (tile_keys[k], vals[k] = Gaussian id), ordered by
 * (tile, depth bits, id).  ranges[2t], ranges[2t+1] = [start, end) of tile t
 * (empty tiles [0, 0)). */
typedef struct {
  uint32_t *tile_keys; /* [capacity], 16-byte aligned (the sort reads it with 128-bit loads) */
  uint32_t *vals;      /* [capacity], 16-byte aligned */
  uint32_t *ranges;    /* [2*TY*TX]  */
  int64_t capacity;    /* in: entries allocated            */
  int64_t n_dup;       /* out (host field): M              */
  uint32_t *order;     /* optional [TY*TX]: work order for A6/A7 = the active tiles by decreasing list
                          length (log2 classes), written by pgsag_bin_sort(_async); NULL = ascending ids */
} pgsag_bins;

/* A6 output (planar float32 [H][W] unless noted).  Only pixels with mask != 0 are
 * written; others are left untouched (R14).  Eq. 1 colour C (+ T bg, R15), Eq. 2
 * normal N, Eq. 3 distance D, alpha A = 1 - T, Eq. 4 unbiased depth Dep (0 = invalid,
 * R3), final transmittance T, blended count g (P:169 g_i), last = index k into
 * bins->vals of the last blended entry (-1 if none; used by the backward). */
typedef struct {
  float *C;     /* [3][H][W] */
  float *N;     /* [3][H][W] */
  float *D, *A, *Dep, *T;
  int32_t *g, *last;
  unsigned long long *counters; /* optional [4]: +E evaluated, +B blended (fwd), +E visited (bwd), 0 */
  /* Optional fused L_GC-load statistics (NEXT-1, Eq. 9).  If gc_w (input, [H][W], the
   * weights of pgsag_gc_weights) is non-NULL, A6 accumulates over the mask pixels
   * gc_stats[0] = N, gc_stats[1] = sum r, gc_stats[2] = sum r^2 with r = g / w (gc_stats is
   * zeroed by the call), and after the compositor gc_stats[3] = L_GC-load = the population std
   * sqrt(sum r^2 / N - (sum r / N)^2) ("std over all pixels"), gc_stats[4] = sum r / N.
   * gc_stats is double[5]. */
  const float *gc_w;
  double *gc_stats;
} pgsag_image;

/* Upstream gradients dL/d(C, N, D, A, Dep) in the pgsag_image layout; any may be NULL (= 0).
 * gc_lambda != 0 adds gc_lambda * L_GC-load (Eq. 11's lambda term) through the soft-count
 * surrogate sum_blended sigmoid(100 (alpha - 1/255)) (R24); it needs the forward's gc_w and
 * gc_stats. */
typedef struct {
  const float *dC, *dN, *dD, *dA, *dDep;
  float gc_lambda;
  /* optional device scalar: if non-NULL, dN and dDep are divided by *nd_div (multiplied by 0 when
   * *nd_div <= 0), e.g. the term count of a mean loss whose sum-gradient was written in one pass
   * (pgsag_ban_loss with mean = 0). */
  const double *nd_div;
} pgsag_image_grad;

/* A8 output, same layouts as pgsag_gaussians; OVERWRITTEN (not accumulated).  Rows of dsh
 * beyond (sh_degree+1)^2*3 are not touched.  absgrad2d optional [n]: sum over pixels of
 * |dL/du_p| + |dL/dv_p| (densification statistic).  Non-LIVE Gaussians get 0. */
typedef struct {
  float *dmean, *dscale, *drot, *dopacity, *dsh, *absgrad2d;
  float *grad2d; /* optional [14][n]: the per-Gaussian screen-space gradients du, dv, d(ca,cb,cc), d o,
                    d rgb[3], d n_cam[3], d d_i, absgrad (A7 sums moments of alpha*dalpha per
                    Gaussian; A8 forms du, dv, the conic and opacity gradients from them) */
  /* Optional densification statistic (NEXT-3, R31), ACCUMULATED across calls: for every Gaussian with
   * tiles_touched > 0, densify_accum[i] += |(du W/2, dv H/2)| (3DGS's view-space positional gradient
   * norm) and densify_count[i] += 1.  Both NULL or both [n]. */
  float *densify_accum, *densify_count;
} pgsag_gaussian_grad;

/* Bytes of scratch needed by every call for n Gaussians, a width x height image and
 * dup_capacity (tile, Gaussian) entries. */
size_t pgsag_workspace_size(int32_t n, int32_t width, int32_t height, int64_t dup_capacity);

/* A0 + A1.  A0: tile occupancy of the building mask `mask` (u8 [H][W], nonzero =
 * building pixel, the paper's RBM).  A1: per Gaussian, EWA projection
 * (P:78), culling, opacity-aware conservative tile rect (R8), active tiles touched,
 * flattened normal n_i (R4), d_i (Eq. 3, R2), SH colour (R12).  Key-path
 * arithmetic is IEEE float32 with no contraction (bit-exact with the oracle).  ws: scratch of at least
 * pgsag_workspace_size(n, width, height, 0) bytes (A0's word prefixes; the debug finiteness check),
 * normally the workspace the view's pgsag_bin_sort uses. */
int pgsag_preprocess(const pgsag_gaussians *g, const pgsag_camera *cam, const uint8_t *mask,
                     pgsag_tilemask *tm, pgsag_projected *out, void *ws, size_t ws_bytes, void *stream);

/* A2-A5: stable sort of Gaussians by depth, exclusive scan of tiles_touched,
 * duplication of (tile, id) entries for active tiles in each rect, stable radix sort
 * by tile, tile ranges.  Host-synchronises once to read M into bins->n_dup; returns
 * PGSAG_ECAPACITY if M > bins->capacity. */
int pgsag_bin_sort(const pgsag_projected *p, const pgsag_tilemask *tm, const pgsag_camera *cam, int32_t n,
                   pgsag_bins *bins, void *ws, size_t ws_bytes, void *stream);

/* A2-A5 without any host synchronisation (same outputs as pgsag_bin_sort when M <= capacity): every
 * grid is bounded by bins->capacity and the kernels read M on the device.  bins->n_dup is set to -1.
 * If m_out is non-NULL (pinned host or device memory) M is copied there, stream-ordered, after the
 * sort; the caller must check it once the stream has passed this point: if M > capacity the lists
 * are incomplete and the view must be re-sorted with capacity >= M (nothing is written past the
 * capacity; the device-side entry count is then 0, so the later stages see empty lists, and the
 * workspace's overflow flag makes pgsag_render_bwd_adam skip its update). */
int pgsag_bin_sort_async(const pgsag_projected *p, const pgsag_tilemask *tm, const pgsag_camera *cam, int32_t n,
                         pgsag_bins *bins, unsigned long long *m_out, void *ws, size_t ws_bytes, void *stream);

/* A6: per active tile, per masked pixel, front-to-back compositing over the tile's
 * sorted list (Eq. 1-3; alpha = min(0.99, o exp(power)), skip alpha < 1/255,
 * stop when T would drop below 1e-4 — the crossing entry is not blended, R6), then
 * Eq. 4.  bg (host, 3 floats) enters C only via T bg (R15). */
int pgsag_render_fwd(const pgsag_projected *p, const pgsag_bins *bins, const pgsag_tilemask *tm,
                     const pgsag_camera *cam, const uint8_t *mask, const float bg[3], pgsag_image *out,
                     void *ws, size_t ws_bytes, void *stream);

/* A7 + A8: exact reverse-mode gradient of the A6 outputs w.r.t. the Gaussian
 * parameters, decisions (sort, skip, termination, culls, clamps) frozen (R16, R17).
 * fwd must be the pgsag_image A6 wrote for the same inputs. */
int pgsag_render_bwd(const pgsag_gaussians *g, const pgsag_camera *cam, const pgsag_projected *p,
                     const pgsag_bins *bins, const pgsag_tilemask *tm, const uint8_t *mask, const float bg[3],
                     const pgsag_image *fwd, const pgsag_image_grad *dL, pgsag_gaussian_grad *out, void *ws,
                     size_t ws_bytes, void *stream);

/* NEXT-1: Eq. 9's gradient-dependent weights w_i ("gradient-dependent weight nabla I",
 * P:165-169; reading R23): gray = 0.299 R + 0.587 G + 0.114 B of image ([3][H][W] float),
 * 3x3 Sobel magnitude with replicated borders, divided by its mean over the mask pixels,
 * clamped to [0.1, 10] (floor everywhere if that mean is 0); w = 1 off the mask.
 * w is [H][W] float, caller-allocated. */
int pgsag_gc_weights(const float *image, const uint8_t *mask, int32_t width, int32_t height, float *w,
                     void *ws, size_t ws_bytes, void *stream);

/* NEXT-2: boundary band MB ("extract more accurate building masked boundaries"; R25):
 * band = dilation(mask, r) XOR erosion(mask, r) with a (2r+1)^2 square structuring element,
 * zero outside the image.  mask, band: u8 [H][W]; r >= 1. */
int pgsag_boundary_band(const uint8_t *mask, int32_t width, int32_t height, int32_t r, uint8_t *band,
                        void *stream);

/* NEXT-2: boundary-aware normal loss L_ban (Eq. 8; R26, R27).  For each mask pixel
 * whose four axis neighbours are inside the image and the mask with a valid unbiased depth
 * (Dep != 0): P_k = Dep_k K^-1 (x+.5, y+.5, 1); n_depth = normalize((P_right - P_left) x
 * (P_down - P_up)) turned to face the camera ("four neighboring points"); n_rendered =
 * N/|N|; term = w |n_depth - n_rendered|^2 with w = boundary_w on the band ("0.1") and 1
 * elsewhere in the mask.  loss (device, double[2], zeroed by the call) receives
 * (sum of terms, number of terms).  If dN ([3][H][W]) / dDep ([H][W]) are non-NULL the call
 * ADDS lambda * d(S)/dN, lambda * d(S)/dDep, with S = sum (mean = 0) or sum / count (mean = 1),
 * ready to be passed as upstream to pgsag_render_bwd.  N and Dep are A6 outputs.  mean = 0 takes
 * one pass over the image (mean = 1 two); the gradient of the mean is then obtained in A7 by
 * pointing pgsag_image_grad.nd_div at loss + 1. */
int pgsag_ban_loss(const pgsag_camera *cam, const uint8_t *mask, const uint8_t *band, const float *N,
                   const float *Dep, float boundary_w, float lambda, int32_t mean, double *loss, float *dN,
                   float *dDep, void *stream);

/* ------------------------------------------------------------------ NEXT-3: training step
 * Eq. 10-11: L = (1 - lambda) (L_rgb + lambda3 L_s + lambda4 L_ban) + lambda L_GC-load,
 * lambda = 0.41, lambda3 = 100, lambda4 = 0.01; the multi-view PGSR terms (lambda1, lambda2)
 * are out of scope.  The driver composes: A0-A6 -> pgsag_rgb_loss (+ pgsag_ban_loss)
 * -> A7/A8 (gc_lambda = lambda) -> pgsag_adam_step. */

/* The photo as captured: 8-bit interleaved RGB rgb8[H][W][3] -> image[3][H][W] float in [0, 1]
 * (b / 255 correctly rounded), the layout pgsag_rgb_loss / pgsag_gc_weights take.  rgb8 4-byte and
 * image 16-byte aligned, W*H a multiple of 4. */
int pgsag_unpack_rgb8(const uint8_t *rgb8, int32_t width, int32_t height, float *image, void *stream);

/* Scratch bytes for pgsag_rgb_loss on a width x height image (36 W H). */
size_t pgsag_rgb_loss_workspace_size(int32_t width, int32_t height);

/* Masked photometric loss L_rgb = 0.8 L1 + 0.2 (1 - SSIM) over the RBM pixels ("only the refined
 * building masks RBM are involved in these losses"; form R28): x = image m, y = target m (zero off
 * the mask); per channel the 11x11 Gaussian-window (sigma 1.5, zero padding) SSIM map with
 * C1 = 0.01^2, C2 = 0.03^2; L1 and S are means over mask pixels and the 3 channels.
 * image, target: [3][H][W] float; mask u8 [H][W].  loss (device double[6], zeroed by the call):
 * (L_rgb, L1, S, sum |C - I|, sum S, mask pixel count).  If dC ([3][H][W]) is non-NULL it receives
 * weight * dL_rgb/dimage at the mask pixels (other pixels untouched). */
int pgsag_rgb_loss(const float *image, const float *target, const uint8_t *mask, int32_t width, int32_t height,
                   float weight, double *loss, float *dC, void *ws, size_t ws_bytes, void *stream);

/* Optimiser state of one sub-region's Gaussians (device pointers, caller-owned).  The activated
 * arrays (pgsag_gaussians layouts) are rewritten from the raw ones after every step (R30):
 * scale = exp(log_scale), opacity = sigmoid(logit_opacity); mean, rot, sh are their own raw values.
 * m, v: Adam moments, [11 + K3][n] rows mean 0-2, log_scale 3-5, rot 6-9, logit_opacity 10,
 * sh 11.. (K3 = (sh_degree+1)^2 * 3); zero-initialise them before step 1. */
typedef struct {
  float *mean, *scale, *rot, *opacity, *sh;
  float *log_scale;     /* [3][n] */
  float *logit_opacity; /* [n]    */
  float *m, *v;
} pgsag_adam_state;

/* Adam hyper-parameters (host struct).  step = t >= 1 for the bias corrections 1 - beta^t.
 * flatten_weight = the weight of L_s in L ((1 - lambda) lambda3 for Eq. 10-11). */
typedef struct {
  float lr_mean, lr_scale, lr_rot, lr_opacity, lr_sh_dc, lr_sh_rest;
  float beta1, beta2, eps;
  float flatten_weight;
  int32_t step;
} pgsag_adam_hparams;

/* The raw parameters the optimiser updates (R30, 3DGS's parameterisation) from the activated ones:
 * state->log_scale = log(state->scale), state->logit_opacity = log(o / (1 - o)) (evaluated in
 * double, stored as float), for n Gaussians.  Call once before the first pgsag_adam_step. */
int pgsag_adam_init(int32_t n, pgsag_adam_state *state, void *stream);

/* Eq. 11 on the device: total[0] = (1 - lambda) (rgb_loss[0] + lambda3 flatten_loss[0] +
 * lambda4 L_ban) + lambda gc_stats[3], with L_ban = ban_loss[0] / ban_loss[1] (ban_mean = 1; 0 if
 * the count is 0) or ban_loss[0] (ban_mean = 0).  rgb_loss is pgsag_rgb_loss's output, flatten_loss
 * pgsag_adam_step's, ban_loss pgsag_ban_loss's, gc_stats pgsag_render_fwd's (pgsag_image.gc_stats);
 * flatten_loss, ban_loss and gc_stats may be NULL (term absent).  All device pointers. */
int pgsag_loss_total(const double *rgb_loss, const double *flatten_loss, const double *ban_loss, int32_t ban_mean,
                     const double *gc_stats, float lambda, float lambda3, float lambda4, double *total,
                     void *stream);

/* One Adam step (Kingma & Ba) on the raw parameters with the gradients of pgsag_render_bwd (w.r.t.
 * the activated values, chained through exp / sigmoid here) plus flatten_weight * dL_s/dscale,
 * L_s = mean over the n Gaussians of min(scale) (PGSR flattening; R29; ties -> lowest
 * axis).  flatten_loss (device double[1], optional, zeroed by the call) receives L_s evaluated
 * before the update. */
int pgsag_adam_step(int32_t n, int32_t sh_degree, const pgsag_gaussian_grad *grad, pgsag_adam_state *state,
                    const pgsag_adam_hparams *hp, double *flatten_loss, void *stream);

/* A7 + A8 fused with the Adam step: the gradients pgsag_render_bwd computes, applied inside A8 by
 * exactly pgsag_adam_step's update (same float32 gradients, same arithmetic: bitwise the same
 * parameters, moments and L_s) instead of being written to memory (P:82 differentiable rendering +
 * P:171-179 optimisation).  Arguments as pgsag_render_bwd and pgsag_adam_step; state
 * must describe the same Gaussians as g (its mean / scale / rot / opacity / sh are g's arrays).  Of
 * out only absgrad2d, grad2d, densify_accum and densify_count are used (all optional); its
 * parameter-gradient pointers may be NULL.  For one optimiser per sub-region: ranks that average
 * gradients first (NEXT-4) call pgsag_render_bwd, all-reduce, then pgsag_adam_step.
 * ws must be the workspace this view's pgsag_bin_sort(_async) used: if that sort overflowed the
 * capacity (M > capacity, pgsag_bin_sort_async; the lists are then empty) the Adam update is
 * skipped on the device (parameters, moments untouched), so a sync-free caller can detect the
 * overflow afterwards and re-run the view without having applied a step from incomplete lists. */
int pgsag_render_bwd_adam(const pgsag_gaussians *g, const pgsag_camera *cam, const pgsag_projected *p,
                          const pgsag_bins *bins, const pgsag_tilemask *tm, const uint8_t *mask, const float bg[3],
                          const pgsag_image *fwd, const pgsag_image_grad *dL, pgsag_gaussian_grad *out,
                          pgsag_adam_state *state, const pgsag_adam_hparams *hp, double *flatten_loss, void *ws,
                          size_t ws_bytes, void *stream);

/* ------------------------------------------------------------ NEXT-3: densification (R31)
 * 3DGS adaptive density control on a sub-region's optimiser state (the paper
 * trains every group with it, and gives no parameters: 3DGS's conventions). */
typedef struct {
  float grad_threshold; /* densify if accum / count >= this (3DGS 0.0002, NDC units)          */
  float dense_limit;    /* percent_dense * scene extent: clone if max scale <= it, else split */
  float min_opacity;    /* prune if opacity < it (3DGS 0.005)                                 */
  uint64_t seed;        /* split samples: SplitMix64 + Box-Muller counter generator (R31)     */
} pgsag_densify_params;

/* Scratch bytes for pgsag_densify_plan / _apply on n Gaussians. */
size_t pgsag_densify_workspace_size(int32_t n);

/* Plan: action[i] (device u8 [n], out) = 0 drop (opacity < min_opacity), 3 split (accum/count >=
 * grad_threshold and max scale > dense_limit), 2 keep + clone (same, max scale <= dense_limit),
 * 1 keep; every decision in float32.  counts (host int64[3], out) = (kept, cloned, split); the
 * output has n_out = kept + cloned + 2 split Gaussians.  Synchronises the stream once (the caller
 * needs n_out to allocate).  ws must be passed unchanged to pgsag_densify_apply. */
int pgsag_densify_plan(int32_t n, const float *scale, const float *opacity, const float *accum, const float *count,
                       const pgsag_densify_params *dp, uint8_t *action, int64_t counts[3], void *ws, size_t ws_bytes,
                       void *stream);

/* Apply the plan: dst (n_out Gaussians, caller-allocated, same layouts) receives the kept sources
 * (source order), then the clones (source order), then the two children of each split source
 * (source order): mean + R(q)(s * z), scale s / 1.6, log_scale = log of it, rot / opacity / SH
 * copied.  Kept Gaussians keep their Adam moments; clones and children get zero moments.
 * src and dst must not overlap. */
int pgsag_densify_apply(int32_t n, int32_t sh_degree, const pgsag_adam_state *src, const uint8_t *action,
                        const pgsag_densify_params *dp, const int64_t counts[3], pgsag_adam_state *dst,
                        const void *ws, size_t ws_bytes, void *stream);

/* 3DGS opacity reset: opacity = min(opacity, cap), logit_opacity updated, the Adam moments of the
 * opacity row zeroed. */
int pgsag_opacity_reset(int32_t n, pgsag_adam_state *state, float cap, void *stream);

/* Measurement aid: FP32 FMA throughput of the device from independent chains on
 * all SMs; mode 0 = scalar FFMA, mode 1 = packed FFMA2 (FP32x2).  Synchronises; writes TFLOP/s
 * (FMA = 2 flop) to *tflops (host).  scratch: device float[256]. */
int pgsag_microbench_fp32(int32_t mode, int32_t iters, float *scratch, double *tflops, void *stream);

/* Message for the last non-zero status on this thread ("" if none). */
const char *pgsag_last_error(void);

/* Debug checks: level 1 makes pgsag_preprocess verify that every Gaussian parameter is finite
 * (SPEC S:289 makes finiteness a precondition) and return PGSAG_ENONFINITE otherwise; the check
 * reads all parameters and synchronises the stream once (ws must hold >= 256 bytes).  0 (default)
 * disables it.  Process-wide. */
void pgsag_set_checks(int level);

/* Library version string, e.g. "pgsag-b200 0.1 sm_100a". */
const char *pgsag_version(void);

/* Optional per-kernel timing (profiling aid; off by default, process-global).
 * pgsag_timing_enable(1) makes every kernel launch of the library record a CUDA
 * event pair on its own launch stream.  pgsag_timing_collect() synchronises on the
 * recorded events, aggregates them per kernel name, clears the record list and
 * returns the number K of distinct kernels; pgsag_timing_get(k, ...) (0 <= k < K)
 * returns the kernel name (static storage), the summed milliseconds and the number
 * of launches.  Returns PGSAG_EINVAL for k out of range. */
void pgsag_timing_enable(int on);
/* Restrict the timing to kernels whose name starts with prefix (NULL or "" = all), e.g. only
 * the dominant kernel inside a timed region, so the other launches carry no event records. */
void pgsag_timing_filter(const char *prefix);
int pgsag_timing_collect(void);
int pgsag_timing_get(int k, const char **name, double *ms, long long *launches);

#ifdef __cplusplus
}
#endif

#endif /* PGSAG_H */
