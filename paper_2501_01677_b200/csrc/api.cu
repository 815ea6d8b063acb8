// C ABI of libpgsag.so (include/pgsag.h): argument validation, workspace
// carving, stream-ordered launches, error reporting.  No exception or torch type
// crosses this boundary; the library never allocates device memory.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstring>
#include <string>

#include "internal.cuh"

#include <map>
#include <atomic>
#include <mutex>
#include <vector>

using namespace pgsag;

namespace {

// ------------------------------------------------------------ kernel timing
struct TimingRec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_tmu;
bool g_timing = false;
std::string g_timing_prefix;  // only kernels whose name starts with it ("" = all)
std::vector<TimingRec> g_recs;
std::vector<cudaEvent_t> g_pool;
std::vector<std::pair<const char*, std::pair<double, long long>>> g_agg;

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

namespace pgsag {
KTimer::KTimer(const char* name, cudaStream_t s) : slot(-1), st(s) {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (!g_timing) return;
  if (!g_timing_prefix.empty() && strncmp(name, g_timing_prefix.c_str(), g_timing_prefix.size()) != 0) return;
  TimingRec r{name, take_event(), take_event()};
  cudaEventRecord(r.a, st);
  g_recs.push_back(r);
  slot = (int)g_recs.size() - 1;
}
KTimer::~KTimer() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  if (slot < (int)g_recs.size()) cudaEventRecord(g_recs[slot].b, st);
}
}  // namespace pgsag

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  char buf[256];
  snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
  g_err = buf;
  return PGSAG_ECUDA;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int check_cam(const pgsag_camera* c) {
  if (!c) return fail(PGSAG_EINVAL, "camera is NULL");
  if (c->width <= 0 || c->height <= 0) return fail(PGSAG_EINVAL, "width/height must be > 0");
  if (!(c->fx > 0.f) || !(c->fy > 0.f)) return fail(PGSAG_EINVAL, "fx/fy must be > 0");
  if (c->width > (1 << 19) || c->height > (1 << 19)) return fail(PGSAG_EINVAL, "image too large");
  return PGSAG_OK;
}

int check_proj(const pgsag_projected* p) {
  if (!p || !p->mean2d || !p->conic_o || !p->depth || !p->rect || !p->tiles_touched || !p->rgb_d || !p->ncam ||
      !p->flags)
    return fail(PGSAG_EINVAL, "projected buffer is NULL");
  if (!aligned(p->conic_o, 16) || !aligned(p->rgb_d, 16) || !aligned(p->ncam, 16) || !aligned(p->mean2d, 8) ||
      !aligned(p->rect, 8))
    return fail(PGSAG_EINVAL, "projected buffers must be 16-byte aligned (mean2d, rect: 8)");
  return PGSAG_OK;
}

int check_tm(const pgsag_tilemask* tm) {
  if (!tm || !tm->tile_cnt || !tm->active || !tm->n_active || !tm->active_bits)
    return fail(PGSAG_EINVAL, "tilemask buffer is NULL");
  return PGSAG_OK;
}

std::atomic<int> g_checks{0};  // pgsag_set_checks: 1 = finiteness precondition of the Gaussians

int check_g(const pgsag_gaussians* g) {
  if (!g) return fail(PGSAG_EINVAL, "gaussians is NULL");
  if (g->n < 0) return fail(PGSAG_EINVAL, "n < 0");
  if (g->sh_degree < 0 || g->sh_degree > 3) return fail(PGSAG_EINVAL, "sh_degree must be 0..3");
  if (g->n > 0 && (!g->mean || !g->scale || !g->rot || !g->opacity || !g->sh))
    return fail(PGSAG_EINVAL, "gaussian parameter is NULL");
  return PGSAG_OK;
}

int check_ws(void* ws, size_t ws_bytes, size_t need) {
  if (need && !ws) return fail(PGSAG_EINVAL, "workspace is NULL");
  if (ws && !aligned(ws, 256)) return fail(PGSAG_EINVAL, "workspace must be 256-byte aligned");
  if (ws_bytes < need) return fail(PGSAG_EWORKSPACE, "workspace too small (see pgsag_workspace_size)");
  return PGSAG_OK;
}

}  // namespace

extern "C" {

const char* pgsag_last_error(void) { return g_err.c_str(); }

const char* pgsag_version(void) { return "pgsag-b200 0.2 sm_100a"; }

void pgsag_set_checks(int level) { g_checks.store(level); }

void pgsag_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = on != 0;
}

void pgsag_timing_filter(const char* prefix) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing_prefix = prefix ? prefix : "";
}

int pgsag_timing_collect(void) {
  std::lock_guard<std::mutex> lk(g_tmu);
  std::map<std::string, std::pair<double, long long>> agg;
  std::map<std::string, const char*> names;
  for (const TimingRec& r : g_recs) {
    cudaEventSynchronize(r.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& a = agg[r.name];
    a.first += ms;
    a.second += 1;
    names[r.name] = r.name;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  g_agg.clear();
  for (auto& kv : agg) g_agg.push_back({names[kv.first], kv.second});
  return (int)g_agg.size();
}

int pgsag_timing_get(int k, const char** name, double* ms, long long* launches) {
  std::lock_guard<std::mutex> lk(g_tmu);
  if (k < 0 || k >= (int)g_agg.size()) return PGSAG_EINVAL;
  if (name) *name = g_agg[k].first;
  if (ms) *ms = g_agg[k].second.first;
  if (launches) *launches = g_agg[k].second.second;
  return PGSAG_OK;
}

size_t pgsag_workspace_size(int32_t n, int32_t width, int32_t height, int64_t dup_capacity) {
  return ws_layout(n, width, height, dup_capacity).total;
}

int pgsag_preprocess(const pgsag_gaussians* g, const pgsag_camera* cam, const uint8_t* mask, pgsag_tilemask* tm,
                     pgsag_projected* out, void* ws, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_g(g)) || (rc = check_cam(cam)) || (rc = check_tm(tm))) return rc;
  if (!mask) return fail(PGSAG_EINVAL, "mask is NULL");
  if (g->n > 0 && (rc = check_proj(out))) return rc;
  const WsLayout L = ws_layout(g->n, cam->width, cam->height, 0);
  if ((rc = check_ws(ws, ws_bytes, L.a0 + 4 * (size_t)make_dims(cam->width, cam->height).TY *
                                               make_dims(cam->width, cam->height).WPR)))
    return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims d = make_dims(cam->width, cam->height);
  cudaError_t e;
  if (g_checks.load() && g->n > 0) {  // S:289 precondition, debug only (one host sync)
    unsigned int* bad = static_cast<unsigned int*>(ws);
    unsigned int nb = 0;
    e = cudaMemsetAsync(bad, 0, sizeof(unsigned int), st);
    if (e == cudaSuccess) e = launch_finite_check(g, bad, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nb, bad, sizeof(nb), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "finite check");
    if (nb) return fail(PGSAG_ENONFINITE, "non-finite Gaussian parameter (pgsag_set_checks)");
  }
  e = launch_tilemask(mask, d, tm, reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + L.a0), st);
  if (e != cudaSuccess) return cuda_fail(e, "tilemask");
  e = launch_preprocess(g, cam, d, tm, out, st);
  if (e != cudaSuccess) return cuda_fail(e, "preprocess");
  return PGSAG_OK;
}

int pgsag_bin_sort(const pgsag_projected* p, const pgsag_tilemask* tm, const pgsag_camera* cam, int32_t n,
                   pgsag_bins* bins, void* ws, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_cam(cam)) || (rc = check_tm(tm))) return rc;
  if (n < 0) return fail(PGSAG_EINVAL, "n < 0");
  if (n > 0 && (rc = check_proj(p))) return rc;
  if (!bins || !bins->ranges || (bins->capacity > 0 && (!bins->tile_keys || !bins->vals)))
    return fail(PGSAG_EINVAL, "bins buffer is NULL");
  if (!aligned(bins->tile_keys, 16) || !aligned(bins->vals, 16))
    return fail(PGSAG_EINVAL, "bins tile_keys / vals must be 16-byte aligned");
  if (bins->capacity < 0 || bins->capacity >= (int64_t)kLbMask)
    return fail(PGSAG_EINVAL, "bins capacity must be in [0, 2^30)");
  const WsLayout L = ws_layout(n, cam->width, cam->height, bins->capacity);
  if ((rc = check_ws(ws, ws_bytes, L.total))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims d = make_dims(cam->width, cam->height);
  char* w = static_cast<char*>(ws);
  uint32_t* counters = reinterpret_cast<uint32_t*>(w + L.counters);
  cudaError_t e;
  // zero the look-back / histogram / counter state of stage 1 and A2
  e = cudaMemsetAsync(w + L.counters, 0, L.zero_end - L.counters, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  unsigned long long M = 0;
  const uint32_t* ids_sorted = nullptr;
  if (n > 0) {
    e = launch_bin_sort_stage1(p, n, L, w, st, &ids_sorted);
    if (e != cudaSuccess) return cuda_fail(e, "depth sort / scan");
    e = cudaMemcpyAsync(&M, counters + CNT_M, sizeof(M), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "read M");
  }
  bins->n_dup = (int64_t)M;
  if ((int64_t)M > bins->capacity) return fail(PGSAG_ECAPACITY, "bins capacity < M (bins->n_dup holds M)");
  e = launch_duplicate_and_sort(p, tm, d, n, (uint32_t)M, true, ids_sorted, L, w, bins, st);
  if (e != cudaSuccess) return cuda_fail(e, "duplicate / tile sort / ranges");
  return PGSAG_OK;
}

int pgsag_bin_sort_async(const pgsag_projected* p, const pgsag_tilemask* tm, const pgsag_camera* cam, int32_t n,
                         pgsag_bins* bins, unsigned long long* m_out, void* ws, size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_cam(cam)) || (rc = check_tm(tm))) return rc;
  if (n < 0) return fail(PGSAG_EINVAL, "n < 0");
  if (n > 0 && (rc = check_proj(p))) return rc;
  if (!bins || !bins->ranges || (bins->capacity > 0 && (!bins->tile_keys || !bins->vals)))
    return fail(PGSAG_EINVAL, "bins buffer is NULL");
  if (!aligned(bins->tile_keys, 16) || !aligned(bins->vals, 16))
    return fail(PGSAG_EINVAL, "bins tile_keys / vals must be 16-byte aligned");
  if (bins->capacity < 0 || bins->capacity >= (int64_t)kLbMask)
    return fail(PGSAG_EINVAL, "bins capacity must be in [0, 2^30)");
  const WsLayout L = ws_layout(n, cam->width, cam->height, bins->capacity);
  if ((rc = check_ws(ws, ws_bytes, L.total))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims d = make_dims(cam->width, cam->height);
  char* w = static_cast<char*>(ws);
  uint32_t* counters = reinterpret_cast<uint32_t*>(w + L.counters);
  cudaError_t e = cudaMemsetAsync(w + L.counters, 0, L.zero_end - L.counters, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  const uint32_t* ids_sorted = nullptr;
  if (n > 0) {
    e = launch_bin_sort_stage1(p, n, L, w, st, &ids_sorted);
    if (e != cudaSuccess) return cuda_fail(e, "depth sort / scan");
  }
  bins->n_dup = -1;  // unknown on the host until the stream reaches the copy below
  e = launch_duplicate_and_sort(p, tm, d, n, 0u, false, ids_sorted, L, w, bins, st);
  if (e != cudaSuccess) return cuda_fail(e, "duplicate / tile sort / ranges");
  if (m_out) {
    e = cudaMemcpyAsync(m_out, counters + CNT_M, sizeof(unsigned long long), cudaMemcpyDefault, st);
    if (e != cudaSuccess) return cuda_fail(e, "M copy");
  }
  return PGSAG_OK;
}

int pgsag_render_fwd(const pgsag_projected* p, const pgsag_bins* bins, const pgsag_tilemask* tm,
                     const pgsag_camera* cam, const uint8_t* mask, const float bg[3], pgsag_image* out, void* ws,
                     size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_cam(cam)) || (rc = check_tm(tm)) || (rc = check_proj(p))) return rc;
  if (!bins || !bins->vals || !bins->ranges) return fail(PGSAG_EINVAL, "bins buffer is NULL");
  if (!mask || !bg) return fail(PGSAG_EINVAL, "mask/bg is NULL");
  if (!out || !out->C || !out->N || !out->D || !out->A || !out->Dep || !out->T || !out->g || !out->last)
    return fail(PGSAG_EINVAL, "image buffer is NULL");
  const WsLayout L = ws_layout(0, cam->width, cam->height, 0);
  if ((rc = check_ws(ws, ws_bytes, L.total))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims d = make_dims(cam->width, cam->height);
  uint32_t* counters = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + L.counters);
  cudaError_t e = cudaMemsetAsync(counters + CNT_FWD, 0, sizeof(uint32_t), st);
  if (e == cudaSuccess) e = launch_render_fwd(p, bins, tm, d, cam, mask, bg, out, counters + CNT_FWD, st);
  if (e != cudaSuccess) return cuda_fail(e, "render_fwd");
  return PGSAG_OK;
}

int pgsag_render_bwd(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                     const pgsag_bins* bins, const pgsag_tilemask* tm, const uint8_t* mask, const float bg[3],
                     const pgsag_image* fwd, const pgsag_image_grad* dL, pgsag_gaussian_grad* out, void* ws,
                     size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_g(g)) || (rc = check_cam(cam)) || (rc = check_tm(tm))) return rc;
  if (g->n > 0 && (rc = check_proj(p))) return rc;
  if (!bins || !bins->vals || !bins->ranges) return fail(PGSAG_EINVAL, "bins buffer is NULL");
  if (!mask || !bg || !fwd || !dL || !out) return fail(PGSAG_EINVAL, "argument is NULL");
  if (!fwd->N || !fwd->D || !fwd->T || !fwd->g || !fwd->last) return fail(PGSAG_EINVAL, "fwd image is NULL");
  if (g->n > 0 && (!out->dmean || !out->dscale || !out->drot || !out->dopacity || !out->dsh))
    return fail(PGSAG_EINVAL, "gradient output is NULL");
  const WsLayout L = ws_layout(g->n, cam->width, cam->height, 0);
  if ((rc = check_ws(ws, ws_bytes, L.total))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims d = make_dims(cam->width, cam->height);
  char* w = static_cast<char*>(ws);
  uint32_t* counters = reinterpret_cast<uint32_t*>(w + L.counters);
  cudaError_t e = cudaMemsetAsync(counters + CNT_BWD, 0, sizeof(uint32_t), st);
  if (e == cudaSuccess)
    e = launch_render_bwd(g, cam, p, bins, tm, d, mask, bg, fwd, dL, out, reinterpret_cast<float*>(w + L.g2d),
                          counters + CNT_BWD, st);
  if (e != cudaSuccess) return cuda_fail(e, "render_bwd");
  return PGSAG_OK;
}

static int check_state(const pgsag_adam_state* s);

int pgsag_render_bwd_adam(const pgsag_gaussians* g, const pgsag_camera* cam, const pgsag_projected* p,
                          const pgsag_bins* bins, const pgsag_tilemask* tm, const uint8_t* mask, const float bg[3],
                          const pgsag_image* fwd, const pgsag_image_grad* dL, pgsag_gaussian_grad* out,
                          pgsag_adam_state* state, const pgsag_adam_hparams* hp, double* flatten_loss, void* ws,
                          size_t ws_bytes, void* stream) {
  int rc;
  if ((rc = check_g(g)) || (rc = check_cam(cam)) || (rc = check_tm(tm))) return rc;
  if (g->n > 0 && (rc = check_proj(p))) return rc;
  if (!bins || !bins->vals || !bins->ranges) return fail(PGSAG_EINVAL, "bins buffer is NULL");
  if (!mask || !bg || !fwd || !dL || !out || !state || !hp) return fail(PGSAG_EINVAL, "argument is NULL");
  if (!fwd->N || !fwd->D || !fwd->T || !fwd->g || !fwd->last) return fail(PGSAG_EINVAL, "fwd image is NULL");
  if (hp->step < 1) return fail(PGSAG_EINVAL, "adam: step must be >= 1");
  if (g->n > 0 && (rc = check_state(state))) return rc;
  if (g->n > 0 && (state->mean != g->mean || state->scale != g->scale || state->rot != g->rot ||
                   state->opacity != g->opacity || state->sh != g->sh))
    return fail(PGSAG_EINVAL, "render_bwd_adam: state does not hold g's parameter arrays");
  const WsLayout L = ws_layout(g->n, cam->width, cam->height, 0);
  if ((rc = check_ws(ws, ws_bytes, L.total))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Dims d = make_dims(cam->width, cam->height);
  char* w = static_cast<char*>(ws);
  uint32_t* counters = reinterpret_cast<uint32_t*>(w + L.counters);
  cudaError_t e = cudaMemsetAsync(counters + CNT_BWD, 0, sizeof(uint32_t), st);
  if (e == cudaSuccess)
    e = launch_render_bwd(g, cam, p, bins, tm, d, mask, bg, fwd, dL, out, reinterpret_cast<float*>(w + L.g2d),
                          counters + CNT_BWD, st, state, hp, flatten_loss, counters + CNT_OVF);
  if (e != cudaSuccess) return cuda_fail(e, "render_bwd_adam");
  return PGSAG_OK;
}

int pgsag_gc_weights(const float* image, const uint8_t* mask, int32_t width, int32_t height, float* w, void* ws,
                     size_t ws_bytes, void* stream) {
  if (!image || !mask || !w) return fail(PGSAG_EINVAL, "gc_weights: NULL argument");
  if (width <= 0 || height <= 0) return fail(PGSAG_EINVAL, "width/height must be > 0");
  const WsLayout L = ws_layout(0, width, height, 0);
  int rc;
  if ((rc = check_ws(ws, ws_bytes, L.total))) return rc;
  double* acc = reinterpret_cast<double*>(static_cast<char*>(ws) + L.counters + 4 * CNT_GC);
  cudaError_t e = launch_gc_weights(image, mask, width, height, w, acc, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "gc_weights");
  return PGSAG_OK;
}

int pgsag_boundary_band(const uint8_t* mask, int32_t width, int32_t height, int32_t r, uint8_t* band, void* stream) {
  if (!mask || !band) return fail(PGSAG_EINVAL, "boundary_band: NULL argument");
  if (width <= 0 || height <= 0 || r < 1) return fail(PGSAG_EINVAL, "boundary_band: bad size or radius");
  cudaError_t e = launch_boundary_band(mask, width, height, r, band, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "boundary_band");
  return PGSAG_OK;
}

int pgsag_ban_loss(const pgsag_camera* cam, const uint8_t* mask, const uint8_t* band, const float* N,
                   const float* Dep, float boundary_w, float lambda, int32_t mean, double* loss, float* dN,
                   float* dDep, void* stream) {
  int rc;
  if ((rc = check_cam(cam))) return rc;
  if (!mask || !band || !N || !Dep || !loss) return fail(PGSAG_EINVAL, "ban_loss: NULL argument");
  cudaError_t e = launch_ban_loss(cam, mask, band, N, Dep, boundary_w, lambda, mean, loss, dN, dDep,
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "ban_loss");
  return PGSAG_OK;
}

size_t pgsag_rgb_loss_workspace_size(int32_t width, int32_t height) {
  if (width <= 0 || height <= 0) return 0;
  return (size_t)36 * (size_t)width * (size_t)height;
}

int pgsag_rgb_loss(const float* image, const float* target, const uint8_t* mask, int32_t width, int32_t height,
                   float weight, double* loss, float* dC, void* ws, size_t ws_bytes, void* stream) {
  if (!image || !target || !mask || !loss) return fail(PGSAG_EINVAL, "rgb_loss: NULL argument");
  if (width <= 0 || height <= 0) return fail(PGSAG_EINVAL, "width/height must be > 0");
  int rc;
  if ((rc = check_ws(ws, ws_bytes, pgsag_rgb_loss_workspace_size(width, height)))) return rc;
  cudaError_t e = launch_rgb_loss(image, target, mask, width, height, weight, loss, dC, static_cast<float*>(ws),
                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "rgb_loss");
  return PGSAG_OK;
}

int pgsag_adam_step(int32_t n, int32_t sh_degree, const pgsag_gaussian_grad* grad, pgsag_adam_state* state,
                    const pgsag_adam_hparams* hp, double* flatten_loss, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3) return fail(PGSAG_EINVAL, "adam: bad n / sh_degree");
  if (!grad || !state || !hp) return fail(PGSAG_EINVAL, "adam: NULL argument");
  if (hp->step < 1) return fail(PGSAG_EINVAL, "adam: step must be >= 1");
  if (n > 0 && (!grad->dmean || !grad->dscale || !grad->drot || !grad->dopacity || !grad->dsh || !state->mean ||
                !state->scale || !state->rot || !state->opacity || !state->sh || !state->log_scale ||
                !state->logit_opacity || !state->m || !state->v))
    return fail(PGSAG_EINVAL, "adam: NULL buffer");
  cudaError_t e = launch_adam(n, sh_degree, grad, state, hp, flatten_loss, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "adam");
  return PGSAG_OK;
}

int pgsag_adam_init(int32_t n, pgsag_adam_state* state, void* stream) {
  if (n < 0 || !state) return fail(PGSAG_EINVAL, "adam_init: bad argument");
  if (n > 0 && (!state->scale || !state->opacity || !state->log_scale || !state->logit_opacity))
    return fail(PGSAG_EINVAL, "adam_init: NULL buffer");
  cudaError_t e = launch_adam_init(n, state, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "adam_init");
  return PGSAG_OK;
}

int pgsag_loss_total(const double* rgb_loss, const double* flatten_loss, const double* ban_loss, int32_t ban_mean,
                     const double* gc_stats, float lambda, float lambda3, float lambda4, double* total, void* stream) {
  if (!rgb_loss || !total) return fail(PGSAG_EINVAL, "loss_total: NULL argument");
  cudaError_t e = launch_loss_total(rgb_loss, flatten_loss, ban_loss, gc_stats, lambda, lambda3, lambda4, ban_mean,
                                    total, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "loss_total");
  return PGSAG_OK;
}

size_t pgsag_densify_workspace_size(int32_t n) { return n < 0 ? 0 : densify_ws_bytes(n); }

static int check_state(const pgsag_adam_state* s) {
  if (!s || !s->mean || !s->scale || !s->rot || !s->opacity || !s->sh || !s->log_scale || !s->logit_opacity || !s->m ||
      !s->v)
    return fail(PGSAG_EINVAL, "adam state: NULL buffer");
  return PGSAG_OK;
}

int pgsag_densify_plan(int32_t n, const float* scale, const float* opacity, const float* accum, const float* count,
                       const pgsag_densify_params* dp, uint8_t* action, int64_t counts[3], void* ws, size_t ws_bytes,
                       void* stream) {
  if (n < 0 || !dp || !counts) return fail(PGSAG_EINVAL, "densify_plan: bad argument");
  if (n > 0 && (!scale || !opacity || !accum || !count || !action)) return fail(PGSAG_EINVAL, "densify_plan: NULL");
  int rc;
  if ((rc = check_ws(ws, ws_bytes, densify_ws_bytes(n)))) return rc;
  unsigned long long tot[3] = {0, 0, 0};
  cudaError_t e = launch_densify_plan(n, scale, opacity, accum, count, dp, action, ws,
                                      static_cast<cudaStream_t>(stream), tot);
  if (e != cudaSuccess) return cuda_fail(e, "densify_plan");
  for (int k = 0; k < 3; ++k) counts[k] = (int64_t)tot[k];
  return PGSAG_OK;
}

int pgsag_densify_apply(int32_t n, int32_t sh_degree, const pgsag_adam_state* src, const uint8_t* action,
                        const pgsag_densify_params* dp, const int64_t counts[3], pgsag_adam_state* dst,
                        const void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || sh_degree < 0 || sh_degree > 3 || !dp || !counts || !dst) return fail(PGSAG_EINVAL, "densify_apply");
  const int64_t n_out = counts[0] + counts[1] + 2 * counts[2];
  if (counts[0] < 0 || counts[1] < 0 || counts[2] < 0 || counts[0] > n || counts[1] > counts[0] || n_out > INT32_MAX)
    return fail(PGSAG_EINVAL, "densify_apply: counts inconsistent with n");
  int rc;
  if (n > 0 && ((rc = check_state(src)) || !action)) return rc ? rc : fail(PGSAG_EINVAL, "densify_apply: NULL");
  if (n_out > 0 && (rc = check_state(dst))) return rc;
  if ((rc = check_ws(const_cast<void*>(ws), ws_bytes, densify_ws_bytes(n)))) return rc;
  cudaError_t e = launch_densify_apply(n, sh_degree, src, action, dp, dst, (int)n_out, (uint32_t)counts[0],
                                       (uint32_t)counts[1], ws, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "densify_apply");
  return PGSAG_OK;
}

int pgsag_opacity_reset(int32_t n, pgsag_adam_state* state, float cap, void* stream) {
  if (n < 0 || !(cap > 0.f && cap < 1.f)) return fail(PGSAG_EINVAL, "opacity_reset: bad n / cap");
  int rc;
  if (n > 0 && (rc = check_state(state))) return rc;
  cudaError_t e = launch_opacity_reset(n, state, cap, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "opacity_reset");
  return PGSAG_OK;
}

int pgsag_microbench_fp32(int32_t mode, int32_t iters, float* scratch, double* tflops, void* stream) {
  if ((mode != 0 && mode != 1) || iters <= 0 || !scratch || !tflops) return fail(PGSAG_EINVAL, "microbench: bad argument");
  float ms = 0.f;
  double flops = 0.0;
  cudaError_t e = launch_fp32_microbench(mode, iters, scratch, &ms, &flops, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "microbench");
  *tflops = flops / ((double)ms * 1e-3) / 1e12;
  return PGSAG_OK;
}

int pgsag_unpack_rgb8(const uint8_t* rgb8, int32_t width, int32_t height, float* image, void* stream) {
  if (!rgb8 || !image) return fail(PGSAG_EINVAL, "unpack_rgb8: NULL argument");
  if (width <= 0 || height <= 0) return fail(PGSAG_EINVAL, "width/height must be > 0");
  if (!aligned(rgb8, 4) || !aligned(image, 16) || (((size_t)width * height) % 4) != 0)
    return fail(PGSAG_EINVAL, "unpack_rgb8: rgb8 4-byte and image 16-byte aligned, W*H a multiple of 4");
  cudaError_t e = launch_unpack_rgb8(rgb8, width, height, image, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "unpack_rgb8");
  return PGSAG_OK;
}

}  // extern "C"
