"""ctypes binding of libpgsag.so (include/pgsag.h).  Argument marshalling only:
every step of the rasterizer runs in the library's sm_100a kernels.  There is no
CPU fallback: importing a function whose library is missing raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpgsag.so")

PGSAG_OK, PGSAG_EINVAL, PGSAG_ECAPACITY, PGSAG_ECUDA, PGSAG_ENONFINITE, PGSAG_EWORKSPACE = 0, -1, -2, -3, -4, -5
F_VISIBLE, F_DET_OK, F_OPAC_OK, F_RECT, F_LIVE = 1, 2, 4, 8, 15

SYMBOLS = ("pgsag_workspace_size", "pgsag_preprocess", "pgsag_bin_sort", "pgsag_bin_sort_async", "pgsag_render_fwd",
           "pgsag_render_bwd", "pgsag_last_error", "pgsag_version", "pgsag_timing_enable", "pgsag_timing_filter",
           "pgsag_timing_collect", "pgsag_timing_get", "pgsag_gc_weights", "pgsag_boundary_band",
           "pgsag_ban_loss", "pgsag_rgb_loss_workspace_size", "pgsag_rgb_loss", "pgsag_adam_step",
           "pgsag_densify_workspace_size", "pgsag_densify_plan", "pgsag_densify_apply", "pgsag_opacity_reset",
           "pgsag_microbench_fp32", "pgsag_unpack_rgb8", "pgsag_render_bwd_adam", "pgsag_set_checks",
           "pgsag_adam_init", "pgsag_loss_total")

_vp = C.c_void_p


class Camera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32), ("R", C.c_float * 9), ("C", C.c_float * 3),
                ("znear", C.c_float)]


class Gaussians(C.Structure):
    _fields_ = [("n", C.c_int32), ("sh_degree", C.c_int32), ("mean", _vp), ("scale", _vp), ("rot", _vp),
                ("opacity", _vp), ("sh", _vp)]


class Projected(C.Structure):
    _fields_ = [("mean2d", _vp), ("conic_o", _vp), ("depth", _vp), ("rect", _vp), ("tiles_touched", _vp),
                ("rgb_d", _vp), ("ncam", _vp), ("flags", _vp)]


class TileMask(C.Structure):
    _fields_ = [("tile_cnt", _vp), ("sat", _vp), ("active", _vp), ("n_active", _vp), ("active_bits", _vp)]


class Bins(C.Structure):
    _fields_ = [("tile_keys", _vp), ("vals", _vp), ("ranges", _vp), ("capacity", C.c_int64),
                ("n_dup", C.c_int64), ("order", _vp)]


class Image(C.Structure):
    _fields_ = [("C", _vp), ("N", _vp), ("D", _vp), ("A", _vp), ("Dep", _vp), ("T", _vp), ("g", _vp),
                ("last", _vp), ("counters", _vp), ("gc_w", _vp), ("gc_stats", _vp)]


class ImageGrad(C.Structure):
    _fields_ = [("dC", _vp), ("dN", _vp), ("dD", _vp), ("dA", _vp), ("dDep", _vp), ("gc_lambda", C.c_float),
                ("nd_div", _vp)]


class GaussianGrad(C.Structure):
    _fields_ = [("dmean", _vp), ("dscale", _vp), ("drot", _vp), ("dopacity", _vp), ("dsh", _vp),
                ("absgrad2d", _vp), ("grad2d", _vp), ("densify_accum", _vp), ("densify_count", _vp)]


class DensifyParams(C.Structure):
    _fields_ = [("grad_threshold", C.c_float), ("dense_limit", C.c_float), ("min_opacity", C.c_float),
                ("seed", C.c_uint64)]


class AdamState(C.Structure):
    _fields_ = [("mean", _vp), ("scale", _vp), ("rot", _vp), ("opacity", _vp), ("sh", _vp), ("log_scale", _vp),
                ("logit_opacity", _vp), ("m", _vp), ("v", _vp)]


class AdamHparams(C.Structure):
    _fields_ = [("lr_mean", C.c_float), ("lr_scale", C.c_float), ("lr_rot", C.c_float), ("lr_opacity", C.c_float),
                ("lr_sh_dc", C.c_float), ("lr_sh_rest", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float),
                ("eps", C.c_float), ("flatten_weight", C.c_float), ("step", C.c_int32)]


_lib = None
_lock = threading.Lock()


class PgsagError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"pgsag error {code}: {msg}")
        self.code = code


def lib():
    """Load libpgsag.so (fails loudly if it was not built: no fallback path exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = C.CDLL(LIB_PATH)
            P = C.POINTER
            L.pgsag_workspace_size.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int64]
            L.pgsag_workspace_size.restype = C.c_size_t
            L.pgsag_preprocess.argtypes = [P(Gaussians), P(Camera), _vp, P(TileMask), P(Projected), _vp,
                                           C.c_size_t, _vp]
            L.pgsag_bin_sort.argtypes = [P(Projected), P(TileMask), P(Camera), C.c_int32, P(Bins), _vp,
                                         C.c_size_t, _vp]
            L.pgsag_render_fwd.argtypes = [P(Projected), P(Bins), P(TileMask), P(Camera), _vp,
                                           P(C.c_float * 3), P(Image), _vp, C.c_size_t, _vp]
            L.pgsag_render_bwd.argtypes = [P(Gaussians), P(Camera), P(Projected), P(Bins), P(TileMask), _vp,
                                           P(C.c_float * 3), P(Image), P(ImageGrad), P(GaussianGrad), _vp,
                                           C.c_size_t, _vp]
            L.pgsag_bin_sort_async.argtypes = [P(Projected), P(TileMask), P(Camera), C.c_int32, P(Bins), _vp, _vp,
                                               C.c_size_t, _vp]
            for nm in ("pgsag_preprocess", "pgsag_bin_sort", "pgsag_bin_sort_async", "pgsag_render_fwd",
                       "pgsag_render_bwd"):
                getattr(L, nm).restype = C.c_int
            L.pgsag_last_error.restype = C.c_char_p
            L.pgsag_version.restype = C.c_char_p
            L.pgsag_timing_enable.argtypes = [C.c_int]
            L.pgsag_timing_enable.restype = None
            L.pgsag_timing_filter.argtypes = [C.c_char_p]
            L.pgsag_timing_filter.restype = None
            L.pgsag_timing_collect.argtypes = []
            L.pgsag_timing_collect.restype = C.c_int
            L.pgsag_timing_get.argtypes = [C.c_int, P(C.c_char_p), P(C.c_double), P(C.c_longlong)]
            L.pgsag_timing_get.restype = C.c_int
            L.pgsag_gc_weights.argtypes = [_vp, _vp, C.c_int32, C.c_int32, _vp, _vp, C.c_size_t, _vp]
            L.pgsag_gc_weights.restype = C.c_int
            L.pgsag_boundary_band.argtypes = [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, _vp]
            L.pgsag_boundary_band.restype = C.c_int
            L.pgsag_ban_loss.argtypes = [P(Camera), _vp, _vp, _vp, _vp, C.c_float, C.c_float, C.c_int32, _vp,
                                         _vp, _vp, _vp]
            L.pgsag_ban_loss.restype = C.c_int
            L.pgsag_rgb_loss_workspace_size.argtypes = [C.c_int32, C.c_int32]
            L.pgsag_rgb_loss_workspace_size.restype = C.c_size_t
            L.pgsag_rgb_loss.argtypes = [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_float, _vp, _vp, _vp, C.c_size_t,
                                         _vp]
            L.pgsag_rgb_loss.restype = C.c_int
            L.pgsag_adam_step.argtypes = [C.c_int32, C.c_int32, P(GaussianGrad), P(AdamState), P(AdamHparams), _vp,
                                          _vp]
            L.pgsag_adam_step.restype = C.c_int
            L.pgsag_render_bwd_adam.argtypes = [P(Gaussians), P(Camera), P(Projected), P(Bins), P(TileMask), _vp,
                                                P(C.c_float * 3), P(Image), P(ImageGrad), P(GaussianGrad),
                                                P(AdamState), P(AdamHparams), _vp, _vp, C.c_size_t, _vp]
            L.pgsag_render_bwd_adam.restype = C.c_int
            L.pgsag_densify_workspace_size.argtypes = [C.c_int32]
            L.pgsag_densify_workspace_size.restype = C.c_size_t
            L.pgsag_densify_plan.argtypes = [C.c_int32, _vp, _vp, _vp, _vp, P(DensifyParams), _vp, P(C.c_int64 * 3),
                                             _vp, C.c_size_t, _vp]
            L.pgsag_densify_plan.restype = C.c_int
            L.pgsag_densify_apply.argtypes = [C.c_int32, C.c_int32, P(AdamState), _vp, P(DensifyParams),
                                              P(C.c_int64 * 3), P(AdamState), _vp, C.c_size_t, _vp]
            L.pgsag_densify_apply.restype = C.c_int
            L.pgsag_opacity_reset.argtypes = [C.c_int32, P(AdamState), C.c_float, _vp]
            L.pgsag_opacity_reset.restype = C.c_int
            L.pgsag_microbench_fp32.argtypes = [C.c_int32, C.c_int32, _vp, P(C.c_double), _vp]
            L.pgsag_microbench_fp32.restype = C.c_int
            L.pgsag_unpack_rgb8.argtypes = [_vp, C.c_int32, C.c_int32, _vp, _vp]
            L.pgsag_unpack_rgb8.restype = C.c_int
            L.pgsag_set_checks.argtypes = [C.c_int]
            L.pgsag_set_checks.restype = None
            L.pgsag_adam_init.argtypes = [C.c_int32, P(AdamState), _vp]
            L.pgsag_adam_init.restype = C.c_int
            L.pgsag_loss_total.argtypes = [_vp, _vp, _vp, C.c_int32, _vp, C.c_float, C.c_float, C.c_float, _vp, _vp]
            L.pgsag_loss_total.restype = C.c_int
            _lib = L
    return _lib


def timing_enable(on=True):
    lib().pgsag_timing_enable(1 if on else 0)


def timing_filter(prefix=None):
    lib().pgsag_timing_filter(prefix.encode() if prefix else None)


def timing_collect():
    """{kernel name: (total ms, launches)} since the last collect (synchronises on the events)."""
    L = lib()
    k = L.pgsag_timing_collect()
    out = {}
    for i in range(k):
        nm, ms, cnt = C.c_char_p(), C.c_double(), C.c_longlong()
        check(L.pgsag_timing_get(i, C.byref(nm), C.byref(ms), C.byref(cnt)))
        out[nm.value.decode()] = (ms.value, cnt.value)
    return out


def check(rc):
    if rc != PGSAG_OK:
        raise PgsagError(rc, lib().pgsag_last_error().decode())
    return rc


def ptr(t):
    """Device (or host) address of a tensor / None."""
    return None if t is None else C.c_void_p(t.data_ptr())


def workspace_size(n, W, H, cap):
    return int(lib().pgsag_workspace_size(int(n), int(W), int(H), int(cap)))


def preprocess(g, cam, mask, tm, proj, ws, ws_bytes, stream):
    return check(lib().pgsag_preprocess(C.byref(g), C.byref(cam), mask, C.byref(tm), C.byref(proj), ws,
                                        ws_bytes, stream))


def bin_sort_async(proj, tm, cam, n, bins, m_out, ws, ws_bytes, stream):
    return check(lib().pgsag_bin_sort_async(C.byref(proj), C.byref(tm), C.byref(cam), int(n), C.byref(bins), m_out,
                                            ws, ws_bytes, stream))


def bin_sort(proj, tm, cam, n, bins, ws, ws_bytes, stream):
    """Returns the status code (PGSAG_ECAPACITY is returned, not raised; bins.n_dup then holds M)."""
    rc = lib().pgsag_bin_sort(C.byref(proj), C.byref(tm), C.byref(cam), int(n), C.byref(bins), ws, ws_bytes,
                              stream)
    if rc not in (PGSAG_OK, PGSAG_ECAPACITY):
        check(rc)
    return rc


def render_fwd(proj, bins, tm, cam, mask, bg, img, ws, ws_bytes, stream):
    return check(lib().pgsag_render_fwd(C.byref(proj), C.byref(bins), C.byref(tm), C.byref(cam), mask,
                                        C.byref(bg), C.byref(img), ws, ws_bytes, stream))


def render_bwd(g, cam, proj, bins, tm, mask, bg, img, dimg, grad, ws, ws_bytes, stream):
    return check(lib().pgsag_render_bwd(C.byref(g), C.byref(cam), C.byref(proj), C.byref(bins), C.byref(tm),
                                        mask, C.byref(bg), C.byref(img), C.byref(dimg), C.byref(grad), ws,
                                        ws_bytes, stream))


def gc_weights(image, mask, W, H, w, ws, ws_bytes, stream):
    return check(lib().pgsag_gc_weights(image, mask, int(W), int(H), w, ws, ws_bytes, stream))


def boundary_band(mask, W, H, r, band, stream):
    return check(lib().pgsag_boundary_band(mask, int(W), int(H), int(r), band, stream))


def ban_loss(cam, mask, band, N, Dep, bw, lam, mean, loss, dN, dDep, stream):
    return check(lib().pgsag_ban_loss(C.byref(cam), mask, band, N, Dep, float(bw), float(lam), int(mean), loss, dN,
                                      dDep, stream))


def version():
    return lib().pgsag_version().decode()


def rgb_loss_workspace_size(W, H):
    return int(lib().pgsag_rgb_loss_workspace_size(int(W), int(H)))


def rgb_loss(image, target, mask, W, H, weight, loss, dC, ws, ws_bytes, stream):
    return check(lib().pgsag_rgb_loss(image, target, mask, int(W), int(H), float(weight), loss, dC, ws, int(ws_bytes),
                                      stream))


def render_bwd_adam(g, cam, proj, bins, tm, mask, bg, img, dimg, grad, state, hp, flat, ws, ws_bytes, stream):
    return check(lib().pgsag_render_bwd_adam(C.byref(g), C.byref(cam), C.byref(proj), C.byref(bins), C.byref(tm),
                                             mask, C.byref(bg), C.byref(img), C.byref(dimg), C.byref(grad),
                                             C.byref(state), C.byref(hp), flat, ws, ws_bytes, stream))


def adam_step(n, deg, grad, state, hp, flat, stream):
    return check(lib().pgsag_adam_step(int(n), int(deg), C.byref(grad), C.byref(state), C.byref(hp), flat, stream))


def densify_workspace_size(n):
    return int(lib().pgsag_densify_workspace_size(int(n)))


def densify_plan(n, scale, opacity, accum, count, dp, action, ws, ws_bytes, stream):
    counts = (C.c_int64 * 3)()
    check(lib().pgsag_densify_plan(int(n), scale, opacity, accum, count, C.byref(dp), action, C.byref(counts), ws,
                                   int(ws_bytes), stream))
    return [int(c) for c in counts]


def densify_apply(n, deg, src, action, dp, counts, dst, ws, ws_bytes, stream):
    cc = (C.c_int64 * 3)(*counts)
    return check(lib().pgsag_densify_apply(int(n), int(deg), C.byref(src), action, C.byref(dp), C.byref(cc),
                                           C.byref(dst), ws, int(ws_bytes), stream))


def opacity_reset(n, state, cap, stream):
    return check(lib().pgsag_opacity_reset(int(n), C.byref(state), float(cap), stream))


def microbench_fp32(mode, iters, scratch, stream):
    out = C.c_double(0.0)
    check(lib().pgsag_microbench_fp32(int(mode), int(iters), scratch, C.byref(out), stream))
    return out.value


def unpack_rgb8(rgb8, W, H, image, stream):
    return check(lib().pgsag_unpack_rgb8(rgb8, int(W), int(H), image, stream))


def set_checks(level):
    lib().pgsag_set_checks(int(level))


def adam_init(n, state, stream):
    return check(lib().pgsag_adam_init(int(n), C.byref(state), stream))


def loss_total(rgb, flat, ban, ban_mean, gc_stats, lam, lam3, lam4, total, stream):
    return check(lib().pgsag_loss_total(rgb, flat, ban, int(ban_mean), gc_stats, float(lam), float(lam3), float(lam4),
                                        total, stream))
