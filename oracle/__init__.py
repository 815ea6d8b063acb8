"""CPU oracle for the PG-SAG masked rasterizer — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2501_01677_b200) never imports it and shares no code with it.

This module is argument marshalling for oracle/oracle.cpp (a plain,
single-threaded C++ renderer written from PAPER.md §3.1 Eq. 1-4; see the
header of that file and DESIGN.md §3 for the readings).  The library is
compiled on demand with g++ -O2 -ffp-contract=off -fno-fast-math.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

N_GRAD_ROWS = 73  # dmean 3, dscale 3, drot 4, dopac 1, dsh 48 | 2D grads 13 + absgrad (59..72)

F_VISIBLE, F_DET_OK, F_OPAC_OK, F_RECT = 1, 2, 4, 8
F_LIVE = 15


def build(force: bool = False) -> str:
    """Compile liboracle.so (no -march=native: plain IEEE double/float)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               _SRC, "-o", _SO + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            P = C.c_void_p
            i32, i64 = C.c_int, C.c_int64
            L.oracle_tilemask.argtypes = [P, i32, i32, P, P]
            L.oracle_tilemask.restype = None
            for nm in ("oracle_project_f32", "oracle_project_f64"):
                getattr(L, nm).argtypes = [P, P, P, P, P, i32, i32, P, i32, i32, P, P, P, P, P, P, P, P, P, P]
                getattr(L, nm).restype = None
            L.oracle_keys.argtypes = [P, P, P, i32, P, i32, i32, i64, P, P, P]
            L.oracle_keys.restype = i64
            for nm in ("oracle_render_f32", "oracle_render_f64", "oracle_render_f64_fproj"):
                getattr(L, nm).argtypes = [P, P, P, P, P, i32, i32, P, i32, i32, P, P, P, i32, P, P, P, P,
                                           P, i32, P, P, P, P]
                getattr(L, nm).restype = None
            L.oracle_gc_weights.argtypes = [P, P, i32, i32, P]
            L.oracle_gc_weights.restype = None
            L.oracle_gc_load.argtypes = [P, P, i32, P, P]
            L.oracle_gc_load.restype = C.c_double
            L.oracle_boundary_band.argtypes = [P, i32, i32, i32, P]
            L.oracle_boundary_band.restype = None
            L.oracle_ban_loss.argtypes = [P, i32, i32, P, P, P, P, C.c_double, C.c_double, P, P, P]
            L.oracle_ban_loss.restype = None
            L.oracle_rgb_loss.argtypes = [P, P, P, i32, i32, P, P]
            L.oracle_rgb_loss.restype = None
            L.oracle_set_bound_eval.argtypes = [i32]
            L.oracle_set_bound_eval.restype = None
            L.oracle_sh_basis.argtypes = [C.c_double, C.c_double, C.c_double, P]
            L.oracle_sh_basis.restype = None
            L.oracle_lnup_f32.argtypes = [C.c_float]
            L.oracle_lnup_f32.restype = C.c_float
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def cam_array(cam) -> np.ndarray:
    """[fx, fy, cx, cy, R(9), C(3), znear] as float64 (values are the float32 ones)."""
    f32 = lambda v: float(np.float32(v))
    vals = [f32(cam.fx), f32(cam.fy), f32(cam.cx), f32(cam.cy)]
    vals += [float(v) for v in np.asarray(cam.R, np.float32).reshape(-1)]
    vals += [float(v) for v in np.asarray(cam.C, np.float32).reshape(-1)]
    vals += [f32(cam.znear)]
    return np.array(vals, np.float64)


def _params(g, dtype):
    a = [np.ascontiguousarray(np.asarray(x), dtype) for x in (g.mean, g.scale, g.rot, g.opacity, g.sh)]
    return a


def tilemask(mask: np.ndarray):
    H, W = mask.shape
    TX, TY = (W + 15) // 16, (H + 15) // 16
    cnt = np.zeros(TY * TX, np.uint32)
    sat = np.zeros((TY + 1) * (TX + 1), np.int32)
    m = np.ascontiguousarray(mask, np.uint8)
    lib().oracle_tilemask(_p(m), W, H, _p(cnt), _p(sat))
    return cnt.reshape(TY, TX), sat.reshape(TY + 1, TX + 1)


def project(g, cam, mask, dtype=np.float32):
    """O2 for every Gaussian.  Returns dict of numpy arrays (AoS-interleaved as documented)."""
    n = int(np.asarray(g.opacity).shape[0])
    prm = _params(g, dtype)
    m = np.ascontiguousarray(mask, np.uint8)
    out = dict(mean2d=np.zeros((n, 2), dtype), conic_o=np.zeros((n, 4), dtype), depth=np.zeros(n, dtype),
               rect=np.zeros((n, 4), np.int32), tiles=np.zeros(n, np.uint32), rgb=np.zeros((n, 3), dtype),
               ncam=np.zeros((n, 3), dtype), dist=np.zeros(n, dtype), flags=np.zeros(n, np.uint32))
    fn = lib().oracle_project_f32 if dtype == np.float32 else lib().oracle_project_f64
    ca = cam_array(cam)
    fn(*[_p(a) for a in prm], n, int(g.sh_degree), _p(ca), int(cam.width), int(cam.height), _p(m),
       *[_p(out[k]) for k in ("mean2d", "conic_o", "depth", "rect", "tiles", "rgb", "ncam", "dist", "flags")])
    return out


def keys(proj, mask):
    """O3: sorted tile ids, Gaussian ids and ranges [TY*TX][2]."""
    H, W = mask.shape
    n = proj["depth"].shape[0]
    TX, TY = (W + 15) // 16, (H + 15) // 16
    depth = np.ascontiguousarray(proj["depth"], np.float32)
    rect = np.ascontiguousarray(proj["rect"], np.int32)
    flags = np.ascontiguousarray(proj["flags"], np.uint32)
    m = np.ascontiguousarray(mask, np.uint8)
    ranges = np.zeros((TY * TX, 2), np.uint32)
    M = lib().oracle_keys(_p(depth), _p(rect), _p(flags), n, _p(m), W, H, 0, None, None, _p(ranges))
    tiles = np.zeros(M, np.uint32)
    vals = np.zeros(M, np.uint32)
    M2 = lib().oracle_keys(_p(depth), _p(rect), _p(flags), n, _p(m), W, H, M, _p(tiles), _p(vals), _p(ranges))
    assert M2 == M
    return tiles, vals, ranges


def render(g, cam, mask, pixels, bg=(0.0, 0.0, 0.0), dtype=np.float32, certify=False, upstream=None,
           bound=False, fproj=False):
    """O4 (and O5/O6 if upstream is given) for the listed flat pixel indices.

    upstream: (npix, 9) or (npix, 10) float64 = gC(3), gN(3), gD, gA, gDep[, gG] per listed pixel,
    gG = dL/d(soft count) of the L_GC-load surrogate (R24).
    certify: True/1 counts pairs outside the tile rect with alpha >= 1/255 (R8, must be 0); an
    integer 1 + s first shrinks every rect by s tiles per side (the certificate's negative control).
    bound: also return the R19b + R19c float32 accumulation / evaluation bound on rows 0..58
    ("acc": the R19b accumulation part alone, the R19c negative control).
    fproj (dtype float64 only): O2 in float32, Eq. 1-4 / O5 / O6 in double.
    Returns dict: C (npix,3) N (npix,3) D A Dep T (npix,), g, gsoft, last (Gaussian id), near, n_clamped,
    id_sum, evaluated, cert_bad, and grads (73, n) float64 if upstream was given.
    """
    n = int(np.asarray(g.opacity).shape[0])
    prm = _params(g, dtype)
    H, W = mask.shape
    m = np.ascontiguousarray(mask, np.uint8)
    pix = np.ascontiguousarray(pixels, np.int64)
    npix = int(pix.shape[0])
    out = np.zeros((npix, 10), dtype)
    iout = np.zeros((npix, 4), np.int32)
    id_sum = np.zeros(npix, np.float64)
    evaluated = np.zeros(npix, np.int64)
    cert = np.zeros(1, np.int64)
    bgd = np.asarray(bg, np.float64)
    up = None
    if upstream is not None:
        u = np.asarray(upstream, np.float64).reshape(npix, -1)
        up = np.zeros((npix, 10), np.float64)
        up[:, :u.shape[1]] = u
    grads = None if upstream is None else np.zeros((N_GRAD_ROWS, n), np.float64)
    gsoft = np.zeros(npix, np.float64)
    bnd = np.zeros((59, n), np.float64) if (bound and upstream is not None) else None
    fn = lib().oracle_render_f32 if dtype == np.float32 else lib().oracle_render_f64
    lib().oracle_set_bound_eval(0 if bound == "acc" else 1)
    if fproj:
        assert dtype == np.float64
        fn = lib().oracle_render_f64_fproj
    ca = cam_array(cam)
    fn(*[_p(a) for a in prm], n, int(g.sh_degree), _p(ca), W, H, _p(m), _p(bgd), _p(pix), npix, _p(out),
       _p(iout), _p(id_sum), _p(evaluated), _p(gsoft), int(certify), _p(cert), _p(up), _p(grads), _p(bnd))
    res = dict(C=out[:, 0:3], N=out[:, 3:6], D=out[:, 6], A=out[:, 7], Dep=out[:, 8], T=out[:, 9],
               g=iout[:, 0], last=iout[:, 1], near=iout[:, 2], n_clamped=iout[:, 3], id_sum=id_sum,
               evaluated=evaluated, cert_bad=int(cert[0]), gsoft=gsoft)
    if grads is not None:
        res["grads"] = grads
    if bnd is not None:
        res["bound"] = bnd  # R19b + R19c: float32 accumulation / evaluation bound on rows 0..58
    return res


def split_grads(grads, n):
    """(59, n) -> dict of named gradient blocks."""
    return dict(dmean=grads[0:3], dscale=grads[3:6], drot=grads[6:10], dopacity=grads[10], dsh=grads[11:59],
                g2d=grads[59:72], absgrad=grads[72])


def gc_weights(image, mask):
    """Eq. 9 weights w (H, W) from a (3, H, W) image (R23)."""
    H, W = mask.shape
    img = np.ascontiguousarray(image, np.float64).reshape(3, H, W)
    m = np.ascontiguousarray(mask, np.uint8)
    w = np.zeros((H, W), np.float64)
    lib().oracle_gc_weights(_p(img), _p(m), W, H, _p(w))
    return w


def gc_load(g, w):
    """L_GC-load over the listed pixels: (loss, mean ratio, dL/dg per pixel)."""
    g = np.ascontiguousarray(g, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    mu = np.zeros(1, np.float64)
    d = np.zeros(len(g), np.float64)
    L = lib().oracle_gc_load(_p(g), _p(w), len(g), _p(mu), _p(d))
    return float(L), float(mu[0]), d


def boundary_band(mask, r=1):
    """MB = dilation(RBM, r) XOR erosion(RBM, r), square SE, zero padding (R25)."""
    H, W = mask.shape
    m = np.ascontiguousarray(mask, np.uint8)
    band = np.zeros((H, W), np.uint8)
    lib().oracle_boundary_band(_p(m), W, H, int(r), _p(band))
    return band


def ban_loss(cam, mask, band, N, Dep, bw=0.1, lam=1.0, grads=False):
    """Eq. 8 L_ban (R26, R27).  N (3,H,W), Dep (H,W).  Returns (sum, count[, dN, dDep]) with the
    gradients of lam * sum / count."""
    H, W = mask.shape
    m = np.ascontiguousarray(mask, np.uint8)
    b = np.ascontiguousarray(band, np.uint8)
    Nd = np.ascontiguousarray(N, np.float64).reshape(3, H, W)
    Dd = np.ascontiguousarray(Dep, np.float64).reshape(H, W)
    loss = np.zeros(2, np.float64)
    dN = np.zeros((3, H, W), np.float64) if grads else None
    dD = np.zeros((H, W), np.float64) if grads else None
    lib().oracle_ban_loss(_p(cam_array(cam)), W, H, _p(m), _p(b), _p(Nd), _p(Dd), float(bw), float(lam),
                          _p(loss), _p(dN), _p(dD))
    if grads:
        return float(loss[0]), float(loss[1]), dN, dD
    return float(loss[0]), float(loss[1])


def rgb_loss(Cimg, Iimg, mask, grads=False):
    """Masked L_rgb = 0.8 L1 + 0.2 (1 - SSIM) (R28).  Returns (L, L1, S[, dC])."""
    H, W = mask.shape
    c = np.ascontiguousarray(Cimg, np.float64).reshape(3, H, W)
    i = np.ascontiguousarray(Iimg, np.float64).reshape(3, H, W)
    m = np.ascontiguousarray(mask, np.uint8)
    out = np.zeros(3, np.float64)
    dC = np.zeros((3, H, W), np.float64) if grads else None
    lib().oracle_rgb_loss(_p(c), _p(i), _p(m), W, H, _p(out), _p(dC))
    return (float(out[0]), float(out[1]), float(out[2])) + ((dC,) if grads else ())


def flatten_loss(scale):
    """L_s (PGSR flattening): mean over Gaussians of the minimum (activated) scale,
    and its gradient (1/N on the minimum axis, ties -> lowest index as in R4)."""
    s = np.asarray(scale, np.float64)
    k = np.argmin(s, axis=0)
    g = np.zeros_like(s)
    n = s.shape[1]
    g[k, np.arange(n)] = 1.0 / n
    return float(s[k, np.arange(n)].mean()), g


def adam_step(raw, grad, m, v, t, lr, b1=0.9, b2=0.999, eps=1e-15):
    """One Adam step (Kingma & Ba, bias-corrected) on raw parameters, written out plainly."""
    m = b1 * m + (1 - b1) * grad
    v = b2 * v + (1 - b2) * grad * grad
    mh = m / (1 - b1 ** t)
    vh = v / (1 - b2 ** t)
    return raw - lr * mh / (np.sqrt(vh) + eps), m, v


ADAM_ROWS = ("mean", 3), ("log_scale", 3), ("rot", 4), ("logit_opacity", 1)


def raw_grads(scale, opacity, dscale, dopacity, flatten_weight):
    """Chain rule to the raw parameters (R30): d/dlog s = s (dL/ds + w dL_s/ds), d/dlogit o = o (1 - o) dL/do."""
    _, gflat = flatten_loss(scale)
    s = np.asarray(scale, np.float64)
    o = np.asarray(opacity, np.float64)
    return (np.asarray(dscale, np.float64) + flatten_weight * gflat) * s, np.asarray(dopacity, np.float64) * o * (1 - o)


def train_update(p, g, m, v, t, hp, flatten_weight):
    """One NEXT-3 optimiser step, plainly: p = dict(mean, scale, rot, opacity, sh, log_scale, logit_opacity)
    (activated + raw), g = dict(dmean, dscale, drot, dopacity, dsh) (w.r.t. the activated values),
    m, v = [11 + K3][n] moments; hp = dict(lr_mean, lr_scale, lr_rot, lr_opacity, lr_sh_dc, lr_sh_rest,
    beta1, beta2, eps).  Returns (new p, m, v, L_s)."""
    f64 = lambda a: np.asarray(a, np.float64)
    Ls, _ = flatten_loss(p["scale"])
    g_logs, g_logit = raw_grads(p["scale"], p["opacity"], g["dscale"], g["dopacity"], flatten_weight)
    K3 = f64(p["sh"]).shape[0]
    raw = np.vstack([f64(p["mean"]), f64(p["log_scale"]), f64(p["rot"]), f64(p["logit_opacity"])[None], f64(p["sh"])])
    grad = np.vstack([f64(g["dmean"]), g_logs, f64(g["drot"]), g_logit[None], f64(g["dsh"])[:K3]])
    lr = np.array([hp["lr_mean"]] * 3 + [hp["lr_scale"]] * 3 + [hp["lr_rot"]] * 4 + [hp["lr_opacity"]] +
                  [hp["lr_sh_dc"]] * 3 + [hp["lr_sh_rest"]] * (K3 - 3))[:, None]
    raw, m, v = adam_step(raw, grad, f64(m), f64(v), t, lr, hp["beta1"], hp["beta2"], hp["eps"])
    q = dict(mean=raw[0:3], log_scale=raw[3:6], scale=np.exp(raw[3:6]), rot=raw[6:10], logit_opacity=raw[10],
             opacity=1.0 / (1.0 + np.exp(-raw[10])), sh=raw[11:])
    return q, m, v, Ls


# ------------------------------------------------------------------ densification (R31)
_M64 = (1 << 64) - 1


def splitmix64(x):
    """SplitMix64 finaliser of x (python ints, exact 64-bit arithmetic)."""
    z = (x + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def split_normals(seed, i, child):
    """The three N(0, 1) samples of split child `child` (0/1) of source Gaussian i (R31): counter
    c = 4 i + 2 child + k, h_k = splitmix64(seed ^ c) for k = 0, 1; u = (24-bit field + 0.5) / 2^24
    (high field of h_k, then its low field); Box-Muller (z0, z1) = sqrt(-2 ln u_a) (cos, sin)(2 pi u_b)
    on (u_a, u_b) = both fields of h_0, then of h_1; the first three of the four values are used."""
    out = []
    for k in (0, 1):
        h = splitmix64((seed ^ (4 * i + 2 * child + k)) & _M64)
        ua = ((h >> 40) + 0.5) / 16777216.0
        ub = ((h & 0xFFFFFF) + 0.5) / 16777216.0
        r = np.sqrt(-2.0 * np.log(ua))
        out += [r * np.cos(2 * np.pi * ub), r * np.sin(2 * np.pi * ub)]
    return np.array(out[:3])


def densify_actions(scale, opacity, accum, count, grad_threshold, dense_limit, min_opacity):
    """Per Gaussian: 0 drop (opacity < min_opacity), 3 split (mean view-space gradient >= threshold and
    max scale > dense_limit), 2 keep + clone (gradient >= threshold, max scale <= dense_limit), else
    1 keep.  Every decision in float32, as the GPU takes it (mean = accum / count, 0 if count = 0)."""
    f = np.float32
    s = np.asarray(scale, f)
    o = np.asarray(opacity, f)
    a, c = np.asarray(accum, f), np.asarray(count, f)
    avg = np.where(c > 0, a / np.where(c > 0, c, f(1)), f(0)).astype(f)
    big = s.max(axis=0) > f(dense_limit)
    hot = avg >= f(grad_threshold)
    act = np.where(hot, np.where(big, 3, 2), 1).astype(np.uint8)
    act[o < f(min_opacity)] = 0
    return act


def quat_to_rot(q):
    w, x, y, z = np.asarray(q, np.float64) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def densify_apply(p, m, v, act, seed):
    """3DGS clone / split / prune (R31), written out plainly.  Output order: the kept sources
    (actions 1, 2) in source order, then the clones (action 2) in source order, then the two split
    children (action 3) of each split source in source order.  A clone copies the source; a split
    child has mean mu + R(q) (s * z), scale s / 1.6 (log-scale = log of that), the source's rotation,
    opacity and SH; clones and children start with zero Adam moments.  p: dict of the activated and
    raw arrays ([rows][n]); returns (p', m', v')."""
    act = np.asarray(act)
    keep = np.flatnonzero((act == 1) | (act == 2))
    clone = np.flatnonzero(act == 2)
    split = np.flatnonzero(act == 3)
    keys = ("mean", "scale", "rot", "opacity", "sh", "log_scale", "logit_opacity")
    cols = lambda a, idx: np.asarray(a, np.float64)[..., idx]
    out = {k: [cols(p[k], keep), cols(p[k], clone)] for k in keys}
    mm = [cols(m, keep), np.zeros((m.shape[0], len(clone)))]
    vv = [cols(v, keep), np.zeros((v.shape[0], len(clone)))]
    ch = {k: [] for k in keys}
    for i in split:
        s = np.asarray(p["scale"], np.float64)[:, i]
        R = quat_to_rot(np.asarray(p["rot"], np.float64)[:, i])
        for c in (0, 1):
            z = split_normals(seed, int(i), c)
            sc = (np.asarray(p["scale"], np.float32)[:, i] / np.float32(1.6)).astype(np.float64)  # float32 as stored
            ch["mean"].append(np.asarray(p["mean"], np.float64)[:, i] + R @ (s * z))
            ch["scale"].append(sc)
            ch["log_scale"].append(np.log(sc))
            for k in ("rot", "opacity", "sh", "logit_opacity"):
                ch[k].append(np.asarray(p[k], np.float64)[..., i])
    for k in keys:
        base = np.asarray(p[k])
        shape = base.shape[:-1] + (len(split) * 2,)
        out[k].append(np.stack(ch[k], axis=-1) if ch[k] else np.zeros(shape))
        out[k] = np.concatenate(out[k], axis=-1)
    mm.append(np.zeros((m.shape[0], 2 * len(split))))
    vv.append(np.zeros((v.shape[0], 2 * len(split))))
    return out, np.concatenate(mm, axis=1), np.concatenate(vv, axis=1)


def sh_basis(x, y, z):
    Y = np.zeros(16, np.float64)
    lib().oracle_sh_basis(float(x), float(y), float(z), _p(Y))
    return Y


def lnup_f32(y):
    return float(lib().oracle_lnup_f32(float(y)))
