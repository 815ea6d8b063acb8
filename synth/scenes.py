"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the rasterizer's arithmetic (no projection, no
compositing, no keys).  It only draws Gaussians, cameras, building masks and
upstream gradients with the shapes and statistics of the paper's workloads
(SURVEY.md §8(d) "Synthetic inputs"; PAPER.md:188 oblique UAV frames at
5468x3636, PAPER.md:145-146 building groups, PAPER.md:84 flattened Gaussians).

Conventions (shared with include/pgsag.h):
  * Gaussians are SoA float32: mean[3][N], scale[3][N] (activated, > 0),
    rot[4][N] (w, x, y, z; not necessarily unit), opacity[N] in (0, 1),
    sh[(D+1)^2 * 3][N] laid out coefficient-major: row (l*3 + c).
  * Camera: x_cam = R (x_world - C), R row-major world->camera (rows = right,
    down, forward, i.e. the OpenCV frame), pinhole fx, fy, cx, cy.
  * World frame: z up, metres.
  * Mask: uint8 [H][W], nonzero = building pixel (the paper's RBM).

Random numbers come from numpy Generator(Philox(seed)); seed = 1677 + config
number unless overridden.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 1677


# --------------------------------------------------------------------------
# containers
# --------------------------------------------------------------------------
@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray  # (3,3) float32 world->camera, row-major
    C: np.ndarray  # (3,) float32 camera centre
    znear: float = 0.01


@dataclass
class Gaussians:
    mean: np.ndarray     # (3, N) f32
    scale: np.ndarray    # (3, N) f32 activated
    rot: np.ndarray      # (4, N) f32 (w, x, y, z)
    opacity: np.ndarray  # (N,) f32 in (0,1)
    sh: np.ndarray       # ((D+1)^2*3, N) f32
    sh_degree: int

    @property
    def n(self) -> int:
        return int(self.opacity.shape[0])


@dataclass
class Scene:
    name: str
    gaussians: Gaussians
    camera: Camera
    mask: np.ndarray               # (H, W) uint8
    bg: np.ndarray = field(default_factory=lambda: np.zeros(3, np.float32))
    seed: int = 0
    extra: dict = field(default_factory=dict)


# --------------------------------------------------------------------------
# small geometry helpers (scene construction only)
# --------------------------------------------------------------------------
def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """World->camera rotation (rows right, down, forward) and centre."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    if np.linalg.norm(r) < 1e-9:
        r = np.cross(f, np.array([0.0, 1.0, 0.0]))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f]).astype(np.float32)
    return R, eye.astype(np.float32)


def make_camera(eye, target, W, H, fx, fy=None, cx=None, cy=None, znear=0.01):
    R, C = look_at(eye, target)
    fy = fx if fy is None else fy
    cx = W / 2.0 if cx is None else cx
    cy = H / 2.0 if cy is None else cy
    return Camera(float(fx), float(fy), float(cx), float(cy), int(W), int(H), R, C, znear)


def mat_to_quat(Rm):
    """(N,3,3) rotation matrices -> (4,N) quaternions (w,x,y,z)."""
    m = Rm
    n = m.shape[0]
    m00, m11, m22 = m[:, 0, 0], m[:, 1, 1], m[:, 2, 2]
    tr = m00 + m11 + m22
    # Shepperd's method, vectorised: pick the largest of (tr, m00, m11, m22)
    pick = np.argmax(np.stack([tr, m00, m11, m22], axis=1), axis=1)
    q = np.zeros((n, 4))
    for k in range(4):
        sel = pick == k
        if not np.any(sel):
            continue
        a = m[sel]
        if k == 0:
            s = np.sqrt(1.0 + tr[sel]) * 2.0
            q[sel] = np.stack([0.25 * s, (a[:, 2, 1] - a[:, 1, 2]) / s,
                               (a[:, 0, 2] - a[:, 2, 0]) / s, (a[:, 1, 0] - a[:, 0, 1]) / s], 1)
        elif k == 1:
            s = np.sqrt(1.0 + a[:, 0, 0] - a[:, 1, 1] - a[:, 2, 2]) * 2.0
            q[sel] = np.stack([(a[:, 2, 1] - a[:, 1, 2]) / s, 0.25 * s,
                               (a[:, 0, 1] + a[:, 1, 0]) / s, (a[:, 0, 2] + a[:, 2, 0]) / s], 1)
        elif k == 2:
            s = np.sqrt(1.0 + a[:, 1, 1] - a[:, 0, 0] - a[:, 2, 2]) * 2.0
            q[sel] = np.stack([(a[:, 0, 2] - a[:, 2, 0]) / s, (a[:, 0, 1] + a[:, 1, 0]) / s,
                               0.25 * s, (a[:, 1, 2] + a[:, 2, 1]) / s], 1)
        else:
            s = np.sqrt(1.0 + a[:, 2, 2] - a[:, 0, 0] - a[:, 1, 1]) * 2.0
            q[sel] = np.stack([(a[:, 1, 0] - a[:, 0, 1]) / s, (a[:, 0, 2] + a[:, 2, 0]) / s,
                               (a[:, 1, 2] + a[:, 2, 1]) / s, 0.25 * s], 1)
    return q.T


def small_rotations(rng, n, max_deg):
    """(n,3,3) rotations about random axes by angles U[0, max_deg]."""
    ax = rng.normal(size=(n, 3))
    ax /= np.linalg.norm(ax, axis=1, keepdims=True)
    ang = np.deg2rad(rng.uniform(0.0, max_deg, size=n))
    K = np.zeros((n, 3, 3))
    K[:, 0, 1], K[:, 0, 2] = -ax[:, 2], ax[:, 1]
    K[:, 1, 0], K[:, 1, 2] = ax[:, 2], -ax[:, 0]
    K[:, 2, 0], K[:, 2, 1] = -ax[:, 1], ax[:, 0]
    s, c = np.sin(ang)[:, None, None], np.cos(ang)[:, None, None]
    return np.eye(3)[None] + s * K + (1.0 - c) * (K @ K)


# --------------------------------------------------------------------------
# buildings
# --------------------------------------------------------------------------
@dataclass
class Box:
    cx: float
    cy: float
    hx: float   # half extents in the box frame
    hy: float
    h: float    # height (base at z = 0)
    yaw: float  # radians


def make_buildings(rng, centre, extent, pitch=50.0, jitter=8.0):
    """Buildings on a jittered street grid (SURVEY §8(d) common parameters)."""
    boxes = []
    n = max(1, int(round(extent / pitch)))
    x0 = centre[0] - extent / 2 + pitch / 2
    y0 = centre[1] - extent / 2 + pitch / 2
    for i in range(n):
        for j in range(n):
            fx_, fy_ = rng.uniform(12, 40, size=2)
            h = float(np.clip(np.exp(rng.normal(math.log(20.0), 0.5)), 6.0, 80.0))
            boxes.append(Box(
                cx=x0 + i * pitch + rng.uniform(-jitter, jitter),
                cy=y0 + j * pitch + rng.uniform(-jitter, jitter),
                hx=fx_ / 2, hy=fy_ / 2, h=h,
                yaw=math.radians(rng.uniform(0, 90))))
    return boxes


def _box_faces(b: Box):
    """List of (origin, u_axis, v_axis, normal) for the 4 walls and roof; u,v span the face."""
    c, s = math.cos(b.yaw), math.sin(b.yaw)
    ex = np.array([c, s, 0.0])
    ey = np.array([-s, c, 0.0])
    ez = np.array([0.0, 0.0, 1.0])
    ctr = np.array([b.cx, b.cy, 0.0])
    faces = []
    # walls: +x, -x, +y, -y
    for sgn, ax, half, other, ohalf in ((1, ex, b.hx, ey, b.hy), (-1, ex, b.hx, ey, b.hy),
                                        (1, ey, b.hy, ex, b.hx), (-1, ey, b.hy, ex, b.hx)):
        o = ctr + sgn * half * ax - ohalf * other
        faces.append((o, 2 * ohalf * other, b.h * ez, sgn * ax))
    # roof
    o = ctr - b.hx * ex - b.hy * ey + b.h * ez
    faces.append((o, 2 * b.hx * ex, 2 * b.hy * ey, ez))
    return faces


def sample_on_faces(rng, faces, n):
    areas = np.array([np.linalg.norm(np.cross(u, v)) for (_, u, v, _) in faces])
    idx = rng.choice(len(faces), size=n, p=areas / areas.sum())
    a = rng.uniform(size=n)
    b = rng.uniform(size=n)
    O = np.stack([faces[k][0] for k in range(len(faces))])[idx]
    U = np.stack([faces[k][1] for k in range(len(faces))])[idx]
    V = np.stack([faces[k][2] for k in range(len(faces))])[idx]
    Nn = np.stack([faces[k][3] for k in range(len(faces))])[idx]
    P = O + a[:, None] * U + b[:, None] * V
    Uh = U / np.linalg.norm(U, axis=1, keepdims=True)
    return P, Nn, Uh


def surface_gaussians(rng, P, Nn, Uh, jitter_n=0.05, s_lo=0.05, s_hi=0.6, sh_degree=3,
                      dc_std=0.6, hi_std=0.05):
    """Flattened Gaussians lying on surfaces (normal axis = 0.01 x smaller in-plane scale)."""
    n = P.shape[0]
    P = P + rng.normal(0.0, jitter_n, size=(n, 1)) * Nn
    # in-plane frame with random in-plane angle
    Vh = np.cross(Nn, Uh)
    th = rng.uniform(0, 2 * np.pi, size=n)[:, None]
    t1 = np.cos(th) * Uh + np.sin(th) * Vh
    t2 = np.cross(Nn, t1)
    Rm = np.stack([t1, t2, Nn], axis=2)          # columns = axes
    Rm = small_rotations(rng, n, 5.0) @ Rm          # +-5 deg jitter of the normal
    s12 = np.exp(rng.uniform(math.log(s_lo), math.log(s_hi), size=(n, 2)))
    s3 = 0.01 * s12.min(axis=1)
    scale = np.concatenate([s12, s3[:, None]], axis=1).T
    q = mat_to_quat(Rm)
    q *= rng.uniform(0.5, 2.0, size=(1, n))          # un-normalised storage exercises the normalisation
    op = mixture_opacity(rng, n)
    sh = random_sh(rng, n, sh_degree, dc_std, hi_std)
    return P.T, scale, q, op, sh


def mixture_opacity(rng, n):
    """60% U[0.5,0.99] + 40% U[0.002,0.3] (bimodal like trained 3DGS; some below 1/255)."""
    hi = rng.uniform(size=n) < 0.6
    return np.where(hi, rng.uniform(0.5, 0.99, size=n), rng.uniform(0.002, 0.3, size=n))


def random_sh(rng, n, deg, dc_std, hi_std):
    k = (deg + 1) ** 2
    sh = rng.normal(0.0, hi_std, size=(k * 3, n))
    sh[0:3] = rng.normal(0.0, dc_std, size=(3, n))
    return sh


def ray_cast_mask(cam: Camera, boxes, device="cpu"):
    """mask[j][i] = 1 iff the pixel-centre ray hits a building box (buildings stand on
    the ground, so any box hit precedes the ground hit).  Pure scene construction."""
    import torch
    W, H = cam.width, cam.height
    R = torch.tensor(cam.R, dtype=torch.float64, device=device)
    C = torch.tensor(cam.C, dtype=torch.float64, device=device)
    mask = torch.zeros((H, W), dtype=torch.uint8, device=device)
    for b in boxes:
        # pixel bbox of the projected box corners (whole image if any corner is behind)
        cs, sn = math.cos(b.yaw), math.sin(b.yaw)
        corners = []
        for sx in (-1, 1):
            for sy in (-1, 1):
                for z in (0.0, b.h):
                    corners.append([b.cx + sx * b.hx * cs - sy * b.hy * sn,
                                    b.cy + sx * b.hx * sn + sy * b.hy * cs, z])
        pc = (torch.tensor(corners, dtype=torch.float64, device=device) - C) @ R.T
        if bool((pc[:, 2] <= 0.05).any()):
            i0, i1, j0, j1 = 0, W, 0, H
        else:
            u = cam.fx * pc[:, 0] / pc[:, 2] + cam.cx
            v = cam.fy * pc[:, 1] / pc[:, 2] + cam.cy
            i0 = max(0, int(math.floor(float(u.min()))) - 1)
            i1 = min(W, int(math.ceil(float(u.max()))) + 1)
            j0 = max(0, int(math.floor(float(v.min()))) - 1)
            j1 = min(H, int(math.ceil(float(v.max()))) + 1)
            if i0 >= i1 or j0 >= j1:
                continue
        ii = torch.arange(i0, i1, dtype=torch.float64, device=device)
        jj = torch.arange(j0, j1, dtype=torch.float64, device=device)
        dx = ((ii + 0.5 - cam.cx) / cam.fx)[None, :].expand(j1 - j0, -1)
        dy = ((jj + 0.5 - cam.cy) / cam.fy)[:, None].expand(-1, i1 - i0)
        dcam = torch.stack([dx, dy, torch.ones_like(dx)], dim=-1)
        dw = dcam @ R                                   # R^T d  (world direction)
        # into the box frame
        ox, oy, oz = float(C[0]) - b.cx, float(C[1]) - b.cy, float(C[2])
        lox, loy = cs * ox + sn * oy, -sn * ox + cs * oy
        ldx = cs * dw[..., 0] + sn * dw[..., 1]
        ldy = -sn * dw[..., 0] + cs * dw[..., 1]
        ldz = dw[..., 2]
        tmin = torch.full_like(ldx, 0.0)
        tmax = torch.full_like(ldx, float("inf"))
        for o, d, lo, hi in ((lox, ldx, -b.hx, b.hx), (loy, ldy, -b.hy, b.hy), (oz, ldz, 0.0, b.h)):
            inv = 1.0 / torch.where(d.abs() < 1e-12, torch.full_like(d, 1e-12), d)
            t1 = (lo - o) * inv
            t2 = (hi - o) * inv
            tmin = torch.maximum(tmin, torch.minimum(t1, t2))
            tmax = torch.minimum(tmax, torch.maximum(t1, t2))
        hit = (tmax >= tmin) & (tmax > 0)
        mask[j0:j1, i0:i1] |= hit.to(torch.uint8)
    return mask.cpu().numpy()


def _pack(P, scale, q, op, sh, deg) -> Gaussians:
    return Gaussians(
        mean=np.ascontiguousarray(P, np.float32),
        scale=np.ascontiguousarray(scale, np.float32),
        rot=np.ascontiguousarray(q, np.float32),
        opacity=np.ascontiguousarray(op, np.float32),
        sh=np.ascontiguousarray(sh, np.float32),
        sh_degree=deg)


def concat_gaussians(parts, deg):
    return _pack(*(np.concatenate([p[k] for p in parts], axis=-1) for k in range(5)), deg)


# --------------------------------------------------------------------------
# configs (BASELINE.json configs[0..4])
# --------------------------------------------------------------------------
def random_gaussians(rng, n, lo, hi, s_lo=0.03, s_hi=0.3, o_lo=0.05, o_hi=0.99, deg=3, sh_std=0.3):
    """C1-style random Gaussians: uniform box, log-U scales with one axis x0.05, random unit q."""
    P = rng.uniform(lo, hi, size=(n, 3)).T
    sc = np.exp(rng.uniform(math.log(s_lo), math.log(s_hi), size=(3, n)))
    ax = rng.integers(0, 3, size=n)
    sc[ax, np.arange(n)] *= 0.05
    q = rng.normal(size=(4, n))
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    op = rng.uniform(o_lo, o_hi, size=n)
    sh = rng.normal(0.0, sh_std, size=((deg + 1) ** 2 * 3, n))
    return _pack(P, sc, q, op, sh, deg)


def fuzz_scene(seed):
    """Randomised small scene of the parity sweep (tests/test_gpu_fuzz.py) and of the oracle's
    R19c bound pin: image size (ragged, down to one partial tile), Gaussian count, SH degree,
    scale / opacity ranges, mask density, background and focal length all vary with the seed.
    Returns (Scene, bg)."""
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(5, 90)), int(rng.integers(5, 70))
    n = int(rng.integers(1, 700))
    deg = int(rng.integers(0, 4))
    g = random_gaussians(rng, n, [-1.5, -1.2, 1.5], [1.5, 1.2, 7.0],
                         s_lo=float(rng.uniform(0.005, 0.05)), s_hi=float(rng.uniform(0.1, 0.8)),
                         o_lo=float(rng.uniform(0.0, 0.3)), o_hi=float(rng.uniform(0.5, 1.0)), deg=deg,
                         sh_std=float(rng.uniform(0.1, 0.6)))
    f = float(rng.uniform(0.6, 1.6)) * max(W, H)
    cam = Camera(f, f * float(rng.uniform(0.8, 1.25)), W / 2.0 + float(rng.uniform(-3, 3)),
                 H / 2.0 + float(rng.uniform(-3, 3)), W, H, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    mask = (rng.uniform(size=(H, W)) < float(rng.uniform(0.05, 1.0))).astype(np.uint8)
    if not mask.any():
        mask[H // 2, W // 2] = 1
    bg = tuple(float(x) for x in rng.uniform(0, 1, 3)) if rng.uniform() < 0.5 else (0.0, 0.0, 0.0)
    return Scene(f"fuzz{seed}", g, cam, mask, seed=seed), bg


def config1(seed=None, n=1000, W=64, H=64, sh_degree=3, mask_p=0.5):
    """C1: 1000 random Gaussians, one 64x64 camera at the origin looking +z, 50% random mask."""
    seed = SEED_BASE + 1 if seed is None else seed
    rng = np.random.Generator(np.random.Philox(seed))
    g = random_gaussians(rng, n, [-1.5, -1.5, 2.0], [1.5, 1.5, 6.0], deg=sh_degree)
    cam = Camera(64.0 * W / 64, 64.0 * H / 64, W / 2.0, H / 2.0, W, H,
                 np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    mask = (rng.uniform(size=(H, W)) < mask_p).astype(np.uint8)
    return Scene("C1", g, cam, mask, seed=seed)


def urban_scene(rng, n_total, boxes, region_centre, region_extent, cams, sh_degree=3,
                frac_buildings=0.75):
    faces = [f for b in boxes for f in _box_faces(b)]
    nb = int(round(n_total * frac_buildings))
    ng = n_total - nb
    P, Nn, Uh = sample_on_faces(rng, faces, nb)
    part_b = surface_gaussians(rng, P, Nn, Uh, sh_degree=sh_degree)
    gp = np.stack([
        rng.uniform(region_centre[0] - region_extent / 2, region_centre[0] + region_extent / 2, ng),
        rng.uniform(region_centre[1] - region_extent / 2, region_centre[1] + region_extent / 2, ng),
        np.zeros(ng)], axis=1)
    part_g = surface_gaussians(rng, gp, np.tile([0.0, 0.0, 1.0], (ng, 1)),
                               np.tile([1.0, 0.0, 0.0], (ng, 1)), sh_degree=sh_degree)
    return concat_gaussians([part_b, part_g], sh_degree)


def config2(seed=None, n=100_000, W=1920, H=1080, f=1400.0, device="cpu"):
    """C2: 3-building cluster, camera 40 m up, 30 m stand-off, pitch ~30 deg, 1080p."""
    seed = SEED_BASE + 2 if seed is None else seed
    rng = np.random.Generator(np.random.Philox(seed))
    boxes = [Box(-22.0, 8.0, 8.0, 7.0, 24.0, math.radians(10)),
             Box(0.0, 12.0, 9.0, 9.0, 32.0, math.radians(35)),
             Box(22.0, 6.0, 7.0, 8.0, 20.0, math.radians(60))]
    cam = make_camera([0.0, -30.0 - 35.0, 40.0], [0.0, 8.0, 12.0], W, H, f)
    g = urban_scene(rng, n, boxes, (0.0, 8.0), 90.0, [cam])
    return Scene("C2", g, cam, ray_cast_mask(cam, boxes, device), seed=seed, extra={"boxes": boxes})


def aerial_camera(centre, heading_deg, ground_dist, altitude, W, H, f):
    h = math.radians(heading_deg)
    eye = [centre[0] - ground_dist * math.cos(h), centre[1] - ground_dist * math.sin(h), altitude]
    return make_camera(eye, [centre[0], centre[1], 0.0], W, H, f)


def config3(seed=None, n=2_000_000, W=5472, H=3648, f=3648.0, device="cpu"):
    """C3: one 250 m sub-region, oblique camera at 120 m altitude, pitch 45 deg, 5472x3648."""
    seed = SEED_BASE + 3 if seed is None else seed
    rng = np.random.Generator(np.random.Philox(seed))
    centre = (0.0, 0.0)
    boxes = make_buildings(rng, centre, 250.0)
    cam = aerial_camera(centre, 30.0, 120.0, 120.0, W, H, f)
    g = urban_scene(rng, n, boxes, centre, 250.0, [cam])
    return Scene("C3", g, cam, ray_cast_mask(cam, boxes, device), seed=seed, extra={"boxes": boxes})


def subregion(region: int, n=1_500_000, W=5472, H=3648, f=3648.0, n_views=40, seed=None):
    """C4 sub-region r: its own buildings + Gaussians; 40 cameras = 8 headings x 5 ring radii
    in [80,160] m at 120 m altitude looking at the sub-region centre.  Masks are cast lazily
    (view_mask) because 40 full-res masks are ~800 MB."""
    seed = SEED_BASE + 4 * 1000 + region if seed is None else seed
    rng = np.random.Generator(np.random.Philox(seed))
    centre = (300.0 * (region % 4), 300.0 * (region // 4))
    boxes = make_buildings(rng, centre, 200.0)
    cams = []
    for k in range(n_views):
        heading = 45.0 * (k % 8) + 7.0 * region
        radius = 80.0 + 20.0 * (k // 8)
        cams.append(aerial_camera(centre, heading, radius, 120.0, W, H, f))
    g = urban_scene(rng, n, boxes, centre, 200.0, cams)
    return {"gaussians": g, "boxes": boxes, "cameras": cams, "seed": seed, "centre": centre}


def config5(seed=None, n=3_000_000, W=3840, H=2160, f=2800.0, device="cpu"):
    """C5 load-imbalance stress: 80% of Gaussians on 3 facade patches covering ~6% of the
    frame, 20% uniform over the region; heavy-tailed per-tile counts."""
    seed = SEED_BASE + 5 if seed is None else seed
    rng = np.random.Generator(np.random.Philox(seed))
    boxes = [Box(-30.0, 0.0, 10.0, 10.0, 30.0, 0.0), Box(0.0, 20.0, 12.0, 8.0, 45.0, 0.0),
             Box(35.0, 5.0, 9.0, 11.0, 25.0, 0.0)]
    cam = make_camera([0.0, -110.0, 30.0], [0.0, 10.0, 20.0], W, H, f)
    # three dense patches: a 12x10 m window of the camera-facing (-y) wall of each box
    parts = []
    n_dense = int(0.8 * n)
    per = [n_dense // 3, n_dense // 3, n_dense - 2 * (n_dense // 3)]
    for b, m in zip(boxes, per):
        o = np.array([b.cx - 6.0, b.cy - b.hy, 0.3 * b.h])
        faces = [(o, np.array([12.0, 0.0, 0.0]), np.array([0.0, 0.0, 10.0]), np.array([0.0, -1.0, 0.0]))]
        P, Nn, Uh = sample_on_faces(rng, faces, m)
        parts.append(surface_gaussians(rng, P, Nn, Uh))
    nu = n - n_dense
    faces = [f_ for b in boxes for f_ in _box_faces(b)]
    P, Nn, Uh = sample_on_faces(rng, faces, nu // 2)
    parts.append(surface_gaussians(rng, P, Nn, Uh))
    ng = nu - nu // 2
    gp = np.stack([rng.uniform(-80, 80, ng), rng.uniform(-40, 80, ng), np.zeros(ng)], axis=1)
    parts.append(surface_gaussians(rng, gp, np.tile([0.0, 0.0, 1.0], (ng, 1)),
                                   np.tile([1.0, 0.0, 0.0], (ng, 1))))
    g = concat_gaussians(parts, 3)
    return Scene("C5", g, cam, ray_cast_mask(cam, boxes, device), seed=seed, extra={"boxes": boxes})


def make_config(cfg: int, **kw) -> Scene:
    return {1: config1, 2: config2, 3: config3, 5: config5}[cfg](**kw)


def upstream_grads(H, W, seed, mask=None, sparse_pixels=None):
    """Upstream dL/d(C,N,D,A,Dep) ~ N(0,1) per channel (planar float32).  With
    sparse_pixels (flat indices), every other pixel gets 0."""
    rng = np.random.Generator(np.random.Philox(seed))
    g = {
        "dC": rng.normal(size=(3, H, W)).astype(np.float32),
        "dN": rng.normal(size=(3, H, W)).astype(np.float32),
        "dD": rng.normal(size=(H, W)).astype(np.float32),
        "dA": rng.normal(size=(H, W)).astype(np.float32),
        "dDep": rng.normal(size=(H, W)).astype(np.float32),
    }
    keep = None
    if sparse_pixels is not None:
        keep = np.zeros(H * W, bool)
        keep[np.asarray(sparse_pixels)] = True
        keep = keep.reshape(H, W)
    if mask is not None:
        keep = (mask != 0) if keep is None else (keep & (mask != 0))
    if keep is not None:
        for k in g:
            g[k] = np.where(keep, g[k], np.float32(0.0)).astype(np.float32)
    return g


def sample_pixels(mask, n, seed):
    """Fixed-seed sample of n masked pixel flat indices."""
    rng = np.random.Generator(np.random.Philox(seed))
    idx = np.flatnonzero(mask.reshape(-1))
    if idx.size <= n:
        return idx
    return np.sort(rng.choice(idx, size=n, replace=False))


def reference_image(H, W, seed):
    """Synthetic 'photo' (3, H, W) float32 in [0, 1]: smooth shading, a few sharp-edged
    rectangles (facade-like structure) and mild noise — input for Eq. 9's nabla I weights."""
    rng = np.random.Generator(np.random.Philox(seed))
    yy, xx = np.mgrid[0:H, 0:W].astype(np.float64)
    img = np.empty((3, H, W))
    for c in range(3):
        img[c] = 0.4 + 0.2 * np.sin(xx / max(W, 1) * rng.uniform(2, 6) + c) * np.cos(yy / max(H, 1) * rng.uniform(2, 6))
    for _ in range(max(3, (H * W) // 400)):
        x0, y0 = rng.integers(0, W), rng.integers(0, H)
        x1, y1 = min(W, x0 + rng.integers(2, max(3, W // 4))), min(H, y0 + rng.integers(2, max(3, H // 4)))
        img[:, y0:y1, x0:x1] += rng.uniform(-0.3, 0.3, size=(3, 1, 1))
    img += rng.normal(0, 0.01, size=img.shape)
    return np.clip(img, 0, 1).astype(np.float32)
