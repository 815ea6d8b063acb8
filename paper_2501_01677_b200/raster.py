"""Thin Python driver over the C ABI: owns the device buffers (PyTorch is used
for device memory and streams only) and calls pgsag_preprocess -> pgsag_bin_sort
-> pgsag_render_fwd -> pgsag_render_bwd on the current torch stream.

All arithmetic of the path runs in libpgsag.so; this module only allocates,
marshals pointers and re-allocates the entry buffers when M outgrows them.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L

TILE = 16


def make_camera(fx, fy, cx, cy, width, height, R, Cw, znear=0.01) -> L.Camera:
    cam = L.Camera()
    cam.fx, cam.fy, cam.cx, cam.cy = float(fx), float(fy), float(cx), float(cy)
    cam.width, cam.height = int(width), int(height)
    Rf = [float(v) for v in (R.reshape(-1).tolist() if hasattr(R, "reshape") else R)]
    Cf = [float(v) for v in (Cw.reshape(-1).tolist() if hasattr(Cw, "reshape") else Cw)]
    for k in range(9):
        cam.R[k] = Rf[k]
    for k in range(3):
        cam.C[k] = Cf[k]
    cam.znear = float(znear)
    return cam


def camera_from(obj) -> L.Camera:
    """From any object with fx, fy, cx, cy, width, height, R, C, znear (e.g. synth.scenes.Camera)."""
    return make_camera(obj.fx, obj.fy, obj.cx, obj.cy, obj.width, obj.height, obj.R, obj.C,
                       getattr(obj, "znear", 0.01))


@dataclass
class GaussianTensors:
    mean: torch.Tensor     # (3, n) f32
    scale: torch.Tensor    # (3, n)
    rot: torch.Tensor      # (4, n)
    opacity: torch.Tensor  # (n,)
    sh: torch.Tensor       # ((deg+1)^2*3, n)
    sh_degree: int

    @property
    def n(self):
        return int(self.opacity.shape[0])

    @staticmethod
    def from_numpy(g, device="cuda"):
        t = lambda a: torch.as_tensor(a, dtype=torch.float32).contiguous().to(device)
        return GaussianTensors(t(g.mean), t(g.scale), t(g.rot), t(g.opacity), t(g.sh), int(g.sh_degree))

    def struct(self) -> L.Gaussians:
        s = L.Gaussians()
        s.n, s.sh_degree = self.n, self.sh_degree
        s.mean, s.scale, s.rot = self.mean.data_ptr(), self.scale.data_ptr(), self.rot.data_ptr()
        s.opacity, s.sh = self.opacity.data_ptr(), self.sh.data_ptr()
        return s


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Rasterizer:
    """Buffers for one (n, width, height, sh_degree) problem; reusable across views."""

    def __init__(self, n, width, height, sh_degree=3, capacity=None, device="cuda", counters=True, sat=True,
                 absgrad=False, sync_free=False):
        """sync_free: use pgsag_bin_sort_async (no host synchronisation per view; M is read back
        lazily and check_capacity() re-sorts a view whose M exceeded the capacity)."""
        self.want_sat = bool(sat)
        self.sync_free = bool(sync_free)
        self._m_host = torch.zeros(1, dtype=torch.int64, pin_memory=torch.cuda.is_available())
        self.want_absgrad = bool(absgrad)
        self.n, self.W, self.H, self.deg = int(n), int(width), int(height), int(sh_degree)
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        dev = self.device
        n = max(self.n, 1)
        self.TX, self.TY = (self.W + TILE - 1) // TILE, (self.H + TILE - 1) // TILE
        T = self.TX * self.TY
        f32, i32, u8 = torch.float32, torch.int32, torch.uint8
        e = lambda *shape, dtype=f32: torch.empty(*shape, dtype=dtype, device=dev)
        # A0 / A1 outputs
        self.tile_cnt = e(T, dtype=i32)
        self.sat = e((self.TY + 1) * (self.TX + 1), dtype=i32)
        self.active = e(T, dtype=i32)
        self.n_active = e(1, dtype=i32)
        self.active_bits = e(self.TY * ((self.TX + 31) // 32), dtype=i32)
        self.mean2d = e(n, 2)
        self.conic_o = e(n, 4)
        self.depth = e(n)
        self.rect = e(n, 4, dtype=torch.int16)
        self.tiles_touched = e(n, dtype=i32)
        self.rgb_d = e(n, 4)
        self.ncam = e(n, 4)
        self.flags = e(n, dtype=i32)
        # A6 outputs
        HW = self.H * self.W
        self.img_C = torch.zeros(3, self.H, self.W, dtype=f32, device=dev)
        self.img_N = torch.zeros(3, self.H, self.W, dtype=f32, device=dev)
        self.img_D = torch.zeros(self.H, self.W, dtype=f32, device=dev)
        self.img_A = torch.zeros(self.H, self.W, dtype=f32, device=dev)
        self.img_Dep = torch.zeros(self.H, self.W, dtype=f32, device=dev)
        self.img_T = torch.ones(self.H, self.W, dtype=f32, device=dev)
        self.img_g = torch.zeros(self.H, self.W, dtype=i32, device=dev)
        self.img_last = torch.full((self.H, self.W), -1, dtype=i32, device=dev)
        self.counters = torch.zeros(4, dtype=torch.int64, device=dev) if counters else None
        self.gc_stats = torch.zeros(5, dtype=torch.float64, device=dev)  # NEXT-1: N, sum r, sum r^2, L, mean r
        self.gc_w = None
        # A8 outputs
        K3 = (self.deg + 1) ** 2 * 3
        self.dmean = e(3, n)
        self.dscale = e(3, n)
        self.drot = e(4, n)
        self.dopacity = e(n)
        self.dsh = torch.zeros(K3, n, dtype=f32, device=dev)
        self.absgrad = e(n)
        self.grad2d = e(14, n)
        self.ranges = e(2 * T, dtype=i32)
        self.order = e(T, dtype=i32)  # LPT work order of the active tiles (pgsag_bins.order)
        self._alloc_bins(capacity if capacity is not None else max(1024, 8 * self.n))
        self.M = 0
        self._build_structs()
        del HW, u8

    # ------------------------------------------------------------ buffers
    def _alloc_bins(self, cap):
        self.capacity = int(cap)
        self.tile_keys = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=self.device)
        self.vals = torch.empty(max(self.capacity, 1), dtype=torch.int32, device=self.device)
        self.ws_bytes = L.workspace_size(self.n, self.W, self.H, self.capacity)
        self.ws = torch.empty(max(self.ws_bytes, 256), dtype=torch.uint8, device=self.device)

    def _build_structs(self):
        p = L.Projected()
        p.mean2d, p.conic_o, p.depth = self.mean2d.data_ptr(), self.conic_o.data_ptr(), self.depth.data_ptr()
        p.rect, p.tiles_touched = self.rect.data_ptr(), self.tiles_touched.data_ptr()
        p.rgb_d, p.ncam, p.flags = self.rgb_d.data_ptr(), self.ncam.data_ptr(), self.flags.data_ptr()
        self._proj = p
        tm = L.TileMask()
        tm.tile_cnt, tm.active = self.tile_cnt.data_ptr(), self.active.data_ptr()
        tm.sat = self.sat.data_ptr() if self.want_sat else None
        tm.n_active, tm.active_bits = self.n_active.data_ptr(), self.active_bits.data_ptr()
        self._tm = tm
        self._build_bins()
        im = L.Image()
        im.C, im.N, im.D, im.A = self.img_C.data_ptr(), self.img_N.data_ptr(), self.img_D.data_ptr(), \
            self.img_A.data_ptr()
        im.Dep, im.T, im.g, im.last = self.img_Dep.data_ptr(), self.img_T.data_ptr(), self.img_g.data_ptr(), \
            self.img_last.data_ptr()
        im.counters = self.counters.data_ptr() if self.counters is not None else None
        self._img = im
        gg = L.GaussianGrad()
        gg.dmean, gg.dscale, gg.drot = self.dmean.data_ptr(), self.dscale.data_ptr(), self.drot.data_ptr()
        gg.dopacity, gg.dsh = self.dopacity.data_ptr(), self.dsh.data_ptr()
        gg.absgrad2d = self.absgrad.data_ptr() if self.want_absgrad else None
        gg.grad2d = None
        self._grad = gg

    def _build_bins(self):
        """The pgsag_bins struct over the current entry buffers (the only struct a capacity change
        touches: the image / gradient structs keep their per-call fields across a retry)."""
        b = L.Bins()
        b.tile_keys, b.vals, b.ranges = self.tile_keys.data_ptr(), self.vals.data_ptr(), self.ranges.data_ptr()
        b.capacity, b.n_dup = self.capacity, 0
        b.order = self.order.data_ptr()
        self._bins = b

    def export_grad2d(self, on=True):
        """Also copy A7's per-Gaussian screen-space gradients into self.grad2d ([14][n])."""
        self._grad.grad2d = self.grad2d.data_ptr() if on else None

    # ---------------------------------------------------------- the path
    def gc_weights(self, image: torch.Tensor, mask: torch.Tensor) -> torch.Tensor:
        """Eq. 9 weights w (H, W) of a (3, H, W) float32 image on the mask (pgsag_gc_weights)."""
        assert image.dtype == torch.float32 and tuple(image.shape) == (3, self.H, self.W) and image.is_contiguous()
        w = torch.empty(self.H, self.W, dtype=torch.float32, device=self.device)
        L.gc_weights(C.c_void_p(image.data_ptr()), C.c_void_p(mask.data_ptr()), self.W, self.H,
                     C.c_void_p(w.data_ptr()), C.c_void_p(self.ws.data_ptr()), self.ws_bytes, _stream())
        return w

    def boundary_band(self, mask: torch.Tensor, r: int = 1) -> torch.Tensor:
        """NEXT-2 boundary band MB of the building mask (pgsag_boundary_band)."""
        band = torch.empty_like(mask)
        L.boundary_band(C.c_void_p(mask.data_ptr()), self.W, self.H, r, C.c_void_p(band.data_ptr()), _stream())
        return band

    def ban_loss(self, band: torch.Tensor, lam=1.0, bw=0.1, mean=True, dN=None, dDep=None):
        """NEXT-2 L_ban (Eq. 8) on the last forward's N and Dep; returns the device (sum, count) and ADDS
        lam * dS/dN, lam * dS/dDep into dN / dDep when given (S = sum/count if mean)."""
        loss = torch.zeros(2, dtype=torch.float64, device=self.device)
        p = lambda t: None if t is None else C.c_void_p(t.data_ptr())
        L.ban_loss(self._cam, C.c_void_p(self._mask.data_ptr()), p(band), p(self.img_N), p(self.img_Dep), bw, lam,
                   int(mean), p(loss), p(dN), p(dDep), _stream())
        return loss

    def gc_load(self):
        """(L_GC-load, mean ratio, N) from the last forward with gc_w (A6's fused statistics, Eq. 9
        evaluated on the device: pgsag_image.gc_stats[3], [4])."""
        n, _, _, L_, mu = self.gc_stats.tolist()
        return L_, mu, n

    def forward(self, g: GaussianTensors, cam: L.Camera, mask: torch.Tensor, bg=(0.0, 0.0, 0.0), gc_w=None,
                wait_before_render=None):
        """A0-A6.  wait_before_render: optional torch.cuda.Event the stream waits on between the
        sort and A6 (e.g. gc_w computed concurrently on another stream)."""
        assert g.n == self.n and g.sh_degree == self.deg
        assert mask.dtype == torch.uint8 and tuple(mask.shape) == (self.H, self.W) and mask.is_contiguous()
        st = _stream()
        self.gc_w = gc_w
        self._img.gc_w = None if gc_w is None else gc_w.data_ptr()
        self._img.gc_stats = self.gc_stats.data_ptr()
        self._g = g.struct()
        self._gt = g
        self._cam = cam
        self._mask = mask
        self._bg = (C.c_float * 3)(*[float(v) for v in bg])
        if self.counters is not None:
            self.counters.zero_()
        ws = C.c_void_p(self.ws.data_ptr())
        L.preprocess(self._g, cam, C.c_void_p(mask.data_ptr()), self._tm, self._proj, ws, self.ws_bytes, st)
        if self.sync_free:
            L.bin_sort_async(self._proj, self._tm, cam, self.n, self._bins, C.c_void_p(self._m_host.data_ptr()), ws,
                             self.ws_bytes, st)
            self.M = None  # known after the stream passes the sort: see check_capacity()
            if wait_before_render is not None:
                torch.cuda.current_stream().wait_event(wait_before_render)
            L.render_fwd(self._proj, self._bins, self._tm, cam, C.c_void_p(mask.data_ptr()), self._bg, self._img,
                         ws, self.ws_bytes, st)
            return dict(C=self.img_C, N=self.img_N, D=self.img_D, A=self.img_A, Dep=self.img_Dep, T=self.img_T,
                        g=self.img_g, last=self.img_last)
        rc = L.bin_sort(self._proj, self._tm, cam, self.n, self._bins, ws, self.ws_bytes, st)
        if rc == L.PGSAG_ECAPACITY:
            self._alloc_bins(int(self._bins.n_dup * 1.25) + 1024)
            self._build_bins()
            ws = C.c_void_p(self.ws.data_ptr())
            rc = L.bin_sort(self._proj, self._tm, cam, self.n, self._bins, ws, self.ws_bytes, st)
            L.check(rc)
        self.M = int(self._bins.n_dup)
        if wait_before_render is not None:
            torch.cuda.current_stream().wait_event(wait_before_render)
        L.render_fwd(self._proj, self._bins, self._tm, cam, C.c_void_p(mask.data_ptr()), self._bg, self._img, ws,
                     self.ws_bytes, st)
        return dict(C=self.img_C, N=self.img_N, D=self.img_D, A=self.img_A, Dep=self.img_Dep, T=self.img_T,
                    g=self.img_g, last=self.img_last)

    def _image_grad(self, dC, dN, dD, dA, dDep, gc_lambda, nd_div):
        ig = L.ImageGrad()
        ig.gc_lambda = float(gc_lambda)
        ig.nd_div = None if nd_div is None else nd_div.data_ptr()
        for k, t in (("dC", dC), ("dN", dN), ("dD", dD), ("dA", dA), ("dDep", dDep)):
            if t is not None:
                assert t.dtype == torch.float32 and t.is_contiguous() and t.device == self.device
            setattr(ig, k, None if t is None else t.data_ptr())
        self._keep = (dC, dN, dD, dA, dDep)
        return ig

    def backward_adam(self, state, hparams, flat, dC=None, dN=None, dD=None, dA=None, dDep=None, gc_lambda=0.0,
                      nd_div=None):
        """A7 + A8 with the Adam step fused into A8 (pgsag_render_bwd_adam): state (L.AdamState over the
        last forward's Gaussians) is updated in place; no parameter gradients are written."""
        ig = self._image_grad(dC, dN, dD, dA, dDep, gc_lambda, nd_div)
        L.render_bwd_adam(self._g, self._cam, self._proj, self._bins, self._tm, C.c_void_p(self._mask.data_ptr()),
                          self._bg, self._img, ig, self._grad, state, hparams, flat,
                          C.c_void_p(self.ws.data_ptr()), self.ws_bytes, _stream())

    def backward(self, dC=None, dN=None, dD=None, dA=None, dDep=None, gc_lambda=0.0, nd_div=None):
        """nd_div: optional device float64 scalar dividing dN and dDep (pgsag_image_grad.nd_div)."""
        ig = self._image_grad(dC, dN, dD, dA, dDep, gc_lambda, nd_div)
        L.render_bwd(self._g, self._cam, self._proj, self._bins, self._tm, C.c_void_p(self._mask.data_ptr()),
                     self._bg, self._img, ig, self._grad, C.c_void_p(self.ws.data_ptr()), self.ws_bytes, _stream())
        K3 = (self.deg + 1) ** 2 * 3
        out = dict(dmean=self.dmean, dscale=self.dscale, drot=self.drot, dopacity=self.dopacity,
                   dsh=self.dsh[:K3])
        if self._grad.absgrad2d:
            out["absgrad2d"] = self.absgrad
        if self._grad.grad2d:
            out["grad2d"] = self.grad2d
        return out

    def check_capacity(self) -> bool:
        """sync_free mode: after synchronising, True if the last view's M fitted the capacity; otherwise
        grows the entry buffers (the caller re-runs that view).  An overflowed view was rendered from
        EMPTY lists (the device-side entry count is 0, never a partial prefix) and a fused
        backward_adam of it skipped its update on the device."""
        if not self.sync_free:
            return True
        torch.cuda.current_stream().synchronize()
        self.M = int(self._m_host.item())
        if self.M <= self.capacity:
            return True
        self._alloc_bins(int(self.M * 1.25) + 1024)
        self._build_bins()
        return False

    def stats(self):
        c = self.counters.tolist() if self.counters is not None else [0, 0, 0, 0]
        return dict(M=self.M, evaluated=c[0], blended=c[1], bwd_visited=c[2])
