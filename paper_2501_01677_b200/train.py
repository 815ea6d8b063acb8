"""NEXT-3: one masked training iteration of a sub-region (Eq. 10-11) through the C ABI.

    L = (1 - lambda) (L_rgb + lambda3 L_s + lambda4 L_ban) + lambda L_GC-load
    lambda = 0.41, lambda3 = 100, lambda4 = 0.01

Per iteration: pgsag_preprocess / bin_sort / render_fwd (A0-A6, with the Eq. 9 statistics when
gc weights are given) -> pgsag_rgb_loss (weight 1 - lambda into dC) -> pgsag_ban_loss (weight
(1 - lambda) lambda4 into dN, dDep) -> pgsag_render_bwd (A7/A8, gc_lambda = lambda) ->
pgsag_adam_step (L_s with weight (1 - lambda) lambda3).  The multi-view PGSR terms (lambda1,
lambda2) are out of scope.  This module only allocates and marshals pointers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib as L
from .raster import GaussianTensors, Rasterizer, _stream

LAMBDA, LAMBDA3, LAMBDA4 = 0.41, 100.0, 0.01


@dataclass
class AdamConfig:
    """3DGS's default learning rates (R30); lr_mean is usually scaled by the scene extent."""
    lr_mean: float = 1.6e-4
    lr_scale: float = 5e-3
    lr_rot: float = 1e-3
    lr_opacity: float = 0.05
    lr_sh_dc: float = 2.5e-3
    lr_sh_rest: float = 2.5e-3 / 20
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15


class Trainer:
    """Owns the optimiser state of one sub-region's Gaussians (g is updated in place)."""

    def __init__(self, raster: Rasterizer, g: GaussianTensors, cfg: AdamConfig | None = None, lam=LAMBDA,
                 lam3=LAMBDA3, lam4=LAMBDA4, boundary_w=0.1):
        self.r, self.g, self.cfg = raster, g, cfg or AdamConfig()
        self.lam, self.lam3, self.lam4, self.bw = float(lam), float(lam3), float(lam4), float(boundary_w)
        dev, n, H, W = raster.device, g.n, raster.H, raster.W
        K3 = (g.sh_degree + 1) ** 2 * 3
        # raw parameters (one-time initialisation from the activated values)
        self.log_scale = torch.log(g.scale).contiguous()
        self.logit_opacity = torch.logit(g.opacity.double()).float().contiguous()
        self.m = torch.zeros(11 + K3, max(n, 1), dtype=torch.float32, device=dev)
        self.v = torch.zeros_like(self.m)
        self.dC = torch.zeros(3, H, W, dtype=torch.float32, device=dev)
        self.dN = torch.zeros(3, H, W, dtype=torch.float32, device=dev)
        self.dDep = torch.zeros(H, W, dtype=torch.float32, device=dev)
        self.rgb_ws_bytes = L.rgb_loss_workspace_size(W, H)
        self.rgb_ws = torch.empty(self.rgb_ws_bytes, dtype=torch.uint8, device=dev)
        self.loss_rgb = torch.zeros(6, dtype=torch.float64, device=dev)
        self.loss_ban = torch.zeros(2, dtype=torch.float64, device=dev)
        self.loss_flat = torch.zeros(1, dtype=torch.float64, device=dev)
        st = L.AdamState()
        st.mean, st.scale, st.rot = g.mean.data_ptr(), g.scale.data_ptr(), g.rot.data_ptr()
        st.opacity, st.sh = g.opacity.data_ptr(), g.sh.data_ptr()
        st.log_scale, st.logit_opacity = self.log_scale.data_ptr(), self.logit_opacity.data_ptr()
        st.m, st.v = self.m.data_ptr(), self.v.data_ptr()
        self._state = st
        self.t = 0
        self.used_ban = self.used_gc = False

    def hparams(self) -> L.AdamHparams:
        c, hp = self.cfg, L.AdamHparams()
        hp.lr_mean, hp.lr_scale, hp.lr_rot, hp.lr_opacity = c.lr_mean, c.lr_scale, c.lr_rot, c.lr_opacity
        hp.lr_sh_dc, hp.lr_sh_rest, hp.beta1, hp.beta2, hp.eps = c.lr_sh_dc, c.lr_sh_rest, c.beta1, c.beta2, c.eps
        hp.flatten_weight = (1.0 - self.lam) * self.lam3
        hp.step = self.t
        return hp

    def step(self, cam, mask: torch.Tensor, target: torch.Tensor, gc_w: torch.Tensor | None = None,
             band: torch.Tensor | None = None, bg=(0.0, 0.0, 0.0)):
        """One iteration on one view; returns nothing (losses stay on the device, see losses())."""
        r = self.r
        self.t += 1
        st = _stream()
        p = lambda t: C.c_void_p(t.data_ptr())
        r.forward(self.g, cam, mask, bg, gc_w=gc_w)
        assert target.dtype == torch.float32 and target.is_contiguous() and tuple(target.shape) == (3, r.H, r.W)
        L.rgb_loss(p(r.img_C), p(target), p(mask), r.W, r.H, 1.0 - self.lam, p(self.loss_rgb), p(self.dC),
                   p(self.rgb_ws), self.rgb_ws_bytes, st)
        self.used_ban = band is not None
        if self.used_ban:
            self.dN.zero_()
            self.dDep.zero_()
            L.ban_loss(cam, p(mask), p(band), p(r.img_N), p(r.img_Dep), self.bw, (1.0 - self.lam) * self.lam4, 1,
                       p(self.loss_ban), p(self.dN), p(self.dDep), st)
        self.used_gc = gc_w is not None
        r.backward(dC=self.dC, dN=self.dN if self.used_ban else None, dDep=self.dDep if self.used_ban else None,
                   gc_lambda=self.lam if self.used_gc else 0.0)
        L.adam_step(self.g.n, self.g.sh_degree, r._grad, self._state, self.hparams(), p(self.loss_flat), st)

    def losses(self) -> dict:
        """Host read of the last iteration's terms and the Eq. 11 total."""
        rgb = self.loss_rgb.tolist()
        Ls = float(self.loss_flat.item())
        ban = self.loss_ban.tolist()
        Lban = ban[0] / ban[1] if self.used_ban and ban[1] > 0 else 0.0
        Lgc = self.r.gc_load()[0] if self.used_gc else 0.0
        total = (1 - self.lam) * (rgb[0] + self.lam3 * Ls + self.lam4 * Lban) + self.lam * Lgc
        return dict(total=total, rgb=rgb[0], l1=rgb[1], ssim=rgb[2], flat=Ls, ban=Lban, gc_load=Lgc)
