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
from . import shard
from .raster import GaussianTensors, Rasterizer, _stream

LAMBDA, LAMBDA3, LAMBDA4 = 0.41, 100.0, 0.01


@dataclass
class DensifyConfig:
    """3DGS adaptive density control (R31): 3DGS's defaults; dense_limit = percent_dense (0.01) x the
    scene extent."""
    grad_threshold: float = 2e-4
    dense_limit: float = 0.01
    min_opacity: float = 0.005
    seed: int = 1677


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
                 lam3=LAMBDA3, lam4=LAMBDA4, boundary_w=0.1, fused=True):
        """fused: single-rank steps apply Adam inside A8 (pgsag_render_bwd_adam); False runs A8 then
        pgsag_adam_step (bitwise the same result; the gradients land in raster.dmean etc.)."""
        self.r, self.g, self.cfg = raster, g, cfg or AdamConfig()
        self.fused = bool(fused)
        self.lam, self.lam3, self.lam4, self.bw = float(lam), float(lam3), float(lam4), float(boundary_w)
        dev, n, H, W = raster.device, g.n, raster.H, raster.W
        K3 = (g.sh_degree + 1) ** 2 * 3
        # raw parameters (one-time initialisation from the activated values, pgsag_adam_init)
        self.log_scale = torch.empty(3, max(n, 1), dtype=torch.float32, device=dev)
        self.logit_opacity = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
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
        L.adam_init(n, st, _stream())
        self.loss_all = torch.zeros(1, dtype=torch.float64, device=dev)  # Eq. 11's total (pgsag_loss_total)
        self.t = 0
        self.used_ban = self.used_gc = False
        self._alloc_stats(n)

    def _alloc_stats(self, n):
        dev = self.r.device
        self.accum = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
        self.count = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)

    def hparams(self) -> L.AdamHparams:
        c, hp = self.cfg, L.AdamHparams()
        hp.lr_mean, hp.lr_scale, hp.lr_rot, hp.lr_opacity = c.lr_mean, c.lr_scale, c.lr_rot, c.lr_opacity
        hp.lr_sh_dc, hp.lr_sh_rest, hp.beta1, hp.beta2, hp.eps = c.lr_sh_dc, c.lr_sh_rest, c.beta1, c.beta2, c.eps
        hp.flatten_weight = (1.0 - self.lam) * self.lam3
        hp.step = self.t
        return hp

    def _side(self):
        if getattr(self, "_side_stream", None) is None:
            self._side_stream = torch.cuda.Stream(device=self.r.device)
        return self._side_stream

    def step(self, cam, mask: torch.Tensor, target: torch.Tensor, gc_w: torch.Tensor | None = None,
             band: torch.Tensor | None = None, bg=(0.0, 0.0, 0.0), dp_group=None, gc_ready=None):
        """One iteration on one view; returns nothing (losses stay on the device, see losses()).
        dp_group: process group of the ranks training the same sub-region view-parallel (NEXT-4);
        their parameter gradients are averaged before the (identical) Adam step.  L_ban runs on a
        side stream concurrently with L_rgb (both only read A6's outputs).  gc_ready: event after
        which gc_w / band are valid (A6 waits for it)."""
        r = self.r
        if (dp_group is not None or not self.fused) and r.sync_free:
            # the separate pgsag_adam_step (averaged / unfused path) has no view-overflow guard
            raise ValueError("dp_group / fused=False steps need a synchronising rasterizer (sync_free=False)")
        self.t += 1
        st = _stream()
        main = torch.cuda.current_stream()
        p = lambda t: C.c_void_p(t.data_ptr())
        r.forward(self.g, cam, mask, bg, gc_w=gc_w, wait_before_render=gc_ready)
        assert target.dtype == torch.float32 and target.is_contiguous() and tuple(target.shape) == (3, r.H, r.W)
        self.used_ban = band is not None
        if self.used_ban:
            side = self._side()
            ev_fwd = torch.cuda.Event()
            ev_fwd.record(main)
            with torch.cuda.stream(side):
                side.wait_event(ev_fwd)
                self.dN.zero_()
                self.dDep.zero_()
                # one pass: loss sums + the gradient of the SUM; A7 divides dN / dDep by the term
                # count (pgsag_image_grad.nd_div), which makes it the gradient of the mean (R27)
                L.ban_loss(cam, p(mask), p(band), p(r.img_N), p(r.img_Dep), self.bw, (1.0 - self.lam) * self.lam4,
                           0, p(self.loss_ban), p(self.dN), p(self.dDep), C.c_void_p(side.cuda_stream))
                ev_ban = torch.cuda.Event()
                ev_ban.record(side)
        L.rgb_loss(p(r.img_C), p(target), p(mask), r.W, r.H, 1.0 - self.lam, p(self.loss_rgb), p(self.dC),
                   p(self.rgb_ws), self.rgb_ws_bytes, st)
        if self.used_ban:
            main.wait_event(ev_ban)
        self.used_gc = gc_w is not None
        r._grad.densify_accum, r._grad.densify_count = self.accum.data_ptr(), self.count.data_ptr()
        up = dict(dC=self.dC, dN=self.dN if self.used_ban else None, dDep=self.dDep if self.used_ban else None,
                  gc_lambda=self.lam if self.used_gc else 0.0, nd_div=self.loss_ban[1:] if self.used_ban else None)
        try:
            if dp_group is None and self.fused:  # A8 applies the Adam step: no gradient round trip
                r.backward_adam(self._state, self.hparams(), p(self.loss_flat), **up)
            else:
                r.backward(**up)
        finally:
            r._grad.densify_accum = r._grad.densify_count = None
        if dp_group is not None or not self.fused:
            if dp_group is not None:
                K3 = (self.g.sh_degree + 1) ** 2 * 3
                shard.allreduce_mean([r.dmean, r.dscale, r.drot, r.dopacity, r.dsh[:K3]], dp_group)
            L.adam_step(self.g.n, self.g.sh_degree, r._grad, self._state, self.hparams(), p(self.loss_flat), st)

    def step_photo(self, cam, mask: torch.Tensor, target: torch.Tensor, bg=(0.0, 0.0, 0.0), dp_group=None,
                   band_radius=1):
        """step() with the Eq. 9 weights and the boundary band derived from this view's photo and
        mask on the side stream, concurrently with A0-A5 (A6 waits for them)."""
        r, dev = self.r, self.r.device
        if getattr(self, "_gc_w", None) is None:
            self._gc_w = torch.empty(r.H, r.W, dtype=torch.float32, device=dev)
            self._band = torch.empty(r.H, r.W, dtype=torch.uint8, device=dev)
            self._gc_ws_bytes = L.workspace_size(0, r.W, r.H, 0)
            self._gc_ws = torch.empty(max(self._gc_ws_bytes, 256), dtype=torch.uint8, device=dev)
        side, main = self._side(), torch.cuda.current_stream()
        p = lambda t: C.c_void_p(t.data_ptr())
        ev_in = torch.cuda.Event()
        ev_in.record(main)
        with torch.cuda.stream(side):
            side.wait_event(ev_in)
            ss = C.c_void_p(side.cuda_stream)
            L.gc_weights(p(target), p(mask), r.W, r.H, p(self._gc_w), p(self._gc_ws), self._gc_ws_bytes, ss)
            L.boundary_band(p(mask), r.W, r.H, band_radius, p(self._band), ss)
            ev_gc = torch.cuda.Event()
            ev_gc.record(side)
        self.step(cam, mask, target, gc_w=self._gc_w, band=self._band, bg=bg, dp_group=dp_group, gc_ready=ev_gc)

    def losses(self) -> dict:
        """Host read of the last iteration's terms and the Eq. 11 total.  With a sync-free rasterizer
        it also checks the last view's entry capacity: overflowed = True means that view was skipped
        (empty lists, no Adam update, pgsag_render_bwd_adam) and the buffers have grown for a re-run."""
        p = lambda t: C.c_void_p(t.data_ptr())
        L.loss_total(p(self.loss_rgb), p(self.loss_flat), p(self.loss_ban) if self.used_ban else None, 1,
                     p(self.r.gc_stats) if self.used_gc else None, self.lam, self.lam3, self.lam4, p(self.loss_all),
                     _stream())
        rgb = self.loss_rgb.tolist()
        overflowed = not self.r.check_capacity()
        Ls = float(self.loss_flat.item())
        ban = self.loss_ban.tolist()
        Lban = ban[0] / ban[1] if self.used_ban and ban[1] > 0 else 0.0
        Lgc = float(self.r.gc_stats[3].item()) if self.used_gc else 0.0
        total = float(self.loss_all.item())
        return dict(total=total, rgb=rgb[0], l1=rgb[1], ssim=rgb[2], flat=Ls, ban=Lban, gc_load=Lgc,
                    overflowed=overflowed)

    # ------------------------------------------------------------ densification (R31)
    def _state_tensors(self, n, K3, dev):
        f = lambda *sh: torch.empty(*sh, dtype=torch.float32, device=dev)
        return dict(mean=f(3, n), scale=f(3, n), rot=f(4, n), opacity=f(n), sh=f(K3, n), log_scale=f(3, n),
                    logit_opacity=f(n), m=f(11 + K3, n), v=f(11 + K3, n))

    @staticmethod
    def _state_struct(t) -> L.AdamState:
        st = L.AdamState()
        for k in ("mean", "scale", "rot", "opacity", "sh", "log_scale", "logit_opacity", "m", "v"):
            setattr(st, k, t[k].data_ptr())
        return st

    def densify(self, cfg: DensifyConfig | None = None, capacity_per_gaussian=24, dp_group=None):
        """Clone / split / prune from the statistics accumulated since the last call (pgsag_densify_plan /
        _apply), then re-allocate the optimiser state and the rasterizer for the new count.  Returns
        (kept, cloned, split).  With dp_group the statistics are summed over the group first, so every
        member takes the same decisions (same seed) and stays in sync."""
        cfg = cfg or DensifyConfig()
        if dp_group is not None:
            shard.allreduce_sum([self.accum, self.count], dp_group)
        g, r, dev = self.g, self.r, self.r.device
        n, K3 = g.n, (g.sh_degree + 1) ** 2 * 3
        dp = L.DensifyParams(cfg.grad_threshold, cfg.dense_limit, cfg.min_opacity, int(cfg.seed) + self.t)
        action = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
        wsb = L.densify_workspace_size(n)
        ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
        st = _stream()
        p = lambda t: C.c_void_p(t.data_ptr())
        counts = L.densify_plan(n, p(g.scale), p(g.opacity), p(self.accum), p(self.count), dp, p(action), p(ws), wsb,
                                st)
        n_out = counts[0] + counts[1] + 2 * counts[2]
        new = self._state_tensors(max(n_out, 1), K3, dev)
        L.densify_apply(n, g.sh_degree, self._state, p(action), dp, counts, self._state_struct(new), p(ws), wsb, st)
        sl = lambda t: t[..., :n_out].contiguous() if n_out != t.shape[-1] else t
        self.g = GaussianTensors(sl(new["mean"]), sl(new["scale"]), sl(new["rot"]), sl(new["opacity"]), sl(new["sh"]),
                                 g.sh_degree)
        self.log_scale, self.logit_opacity = sl(new["log_scale"]), sl(new["logit_opacity"])
        self.m, self.v = new["m"], new["v"]
        if n_out != self.m.shape[-1]:
            self.m, self.v = self.m[:, :n_out].contiguous(), self.v[:, :n_out].contiguous()
        self._state = self._state_struct(dict(mean=self.g.mean, scale=self.g.scale, rot=self.g.rot,
                                              opacity=self.g.opacity, sh=self.g.sh, log_scale=self.log_scale,
                                              logit_opacity=self.logit_opacity, m=self.m, v=self.v))
        self.r = Rasterizer(n_out, r.W, r.H, g.sh_degree, capacity=max(1024, capacity_per_gaussian * n_out),
                            device=dev, counters=r.counters is not None, sat=r.want_sat, absgrad=r.want_absgrad,
                            sync_free=r.sync_free)
        self._alloc_stats(n_out)
        return tuple(counts)

    def reset_opacity(self, cap=0.01):
        """3DGS opacity reset (pgsag_opacity_reset)."""
        L.opacity_reset(self.g.n, self._state, cap, _stream())
