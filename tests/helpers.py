"""Tiny hand-built scenes for the pins (no method arithmetic here)."""
import math

import numpy as np

from synth.scenes import Camera, Gaussians

SH_C0 = 0.28209479177387814  # Y_0^0 = 1/(2 sqrt(pi)), pinned against scipy in test_oracle_pins


def cam_identity(W=64, H=64, fx=64.0, fy=None, cx=None, cy=None):
    fy = fx if fy is None else fy
    cx = W / 2.0 if cx is None else cx
    cy = H / 2.0 if cy is None else cy
    return Camera(float(fx), float(fy), float(cx), float(cy), W, H, np.eye(3, dtype=np.float32),
                  np.zeros(3, np.float32))


def quat_axis_angle(axis, ang):
    axis = np.asarray(axis, float) / np.linalg.norm(axis)
    return np.array([math.cos(ang / 2), *(math.sin(ang / 2) * axis)])


def gaussians(means, scales, quats=None, opac=None, rgb=None, deg=0, sh=None, dtype=np.float64):
    """Build SoA Gaussians; rgb sets the DC term so that colour = rgb (degree-0 part)."""
    means = np.asarray(means, float).reshape(-1, 3)
    n = means.shape[0]
    scales = np.asarray(scales, float).reshape(n, 3)
    quats = np.tile([1.0, 0, 0, 0], (n, 1)) if quats is None else np.asarray(quats, float).reshape(n, 4)
    opac = np.full(n, 0.5) if opac is None else np.asarray(opac, float).reshape(n)
    K = (deg + 1) ** 2
    if sh is None:
        sh = np.zeros((K * 3, n))
        if rgb is not None:
            rgb = np.asarray(rgb, float).reshape(n, 3)
            sh[0:3] = ((rgb - 0.5) / SH_C0).T
    return Gaussians(mean=np.ascontiguousarray(means.T, dtype), scale=np.ascontiguousarray(scales.T, dtype),
                     rot=np.ascontiguousarray(quats.T, dtype), opacity=np.ascontiguousarray(opac, dtype),
                     sh=np.ascontiguousarray(sh, dtype), sh_degree=deg)


def full_mask(H, W):
    return np.ones((H, W), np.uint8)


def all_pixels(mask):
    return np.flatnonzero(mask.reshape(-1))
