"""Pins of the L_ban oracle (NEXT-2; Eq. 8, P:153 normal from depth; R25-R27)."""
import math

import numpy as np
import pytest
from scipy import ndimage

import oracle
from tests.helpers import cam_identity


@pytest.mark.parametrize("r", [1, 2])
def test_boundary_band_vs_scipy(r):
    """R25: MB = dilation XOR erosion with a (2r+1)^2 square, zero outside the image."""
    rng = np.random.default_rng(r)
    m = ndimage.binary_opening(rng.uniform(size=(40, 50)) < 0.55, iterations=1)
    se = np.ones((2 * r + 1, 2 * r + 1), bool)
    ref = ndimage.binary_dilation(m, se) ^ ndimage.binary_erosion(m, se, border_value=0)
    np.testing.assert_array_equal(oracle.boundary_band(m.astype(np.uint8), r), ref.astype(np.uint8))


def test_boundary_band_special_cases():
    """SPEC extract_boundary examples: empty mask -> empty band; full mask -> border frame of
    width r; a w x h rectangle, r = 1 -> 2 (2w + 2h) band pixels (square SE)."""
    assert oracle.boundary_band(np.zeros((9, 11), np.uint8)).sum() == 0
    full = oracle.boundary_band(np.ones((9, 11), np.uint8), 2)
    frame = np.ones((9, 11), np.uint8)
    frame[2:-2, 2:-2] = 0
    np.testing.assert_array_equal(full, frame)
    m = np.zeros((20, 30), np.uint8)
    w, h = 9, 6
    m[5:5 + h, 7:7 + w] = 1
    assert oracle.boundary_band(m, 1).sum() == 2 * (2 * w + 2 * h)


def plane_depth(cam, W, H, n, d):
    """Depth (camera z) of the plane n.X = d along each pixel-centre ray r = K^-1 p~."""
    x, y = np.meshgrid(np.arange(W) + 0.5, np.arange(H) + 0.5)
    r = np.stack([(x - cam.cx) / cam.fx, (y - cam.cy) / cam.fy, np.ones_like(x)])
    return d / np.tensordot(n, r, axes=1)


def test_fronto_parallel_depth_gives_camera_facing_normal():
    """P:153 / S:305-313: a constant-depth plane has n_depth = (0, 0, -1) at every interior pixel:
    L_ban = 0 with N = (0,0,-1), and every term is |(0,0,-1)-(0,0,1)|^2 = 4 with N flipped."""
    W, H = 24, 18
    cam = cam_identity(W=W, H=H, fx=20.0)
    mask = np.ones((H, W), np.uint8)
    band = np.zeros((H, W), np.uint8)
    Dep = np.full((H, W), 5.0)
    N = np.zeros((3, H, W))
    N[2] = -0.7  # unnormalised (R26: n_r = N / |N|)
    s, c = oracle.ban_loss(cam, mask, band, N, Dep)
    assert c == (W - 2) * (H - 2) and s < 1e-20
    s, c = oracle.ban_loss(cam, mask, band, -N, Dep)
    assert abs(s - 4 * c) < 1e-9


def test_tilted_plane_normal_matches_analytic():
    """A 45-degree plane through (0, 0, 5): n_depth equals the analytic (camera-facing) plane
    normal, so L_ban = 0 when N is that normal."""
    W, H = 30, 22
    cam = cam_identity(W=W, H=H, fx=25.0)
    n = np.array([0.0, -math.sin(math.pi / 4), math.cos(math.pi / 4)])
    n = -n if n @ np.array([0, 0, 5.0]) > 0 else n
    d = n @ np.array([0, 0, 5.0])
    Dep = plane_depth(cam, W, H, n, d)
    mask = np.ones((H, W), np.uint8)
    N = np.broadcast_to(n[:, None, None], (3, H, W)).copy()
    s, c = oracle.ban_loss(cam, mask, np.zeros_like(mask), N, Dep)
    assert c > 0 and s < 1e-18


def test_band_weighting_arithmetic():
    """Eq. 8 weights (R27): with every term equal to 4, L = 4 sum_p w_p / #valid with w = 0.1 on
    the boundary band inside the mask, 1 elsewhere (S:391 example generalised)."""
    W, H = 26, 20
    cam = cam_identity(W=W, H=H, fx=20.0)
    mask = np.zeros((H, W), np.uint8)
    mask[3:17, 4:22] = 1
    band = oracle.boundary_band(mask, 1)
    Dep = np.full((H, W), 3.0)
    N = np.zeros((3, H, W))
    N[2] = 1.0
    s, c = oracle.ban_loss(cam, mask, band, N, Dep)
    valid = np.zeros((H, W), bool)
    valid[4:16, 5:21] = True  # interior: all four neighbours inside the mask
    w = np.where(band[valid] != 0, 0.1, 1.0)
    assert c == valid.sum()
    assert abs(s - 4 * w.sum()) < 1e-9


def test_ban_gradients_fd():
    """Exact reverse mode of lambda * sum / count w.r.t. N and Dep vs central differences."""
    rng = np.random.default_rng(9)
    W, H = 14, 11
    cam = cam_identity(W=W, H=H, fx=12.0)
    mask = np.ones((H, W), np.uint8)
    mask[:, :2] = 0
    band = oracle.boundary_band(mask, 1)
    x, y = np.meshgrid(np.arange(W), np.arange(H))
    Dep = 4.0 + 0.3 * np.sin(x / 3.0) + 0.2 * np.cos(y / 2.0) + 0.01 * rng.normal(size=(H, W))
    N = rng.normal(size=(3, H, W))
    N[2] -= 2.0
    lam = 0.37
    s, c, dN, dD = oracle.ban_loss(cam, mask, band, N, Dep, lam=lam, grads=True)
    f = lambda NN, DD: lam * oracle.ban_loss(cam, mask, band, NN, DD)[0] / c
    h = 1e-6
    for _ in range(25):
        k, j, i = rng.integers(0, 3), rng.integers(0, H), rng.integers(0, W)
        Np, Nm = N.copy(), N.copy()
        Np[k, j, i] += h
        Nm[k, j, i] -= h
        fd = (f(Np, Dep) - f(Nm, Dep)) / (2 * h)
        assert abs(fd - dN[k, j, i]) <= 1e-6 * max(1.0, abs(fd))
        Dp, Dm = Dep.copy(), Dep.copy()
        Dp[j, i] += h
        Dm[j, i] -= h
        fd = (f(N, Dp) - f(N, Dm)) / (2 * h)
        assert abs(fd - dD[j, i]) <= 1e-6 * max(1.0, abs(fd))
