"""Parity on code paths the synthetic workloads rarely reach: the 0.99 alpha clamp (R6, R16),
SH degrees 0-2 (R12), the Jacobian clamp of splats outside the frustum (R9), very large
multi-tile splats (long per-tile lists, many batches), and non-zero backgrounds."""
import numpy as np
import pytest

import oracle
from synth import scenes as S
from tests.gpu_util import compare_grads, compare_pixels, run_gpu, upstream_at
from tests.helpers import all_pixels, cam_identity, gaussians

pytestmark = pytest.mark.gpu


def _check(sc, bg=(0.2, 0.4, 0.1), seed=1):
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
    planes, per = upstream_at(pix, H, W, seed=seed, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    res = run_gpu(sc, bg=bg, upstream=planes)
    compare_pixels(res["img"], ora0, pix, W, res["vals"], cam=sc.camera)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per)
    compare_grads(res["grads"], ora["grads"], sc.gaussians.sh_degree)
    return ora0


def test_alpha_clamp_path():
    """Opacities in [0.97, 1.0]: many pairs reach o*rho > 0.99 (clamped alpha, zero gradient
    through the clamp, R16)."""
    sc = S.config1(seed=21, n=300)
    rng = np.random.default_rng(21)
    sc.gaussians.opacity[:] = rng.uniform(0.995, 1.0, sc.gaussians.n).astype(np.float32)
    sc.gaussians.scale *= np.float32(4.0)  # wide splats: rho > 0.99 on a disc of a few pixels each
    ora = _check(sc)
    assert ora["n_clamped"].sum() > 30


@pytest.mark.parametrize("deg", [0, 1, 2])
def test_sh_degrees(deg):
    sc = S.config1(seed=30 + deg, n=500, sh_degree=deg)
    _check(sc)


def test_jacobian_clamp_and_large_splats():
    """Large splats whose centres lie outside the 1.3 x half-FoV window (x/z clamped inside J,
    R9) but whose footprints still cover the image, plus splats covering most tiles."""
    rng = np.random.default_rng(40)
    n_out, n_big = 40, 30
    W = H = 48
    cam = cam_identity(W=W, H=H, fx=40.0)
    z = rng.uniform(2.0, 4.0, n_out)
    side = rng.choice([-1, 1], n_out)
    x = side * z * rng.uniform(0.8, 1.1)  # |x/z| beyond 1.3 * (0.5 W / fx) = 0.78
    y = rng.uniform(-0.5, 0.5, n_out) * z
    means = np.concatenate([np.c_[x, y, z], np.c_[rng.uniform(-0.3, 0.3, n_big), rng.uniform(-0.3, 0.3, n_big),
                                                  rng.uniform(3, 6, n_big)]])
    scales = np.concatenate([rng.uniform(0.3, 0.8, (n_out, 3)), rng.uniform(0.3, 1.2, (n_big, 3))])
    scales[np.arange(len(scales)), rng.integers(0, 3, len(scales))] *= 0.1
    n = n_out + n_big
    g = gaussians(means, scales, rng.normal(size=(n, 4)), rng.uniform(0.05, 0.6, n), deg=3,
                  sh=rng.normal(0, 0.3, (48, n)))
    mask = (rng.uniform(size=(H, W)) < 0.7).astype(np.uint8)
    sc = S.Scene("clamp", g, cam, mask)
    p = oracle.project(g, cam, mask)
    live = (p["flags"] & 15) == 15
    assert ((p["flags"] & (16 | 32)) != 0)[live].sum() >= 5  # clamped Jacobians among emitting splats
    assert p["tiles"].max() >= 9
    _check(sc)


@pytest.mark.parametrize("absgrad", [True, False])
def test_screen_space_gradients_and_absgrad(absgrad):
    """A7's 14 per-Gaussian screen-space values (exported grad2d: du dv dca dcb dcc dop drgb dncam ddist
    absgrad) and the absgrad2d output against the oracle's rows 59-72.  With absgrad off, A7 takes its
    sums-only path for (du, dv) and the export is requested without it (row 13 then still exported)."""
    import torch
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
    sc = S.config1(seed=77, n=700)
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    planes, per = upstream_at(pix, H, W, seed=77, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    ref = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, upstream=per)["grads"]
    g = GaussianTensors.from_numpy(sc.gaussians)
    r = Rasterizer(g.n, W, H, g.sh_degree, absgrad=absgrad)
    r.export_grad2d(absgrad)
    r.forward(g, camera_from(sc.camera), torch.from_numpy(np.ascontiguousarray(sc.mask)).cuda())
    out = r.backward(**{k: torch.from_numpy(v).cuda() for k, v in planes.items()})
    torch.cuda.synchronize()
    got = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in out.items()}
    compare_grads(got, ref, sc.gaussians.sh_degree)
    if absgrad:
        g2 = r.grad2d.cpu().numpy().astype(np.float64)
        for c in range(14):
            a, b = g2[c], ref[59 + c]
            scale = max(np.abs(b).max(), 1e-30)
            assert (np.abs(a - b) <= 1e-3 * np.maximum(np.abs(b), 1e-2 * scale)).all(), c
        assert np.allclose(got["absgrad2d"], ref[72], rtol=1e-3, atol=1e-5 * np.abs(ref[72]).max())
    else:
        assert "absgrad2d" not in got
