"""Randomised parity sweep: many small seeded scenes that vary the knobs the fixed configs keep
constant — image size (ragged in both directions, down to a single partial tile), Gaussian
count, SH degree, scale and opacity ranges, mask density, background, camera focal length —
each checked forward (every mask pixel) and backward (upstream at every mask pixel) against
the oracle with the DESIGN.md §6 / R19 tolerances, keys and ranges bit-exact."""
import numpy as np
import pytest

import oracle
from synth import scenes as S
from tests.gpu_util import compare_grads, compare_pixels, run_gpu, upstream_at
from tests.helpers import all_pixels

pytestmark = pytest.mark.gpu


_scene = S.fuzz_scene


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("PGSAG_FUZZ_SEEDS", "64"))))
def test_fuzz_forward_backward(seed):
    sc, bg = _scene(seed)
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
    planes, per = upstream_at(pix, H, W, seed=seed, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    res = run_gpu(sc, bg=bg, upstream=planes, counters=bool(seed % 2))
    p = oracle.project(sc.gaussians, sc.camera, sc.mask, np.float32)
    tl, vl, rg = oracle.keys(p, sc.mask)
    np.testing.assert_array_equal(res["vals"], vl)
    np.testing.assert_array_equal(res["tile_keys"], tl)
    np.testing.assert_array_equal(res["ranges"], rg)
    compare_pixels(res["img"], ora0, pix, W, res["vals"], cam=sc.camera, proj=p)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per, bound=True)
    if np.abs(ora["grads"][:59]).max() > 0:
        compare_grads(res["grads"], ora["grads"], sc.gaussians.sh_degree, bound=ora["bound"])


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_sync_free_sort_equals_sync(seed):
    """pgsag_bin_sort_async gives bitwise the same lists / ranges / forward images as the
    synchronising sort on random scenes (tight capacity: the sizing path is exercised too)."""
    import torch
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
    sc, bg = _scene(100 + seed)
    H, W = sc.mask.shape
    g = GaussianTensors.from_numpy(sc.gaussians)
    cam = camera_from(sc.camera)
    mask = torch.from_numpy(np.ascontiguousarray(sc.mask)).cuda()
    a = Rasterizer(g.n, W, H, g.sh_degree)
    a.forward(g, cam, mask, bg)
    b = Rasterizer(g.n, W, H, g.sh_degree, capacity=max(a.M, 1), sync_free=True)
    b.forward(g, cam, mask, bg)
    assert b.check_capacity() and b.M == a.M
    M = a.M
    assert torch.equal(a.vals[:M], b.vals[:M]) and torch.equal(a.ranges, b.ranges)
    for k in ("img_C", "img_N", "img_D", "img_T", "img_g", "img_last", "img_Dep"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_rgb_loss(seed):
    """Masked L1 + SSIM value and gradient on random sizes (down to 3 px), mask densities and
    image statistics against the oracle (tolerances of R28)."""
    import torch
    from paper_2501_01677_b200 import _lib as L
    rng = np.random.default_rng(300 + seed)
    H, W = int(rng.integers(3, 80)), int(rng.integers(3, 120))
    I = rng.uniform(0, 1, (3, H, W)).astype(np.float32)
    if rng.uniform() < 0.5:  # smooth images: small variances, the cancellation-prone case
        I = np.clip(0.5 + 0.05 * np.cumsum(rng.normal(0, 0.1, (3, H, W)), axis=2), 0, 1).astype(np.float32)
    C = np.clip(I + rng.normal(0, float(rng.uniform(0.001, 0.2)), I.shape), 0, 1).astype(np.float32)
    mask = (rng.uniform(size=(H, W)) < float(rng.uniform(0.05, 1.0))).astype(np.uint8)
    mask[0, 0] = 1
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    c_, i_, m_ = t(C), t(I), t(mask)
    loss = torch.zeros(6, dtype=torch.float64, device="cuda")
    dC = torch.full((3, H, W), -7.0, device="cuda")
    nb = L.rgb_loss_workspace_size(W, H)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    L.rgb_loss(c_.data_ptr(), i_.data_ptr(), m_.data_ptr(), W, H, 1.0, loss.data_ptr(), dC.data_ptr(),
               ws.data_ptr(), nb, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    Lr, L1, Sm, dref = oracle.rgb_loss(C.astype(np.float64), I.astype(np.float64), mask, grads=True)
    lo = loss.cpu().numpy()
    assert lo[5] == mask.sum() and abs(lo[1] - L1) <= 1e-6 * abs(L1) + 1e-9 and abs(lo[2] - Sm) <= 1e-5
    got = dC.cpu().numpy().astype(np.float64)
    on = np.broadcast_to(mask != 0, got.shape)
    err = np.abs(got - dref)[on] / np.maximum(np.abs(dref[on]), 1e-2 * np.abs(dref).max())
    assert err.max() <= 2e-3, err.max()
    assert (got[~on] == -7.0).all()
