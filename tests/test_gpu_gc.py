"""NEXT-1 (L_GC-load, Eq. 9; readings R23, R24) through the C ABI vs the oracle:
Eq. 9 weights, the statistics fused into A6's epilogue, and the soft-count surrogate
gradient inside A7."""
import numpy as np
import pytest
import torch

import oracle
from synth import scenes as S
from tests.gpu_util import compare_grads, run_gpu
from tests.helpers import all_pixels
from tests.test_gpu_parity import ragged_scene
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

pytestmark = pytest.mark.gpu


def _setup(sc, seed):
    H, W = sc.mask.shape
    img = S.reference_image(H, W, seed)
    g = GaussianTensors.from_numpy(sc.gaussians)
    r = Rasterizer(g.n, W, H, g.sh_degree)
    mask = torch.from_numpy(sc.mask).cuda()
    w = r.gc_weights(torch.from_numpy(img).cuda(), mask)
    torch.cuda.synchronize()
    return img, g, r, mask, w


@pytest.mark.parametrize("name", ["C1", "ragged"])
def test_gc_weights_and_fused_stats(name):
    sc = S.config1() if name == "C1" else ragged_scene()
    img, g, r, mask, w = _setup(sc, 31)
    w_ref = oracle.gc_weights(img, sc.mask)
    np.testing.assert_allclose(w.cpu().numpy(), w_ref, rtol=2e-5, atol=1e-6)
    r.forward(g, camera_from(sc.camera), mask, gc_w=w)
    torch.cuda.synchronize()
    L, mu, n = r.gc_load()
    pix = all_pixels(sc.mask)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    Lr, mur, _ = oracle.gc_load(ora["g"].astype(np.float64), w_ref.reshape(-1)[pix])
    assert n == len(pix)
    assert abs(mu - mur) <= 1e-5 * max(1.0, abs(mur))
    assert abs(L - Lr) <= 1e-4 * max(1.0, abs(Lr))


@pytest.mark.parametrize("name", ["C1", "ragged"])
def test_gc_surrogate_gradient(name):
    """lambda * L_GC-load alone as the loss: A7/A8 vs the oracle backward with upstream
    dL/d(soft count) = lambda * (r - mean) / (N L w) (R24); the oracle side is an all-oracle chain
    (its own Eq. 9 weights, its own render's counts g)."""
    sc = S.config1() if name == "C1" else ragged_scene()
    img, g, r, mask, w = _setup(sc, 32)
    lam = 0.41  # Eq. 11's lambda
    r.forward(g, camera_from(sc.camera), mask, gc_w=w)
    grads = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in r.backward(gc_lambda=lam).items()}
    torch.cuda.synchronize()
    pix = all_pixels(sc.mask)
    w_px = oracle.gc_weights(img, sc.mask).astype(np.float64).reshape(-1)[pix]  # all-oracle chain
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    _, _, dLdg = oracle.gc_load(ora0["g"].astype(np.float64), w_px)
    up = np.zeros((len(pix), 10))
    up[:, 9] = lam * dLdg
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, upstream=up)
    compare_grads(grads, ora["grads"], sc.gaussians.sh_degree)
    assert np.abs(grads["dsh"]).max() == 0.0  # the surrogate does not touch colour


def test_gc_weights_full_resolution():
    """Eq. 9 weights at the paper's full image size (5472x3648, the C3/C4 frame) on a blocky mask,
    in the launch configuration the training iteration uses."""
    from paper_2501_01677_b200 import _lib as L
    H, W = 3648, 5472
    rng = np.random.default_rng(77)
    img = S.reference_image(H, W, 77)
    mask = np.zeros((H, W), np.uint8)
    for _ in range(40):
        y, x = rng.integers(0, H), rng.integers(0, W)
        mask[y:y + rng.integers(50, 900), x:x + rng.integers(50, 1200)] = 1
    w_ref = oracle.gc_weights(img, mask)
    m = torch.from_numpy(mask).cuda()
    w = torch.empty(H, W, device="cuda")
    nb = L.workspace_size(1, W, H, 0)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    img_d = torch.from_numpy(img).cuda()  # keep a reference until the kernel has run
    L.gc_weights(img_d.data_ptr(), m.data_ptr(), W, H, w.data_ptr(), ws.data_ptr(), nb,
                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    # float32 Sobel components are 6-term sums of values <= 1 (absolute error <= ~8 ulp(1) = 5e-7); divided
    # by the mean magnitude (~0.1 here) that is <= 5e-6 absolute on w, plus 2e-5 relative for the mean
    np.testing.assert_allclose(w.cpu().numpy(), w_ref, rtol=2e-5, atol=1e-5)
