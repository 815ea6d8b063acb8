"""Pins of the L_GC-load oracle (NEXT-1; Eq. 9; readings R23, R24)."""
import numpy as np
import pytest
from scipy import ndimage

import oracle
from tests.helpers import all_pixels, cam_identity, full_mask
from tests.test_oracle_pins import _fd_scene


def test_gc_weights_match_scipy_sobel():
    """R23: |Sobel(gray)| (replicated borders) normalised by its mask mean, clamped to [0.1, 10];
    pinned against scipy.ndimage.sobel(mode='nearest')."""
    rng = np.random.default_rng(0)
    H, W = 23, 37
    img = rng.uniform(size=(3, H, W))
    img[:, :, 20:] += 2.0  # a vertical edge
    mask = (rng.uniform(size=(H, W)) < 0.6).astype(np.uint8)
    gray = 0.299 * img[0] + 0.587 * img[1] + 0.114 * img[2]
    mag = np.hypot(ndimage.sobel(gray, axis=0, mode="nearest"), ndimage.sobel(gray, axis=1, mode="nearest"))
    m = mag[mask != 0].mean()
    ref = np.where(mask != 0, np.clip(mag / m, 0.1, 10.0), 1.0)
    w = oracle.gc_weights(img, mask)
    np.testing.assert_allclose(w, ref, rtol=1e-12, atol=1e-12)
    # normalisation identity before clamping (SPEC gradient_weight example)
    assert abs((mag / m)[mask != 0].mean() - 1.0) < 1e-12
    # the edge column carries the largest weight
    assert int(np.argmax(w.max(axis=0))) in (19, 20)


def test_gc_weights_constant_image_floor():
    img = np.full((3, 10, 12), 0.3)
    mask = np.ones((10, 12), np.uint8)
    assert (oracle.gc_weights(img, mask) == 0.1).all()


def test_gc_load_values_and_gradient():
    """Eq. 9: population std of g/w (SPEC example ratios {1,1,3,3} -> 1), numpy.std pin, scale
    covariance, proportional null case, and dL/dg against central differences."""
    L, mu, _ = oracle.gc_load([1, 1, 3, 3], [1, 1, 1, 1])
    assert L == 1.0 and mu == 2.0
    rng = np.random.default_rng(1)
    g = rng.integers(0, 40, 200).astype(float)
    w = rng.uniform(0.1, 10, 200)
    L, mu, d = oracle.gc_load(g, w)
    assert abs(L - np.std(g / w)) < 1e-12 and abs(mu - np.mean(g / w)) < 1e-12
    assert abs(oracle.gc_load(3 * g, w)[0] - 3 * L) < 1e-9
    assert oracle.gc_load(2.5 * w, w)[0] < 1e-12
    h = 1e-6
    for k in rng.choice(200, 12, replace=False):
        gp, gm = g.copy(), g.copy()
        gp[k] += h
        gm[k] -= h
        fd = (np.std(gp / w) - np.std(gm / w)) / (2 * h)
        assert abs(fd - d[k]) <= 1e-6 * max(1.0, abs(fd)), (k, fd, d[k])


@pytest.mark.parametrize("seed,n", [(4, 2), (5, 5)])
def test_soft_count_surrogate_gradient_fd(seed, n):
    """R24: with upstream gG on the soft count sum_blended sigmoid(k (alpha - 1/255)), the double
    oracle's backward equals central finite differences of sum_p gG_p * gsoft_p(theta)."""
    g = _fd_scene(seed, n)
    W = H = 20
    cam = cam_identity(W=W, H=H, fx=20.0)
    mask = full_mask(H, W)
    pix = all_pixels(mask)
    rng = np.random.default_rng(200 + seed)
    up = np.zeros((len(pix), 10))
    up[:, 9] = rng.normal(size=len(pix))
    r = oracle.render(g, cam, mask, pix, dtype=np.float64, upstream=up)
    grads = r["grads"]

    def f():
        rr = oracle.render(g, cam, mask, pix, dtype=np.float64)
        state = (rr["g"].copy(), rr["last"].copy(), rr["id_sum"].copy(), rr["n_clamped"].copy())
        return float((rr["gsoft"] * up[:, 9]).sum()), state

    checked = 0
    for name, row0, rows in [("mean", 0, 3), ("scale", 3, 3), ("rot", 6, 4), ("opacity", 10, 1)]:
        arr = getattr(g, name)
        for k in range(rows):
            for i in range(n):
                idx = (k, i) if arr.ndim == 2 else (i,)
                x0 = arr[idx]
                hh = 1e-6 * max(1.0, abs(x0))
                arr[idx] = x0 + hh
                lp, sp = f()
                arr[idx] = x0 - hh
                lm, sm = f()
                arr[idx] = x0
                if not all(np.array_equal(a, b) for a, b in zip(sp, sm)):
                    continue
                fd = (lp - lm) / (2 * hh)
                an = grads[row0 + k, i]
                assert abs(fd - an) <= 2e-5 * max(abs(fd), 1e-3), (name, k, i, fd, an)
                checked += 1
    assert checked >= 0.8 * n * 11
    assert np.abs(grads[11:59]).max() == 0.0  # the soft count does not depend on colour
