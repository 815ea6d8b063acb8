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


def _scene(seed):
    rng = np.random.default_rng(1000 + seed)
    W, H = int(rng.integers(5, 90)), int(rng.integers(5, 70))
    n = int(rng.integers(1, 700))
    deg = int(rng.integers(0, 4))
    g = S.random_gaussians(rng, n, [-1.5, -1.2, 1.5], [1.5, 1.2, 7.0],
                           s_lo=float(rng.uniform(0.005, 0.05)), s_hi=float(rng.uniform(0.1, 0.8)),
                           o_lo=float(rng.uniform(0.0, 0.3)), o_hi=float(rng.uniform(0.5, 1.0)), deg=deg,
                           sh_std=float(rng.uniform(0.1, 0.6)))
    f = float(rng.uniform(0.6, 1.6)) * max(W, H)
    cam = S.Camera(f, f * float(rng.uniform(0.8, 1.25)), W / 2.0 + float(rng.uniform(-3, 3)),
                   H / 2.0 + float(rng.uniform(-3, 3)), W, H, np.eye(3, dtype=np.float32), np.zeros(3, np.float32))
    mask = (rng.uniform(size=(H, W)) < float(rng.uniform(0.05, 1.0))).astype(np.uint8)
    if not mask.any():
        mask[H // 2, W // 2] = 1
    bg = tuple(float(x) for x in rng.uniform(0, 1, 3)) if rng.uniform() < 0.5 else (0.0, 0.0, 0.0)
    return S.Scene(f"fuzz{seed}", g, cam, mask, seed=seed), bg


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("PGSAG_FUZZ_SEEDS", "64"))))
def test_fuzz_forward_backward(seed):
    sc, bg = _scene(seed)
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
    planes, per = upstream_at(pix, H, W, seed=seed, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    res = run_gpu(sc, bg=bg, upstream=planes, counters=bool(seed % 2))
    p = oracle.project(sc.gaussians, sc.camera, sc.mask)
    tl, vl, rg = oracle.keys(p, sc.mask)
    np.testing.assert_array_equal(res["vals"], vl)
    np.testing.assert_array_equal(res["tile_keys"], tl)
    np.testing.assert_array_equal(res["ranges"], rg)
    compare_pixels(res["img"], ora0, pix, W, res["vals"], cam=sc.camera)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per, bound=True)
    if np.abs(ora["grads"][:59]).max() > 0:
        compare_grads(res["grads"], ora["grads"], sc.gaussians.sh_degree, bound=ora["bound"])
