"""CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bars (BASELINE.json north_star): keys, sorted order, ranges,
tiles_touched, flags, rects and the whole A1 key path bit-exact; composited
C/N/D/A/T within 1e-4 abs (1e-4 rel for the unbiased depth), g exact except at
pixels the oracle flags as within rounding of a decision threshold (R18);
gradients within 1e-3 relative.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import scenes as S
from tests.gpu_util import compare_grads, compare_pixels, run_gpu, upstream_at
from tests.helpers import all_pixels, cam_identity, full_mask, gaussians

pytestmark = pytest.mark.gpu


def ragged_scene(seed=11, n=2000, W=100, H=75):
    """Random scene on a 100x75 image: 7x5 tiles with a ragged right/bottom tail."""
    sc = S.config1(seed=seed, n=n, W=W, H=H)
    sc.camera.fx = sc.camera.fy = 80.0
    return sc


SCENES = {
    "C1": lambda: S.config1(),
    "ragged": lambda: ragged_scene(),
    "C2s": lambda: S.config2(n=30000),
}


def check_preprocess(sc, res):
    p = oracle.project(sc.gaussians, sc.camera, sc.mask)
    r = res["r"]
    n = sc.gaussians.n
    fl = r.flags.cpu().numpy().view(np.uint32)[:n]
    np.testing.assert_array_equal(fl, p["flags"])
    live = (p["flags"] & 15) == 15
    vis = (p["flags"] & 1) == 1
    np.testing.assert_array_equal(r.depth.cpu().numpy()[:n][vis], p["depth"][vis])
    np.testing.assert_array_equal(r.mean2d.cpu().numpy()[:n][vis], p["mean2d"][vis])
    np.testing.assert_array_equal(r.conic_o.cpu().numpy()[:n][live], p["conic_o"][live])
    np.testing.assert_array_equal(r.rect.cpu().numpy()[:n].astype(np.int32)[live], p["rect"][live])
    np.testing.assert_array_equal(r.tiles_touched.cpu().numpy().view(np.uint32)[:n], p["tiles"])
    rgbd = r.rgb_d.cpu().numpy()[:n]
    np.testing.assert_allclose(rgbd[live, :3], p["rgb"][live], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(rgbd[live, 3], p["dist"][live], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(r.ncam.cpu().numpy()[:n][live, :3], p["ncam"][live], rtol=1e-6, atol=1e-7)
    # A0
    cnt, sat = oracle.tilemask(sc.mask)
    np.testing.assert_array_equal(r.tile_cnt.cpu().numpy().reshape(cnt.shape), cnt)
    np.testing.assert_array_equal(r.sat.cpu().numpy().reshape(sat.shape), sat)
    na = int(r.n_active.item())
    np.testing.assert_array_equal(r.active.cpu().numpy()[:na], np.flatnonzero(cnt.reshape(-1) > 0))
    return p


@pytest.mark.parametrize("name", list(SCENES))
def test_preprocess_and_keys_bitexact(name):
    """A0, A1 bit-exact; A2-A5 (tile, depth, id) order and ranges bit-exact vs oracle O1-O3."""
    sc = SCENES[name]()
    res = run_gpu(sc)
    p = check_preprocess(sc, res)
    tl, vl, rg = oracle.keys(p, sc.mask)
    assert res["r"].M == len(tl)
    np.testing.assert_array_equal(res["tile_keys"], tl)
    np.testing.assert_array_equal(res["vals"], vl)
    np.testing.assert_array_equal(res["ranges"], rg)


@pytest.mark.parametrize("name", ["C1", "ragged"])
def test_forward_parity_all_pixels(name):
    """A6 vs oracle O4 on every masked pixel; masked-out pixels untouched (R14)."""
    sc = SCENES[name]()
    bg = (0.1, 0.2, 0.3)
    res = run_gpu(sc, bg=bg)
    pix = all_pixels(sc.mask)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
    errs = compare_pixels(res["img"], ora, pix, sc.camera.width, res["vals"], cam=sc.camera)
    assert errs["n_near"] <= max(2, len(pix) // 200)
    off = sc.mask.reshape(-1) == 0
    assert (res["img"]["C"].reshape(3, -1)[:, off] == -7.0).all()
    assert (res["img"]["g"].reshape(-1)[off] == -7).all()
    st = res["stats"]
    # E counts pairs the kernel evaluated after the exact warp-block cull: never more than the
    # oracle's list entries visited, and B (blended pairs) is exact.
    assert 0 < st["evaluated"] <= int(ora["evaluated"].sum())
    assert st["blended"] == int(ora["g"].sum())


def test_forward_parity_sampled_c2():
    """A6 on C2-shaped input (1080p facade scene, ragged bottom row): sampled pixels + two full tiles."""
    sc = SCENES["C2s"]()
    res = run_gpu(sc)
    W = sc.camera.width
    pix = S.sample_pixels(sc.mask, 1500, seed=5)
    ranges = res["ranges"]
    heavy = int(np.argmax(ranges[:, 1] - ranges[:, 0]))
    TX = (W + 15) // 16
    for t in (heavy, int(np.flatnonzero(ranges[:, 1] > ranges[:, 0])[-1])):
        ty, tx = divmod(t, TX)
        ii, jj = np.meshgrid(np.arange(tx * 16, min(tx * 16 + 16, W)),
                             np.arange(ty * 16, min(ty * 16 + 16, sc.camera.height)))
        tp = (jj * W + ii).reshape(-1)
        pix = np.union1d(pix, tp[sc.mask.reshape(-1)[tp] != 0])
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    compare_pixels(res["img"], ora, pix, W, res["vals"], cam=sc.camera)


@pytest.mark.parametrize("name", ["C1", "ragged"])
def test_backward_parity_all_pixels(name):
    """A7+A8 vs oracle O5+O6 (double accumulation) with random upstream at every masked pixel."""
    sc = SCENES[name]()
    H, W = sc.mask.shape
    bg = (0.3, 0.1, 0.2)
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
    planes, per = upstream_at(pix, H, W, seed=3, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    res = run_gpu(sc, bg=bg, upstream=planes)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per)
    compare_grads(res["grads"], ora["grads"], sc.gaussians.sh_degree)


def test_backward_parity_sparse_c2():
    """sparse upstream on sampled pixels of a C2-shaped scene; every Gaussian's gradient
    must match the oracle's backward over exactly those pixels."""
    sc = SCENES["C2s"]()
    H, W = sc.mask.shape
    pix = S.sample_pixels(sc.mask, 1200, seed=9)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    planes, per = upstream_at(pix, H, W, seed=4, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    res = run_gpu(sc, upstream=planes)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, upstream=per)
    compare_grads(res["grads"], ora["grads"], sc.gaussians.sh_degree)


# ------------------------------------------------------------- edge cases
def _tiny(n_g, mask=None, W=40, H=24, seed=0):
    rng = np.random.default_rng(seed)
    means = np.c_[rng.uniform(-0.6, 0.6, n_g), rng.uniform(-0.4, 0.4, n_g), rng.uniform(2, 4, n_g)]
    g = gaussians(means, np.exp(rng.uniform(-3, -1, (n_g, 3))), rng.normal(size=(n_g, 4)),
                  rng.uniform(0.1, 0.95, n_g), deg=1, sh=rng.normal(0, 0.5, (12, n_g)))
    cam = cam_identity(W=W, H=H, fx=30.0)
    return S.Scene("tiny", g, cam, full_mask(H, W) if mask is None else mask)


@pytest.mark.parametrize("case", ["empty_scene", "behind_camera", "empty_mask", "single", "full_mask"])
def test_edge_cases(case):
    if case == "empty_scene":
        sc = _tiny(0)
    elif case == "behind_camera":
        sc = _tiny(20)
        sc.gaussians.mean[2] *= -1
    elif case == "empty_mask":
        sc = _tiny(50, mask=np.zeros((24, 40), np.uint8))
    elif case == "single":
        sc = _tiny(1)
    else:
        sc = _tiny(300)
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=(0.5, 0.25, 0.125)) if len(pix) else None
    planes, per = upstream_at(pix, H, W, seed=1, ora=ora0, cam=sc.camera)
    res = run_gpu(sc, bg=(0.5, 0.25, 0.125), upstream=planes)
    if len(pix):
        ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=(0.5, 0.25, 0.125), upstream=per)
        compare_pixels(res["img"], ora, pix, W, res["vals"], cam=sc.camera)
        if sc.gaussians.n:
            compare_grads(res["grads"], ora["grads"], sc.gaussians.sh_degree)
    else:
        assert res["r"].M == 0 and int(res["r"].n_active.item()) == 0
        assert np.abs(res["grads"]["dmean"]).max(initial=0) == 0


def test_capacity_overflow_retry():
    """PGSAG_ECAPACITY reports M and the driver re-allocates; results equal an ample-capacity run."""
    sc = S.config1()
    small = run_gpu(sc, capacity=16)
    big = run_gpu(sc, capacity=1 << 20)
    assert small["r"].M == big["r"].M and small["r"].capacity >= small["r"].M
    np.testing.assert_array_equal(small["vals"], big["vals"])
    np.testing.assert_array_equal(small["img"]["C"], big["img"]["C"])


def test_determinism_forward():
    """Forward outputs are bitwise reproducible run to run (no atomics on the forward path)."""
    sc = SCENES["ragged"]()
    a, b = run_gpu(sc), run_gpu(sc)
    for k in ("C", "N", "D", "Dep", "T", "g", "last"):
        np.testing.assert_array_equal(a["img"][k], b["img"][k])


def test_masked_render_equals_unmasked_restricted():
    """Metamorphic (SURVEY §8(c) 'tiling is exact'): rendering with the building mask equals the
    full-frame render restricted to the mask pixels (masking only skips work)."""
    sc = SCENES["ragged"]()
    full = S.Scene("full", sc.gaussians, sc.camera, np.ones_like(sc.mask))
    a, b = run_gpu(sc), run_gpu(full)
    m = sc.mask.astype(bool)
    for k in ("C", "N", "D", "Dep", "T", "g"):
        x, y = a["img"][k], b["img"][k]
        if x.ndim == 3:
            np.testing.assert_array_equal(x[:, m], y[:, m])
        else:
            np.testing.assert_array_equal(x[m], y[m])


def test_counting_and_timed_variants_agree():
    """The bench times the non-counting kernel variants (kCount = false); the parity tests mostly run
    the counting ones.  Forward outputs must be bitwise equal, and the non-counting backward must
    match the oracle on its own."""
    sc = S.config1(seed=123, n=900)
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    planes, per = upstream_at(pix, H, W, seed=124, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    a = run_gpu(sc, upstream=planes, counters=True)
    b = run_gpu(sc, upstream=planes, counters=False)
    for k in ("C", "N", "D", "A", "Dep", "T", "g", "last"):
        assert np.array_equal(a["img"][k], b["img"][k]), k
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, upstream=per)
    compare_grads(b["grads"], ora["grads"], sc.gaussians.sh_degree)


def test_sync_free_bin_sort():
    """pgsag_bin_sort_async (no host synchronisation) gives bitwise the same lists, ranges and images
    as pgsag_bin_sort; with a too-small capacity the overflow is detected afterwards and the view
    re-sorted after growing the buffers."""
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
    sc = ragged_scene()
    H, W = sc.mask.shape
    g = GaussianTensors.from_numpy(sc.gaussians)
    cam = camera_from(sc.camera)
    mask = torch.from_numpy(np.ascontiguousarray(sc.mask)).cuda()
    ref = Rasterizer(g.n, W, H, g.sh_degree)
    ref.forward(g, cam, mask)
    fast = Rasterizer(g.n, W, H, g.sh_degree, capacity=16, sync_free=True)
    fast.forward(g, cam, mask)
    assert not fast.check_capacity() and fast.M == ref.M  # overflow detected, buffers grown
    fast.forward(g, cam, mask)
    assert fast.check_capacity() and fast.M == ref.M
    torch.cuda.synchronize()
    M = ref.M
    assert torch.equal(fast.vals[:M], ref.vals[:M]) and torch.equal(fast.tile_keys[:M], ref.tile_keys[:M])
    assert torch.equal(fast.ranges, ref.ranges)
    for k in ("img_C", "img_N", "img_D", "img_T", "img_g", "img_last", "img_Dep"):
        assert torch.equal(getattr(fast, k), getattr(ref, k)), k


@pytest.mark.parametrize("frac", [0.5, 0.97])
def test_sync_free_overflow_gives_empty_lists(frac):
    """when M exceeds the capacity in the sync-free sort, the device-side entry
    count is 0 (no partially written prefix with stale entries), so A5 writes no range and A6
    renders every mask pixel as empty (T = 1, g = 0, C = bg), even with the entry buffers
    pre-filled with 0xFF (out-of-range tile ids); capacity = frac * M makes one splat's entry run
    straddle the capacity."""
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
    sc = ragged_scene()
    H, W = sc.mask.shape
    g = GaussianTensors.from_numpy(sc.gaussians)
    cam = camera_from(sc.camera)
    mask = torch.from_numpy(np.ascontiguousarray(sc.mask)).cuda()
    ref = Rasterizer(g.n, W, H, g.sh_degree)
    ref.forward(g, cam, mask)
    cap = max(1, int(frac * ref.M))
    r = Rasterizer(g.n, W, H, g.sh_degree, capacity=cap, sync_free=True)
    r.tile_keys.fill_(-1)
    r.vals.fill_(-1)
    bg = (0.25, 0.5, 0.75)
    r.forward(g, cam, mask, bg)
    torch.cuda.synchronize()
    m = torch.from_numpy(sc.mask.astype(bool)).cuda()
    assert int(r.ranges.abs().sum().item()) == 0
    assert bool((r.img_T[m] == 1.0).all()) and bool((r.img_g[m] == 0).all()) and bool((r.img_last[m] == -1).all())
    for c in range(3):
        assert bool((r.img_C[c][m] == bg[c]).all())
    assert not r.check_capacity() and r.M == ref.M


def test_capacity_retry_keeps_gc_statistics():
    """a PGSAG_ECAPACITY retry inside forward() keeps the per-call image fields
    (the Eq. 9 weights / statistics): the statistics equal those of an ample-capacity run."""
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
    sc = S.config1()
    H, W = sc.mask.shape
    g = GaussianTensors.from_numpy(sc.gaussians)
    cam = camera_from(sc.camera)
    mask = torch.from_numpy(sc.mask).cuda()
    img = torch.from_numpy(S.reference_image(H, W, 5)).cuda()
    out = []
    for cap in (16, 1 << 20):
        r = Rasterizer(g.n, W, H, g.sh_degree, capacity=cap)
        w = r.gc_weights(img, mask)
        r.forward(g, cam, mask, gc_w=w)
        torch.cuda.synchronize()
        out.append(r.gc_load())
    assert out[0][2] == int(sc.mask.sum()) and out[0] == out[1]


def test_trainer_skips_overflowed_view():
    """a sync-free training step whose view overflows the entry capacity leaves
    the parameters and Adam moments untouched (device-side skip in the fused A8 + Adam) and
    reports the overflow; the re-run view then renders exactly like a synchronising trainer's."""
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
    from paper_2501_01677_b200.train import Trainer
    sc = S.config1()
    H, W = sc.mask.shape
    cam = camera_from(sc.camera)
    mask = torch.from_numpy(sc.mask).cuda()
    tgt = torch.from_numpy(S.reference_image(H, W, 9)).cuda()
    ga, gb = GaussianTensors.from_numpy(sc.gaussians), GaussianTensors.from_numpy(sc.gaussians)
    ta = Trainer(Rasterizer(ga.n, W, H, ga.sh_degree), ga)
    tb = Trainer(Rasterizer(gb.n, W, H, gb.sh_degree, capacity=16, sync_free=True), gb)
    before = [x.clone() for x in (gb.mean, gb.scale, gb.opacity, gb.sh, tb.m, tb.v)]
    tb.step(cam, mask, tgt)
    assert tb.losses()["overflowed"]
    for x, y in zip(before, (gb.mean, gb.scale, gb.opacity, gb.sh, tb.m, tb.v)):
        assert torch.equal(x, y)
    tb.t -= 1  # the skipped step is re-run as the same step
    tb.step(cam, mask, tgt)
    lb = tb.losses()
    assert not lb["overflowed"]
    ta.step(cam, mask, tgt)
    la = ta.losses()
    # same render, same L_s (a sum of per-block atomics in double: equal up to its last bits)
    assert la["rgb"] == lb["rgb"] and abs(la["flat"] - lb["flat"]) <= 1e-12 * abs(la["flat"])
    assert not torch.equal(before[0], gb.mean) and not torch.equal(before[4], tb.m)  # the re-run updated


def test_unaligned_tile_key_buffer():
    """pgsag_bins.tile_keys / vals must be 16-byte aligned (the sort reads them with 128-bit loads):
    a buffer 4 bytes off a 16-byte boundary is rejected with PGSAG_EINVAL before any launch."""
    from paper_2501_01677_b200 import _lib as L
    from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
    sc = ragged_scene(seed=5)
    H, W = sc.mask.shape
    g = GaussianTensors.from_numpy(sc.gaussians)
    cam = camera_from(sc.camera)
    mask = torch.from_numpy(np.ascontiguousarray(sc.mask)).cuda()
    odd = Rasterizer(g.n, W, H, g.sh_degree, capacity=4096)
    base = torch.empty(odd.capacity + 4, dtype=torch.int32, device="cuda")
    odd.tile_keys = base[1:1 + odd.capacity]
    assert odd.tile_keys.data_ptr() % 16 == 4
    odd._build_bins()
    with pytest.raises(L.PgsagError) as ei:
        odd.forward(g, cam, mask)
    assert ei.value.code == L.PGSAG_EINVAL and "16-byte aligned" in str(ei.value)
