"""Pins of the NEXT-3 oracle pieces (masked L_rgb, L_s, Adam) against closed forms,
a library window sum, finite differences and invariances (R28-R30)."""
import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle

C1, C2 = 0.01 ** 2, 0.03 ** 2


def _imgs(H=18, W=23, seed=0, pmask=0.75):
    rng = np.random.default_rng(seed)
    Cimg = rng.uniform(0, 1, (3, H, W))
    Iimg = rng.uniform(0, 1, (3, H, W))
    mask = (rng.uniform(size=(H, W)) < pmask).astype(np.uint8)
    return Cimg, Iimg, mask


def _window():
    k = np.arange(-5, 6)
    g = np.exp(-k * k / (2 * 1.5 ** 2))
    g /= g.sum()
    return np.outer(g, g)


def test_identical_images_zero_loss():
    Cimg, _, mask = _imgs()
    L, L1, S, dC = oracle.rgb_loss(Cimg, Cimg, mask, grads=True)
    assert L == 0.0 and L1 == 0.0 and abs(S - 1.0) < 1e-14
    assert np.abs(dC).max() < 1e-12  # SSIM is maximal at x = y, sign(0) = 0


def test_constant_images_closed_form():
    """x = a, y = b on the whole image (full mask), zero padding: with s_p the in-image weight of
    the window at p, mu_x = a s, E[x^2] = a^2 s, so sigma_x^2 = a^2 s (1 - s), sigma_xy = a b s (1 - s)."""
    H, W, a, b = 13, 17, 0.7, 0.3
    k = np.arange(-5, 6)
    g = np.exp(-k * k / 4.5)
    g /= g.sum()
    s1 = lambda n: np.array([sum(g[d + 5] for d in range(-5, 6) if 0 <= i + d < n) for i in range(n)])
    s = np.outer(s1(H), s1(W))
    ssim = ((2 * a * b * s * s + C1) * (2 * a * b * s * (1 - s) + C2)) / \
        (((a * a + b * b) * s * s + C1) * ((a * a + b * b) * s * (1 - s) + C2))
    L, L1, S = oracle.rgb_loss(np.full((3, H, W), a), np.full((3, H, W), b), np.ones((H, W), np.uint8))
    assert abs(S - ssim.mean()) < 1e-13
    assert abs(L1 - abs(a - b)) < 1e-14
    assert abs(L - (0.8 * abs(a - b) + 0.2 * (1 - ssim.mean()))) < 1e-13


def test_against_library_window_sums():
    Cimg, Iimg, mask = _imgs(seed=3)
    w = _window()
    m = mask.astype(np.float64)
    tot = 0.0
    for c in range(3):
        x, y = Cimg[c] * m, Iimg[c] * m
        f = lambda z: ndi.correlate(z, w, mode="constant", cval=0.0)
        mx, my = f(x), f(y)
        sxx, syy, sxy = f(x * x) - mx * mx, f(y * y) - my * my, f(x * y) - mx * my
        smap = ((2 * mx * my + C1) * (2 * sxy + C2)) / ((mx * mx + my * my + C1) * (sxx + syy + C2))
        tot += smap[mask != 0].sum()
    S_lib = tot / (3 * mask.sum())
    L1_lib = np.abs(Cimg - Iimg)[:, mask != 0].mean()
    L, L1, S = oracle.rgb_loss(Cimg, Iimg, mask)
    assert abs(S - S_lib) < 1e-12 and abs(L1 - L1_lib) < 1e-13
    assert abs(L - (0.8 * L1_lib + 0.2 * (1 - S_lib))) < 1e-12


def test_gradient_finite_differences():
    """Central differences of L on mask and off-mask pixels (|C - I| >= 0.05 keeps the L1 kink away)."""
    H, W = 14, 15
    rng = np.random.default_rng(5)
    Iimg = rng.uniform(0.2, 0.8, (3, H, W))
    Cimg = Iimg + rng.choice([-1, 1], (3, H, W)) * rng.uniform(0.05, 0.2, (3, H, W))
    mask = (rng.uniform(size=(H, W)) < 0.7).astype(np.uint8)
    _, _, _, dC = oracle.rgb_loss(Cimg, Iimg, mask, grads=True)
    h = 1e-6
    for _ in range(40):
        c, j, i = rng.integers(0, 3), rng.integers(0, H), rng.integers(0, W)
        cp, cm = Cimg.copy(), Cimg.copy()
        cp[c, j, i] += h
        cm[c, j, i] -= h
        fd = (oracle.rgb_loss(cp, Iimg, mask)[0] - oracle.rgb_loss(cm, Iimg, mask)[0]) / (2 * h)
        assert abs(fd - dC[c, j, i]) < 1e-7 + 1e-5 * abs(fd), (c, j, i, fd, dC[c, j, i])
        if not mask[j, i]:
            assert dC[c, j, i] == 0.0


def test_off_mask_pixels_do_not_matter():
    Cimg, Iimg, mask = _imgs(seed=7)
    rng = np.random.default_rng(8)
    C2i, I2 = Cimg.copy(), Iimg.copy()
    off = mask == 0
    C2i[:, off] = rng.uniform(size=(3, off.sum()))
    I2[:, off] = rng.uniform(size=(3, off.sum()))
    a = oracle.rgb_loss(Cimg, Iimg, mask, grads=True)
    b = oracle.rgb_loss(C2i, I2, mask, grads=True)
    assert a[:3] == b[:3]
    assert np.array_equal(a[3], b[3])


def test_flatten_loss_brute_force():
    rng = np.random.default_rng(9)
    s = rng.uniform(0.01, 1.0, (3, 50))
    s[:, 0] = [0.2, 0.1, 0.1]  # tie -> lowest index
    L, g = oracle.flatten_loss(s)
    assert abs(L - np.mean([min(s[:, i]) for i in range(50)])) < 1e-15
    for i in range(50):
        k = [0, 1, 2][int(np.argmin(s[:, i]))]
        assert g[k, i] == 1 / 50 and g[:, i].sum() == 1 / 50
    assert g[1, 0] == 1 / 50


def test_adam_first_steps_closed_form():
    """Step 1: m_hat = g, v_hat = g^2, so the update is -lr g / (|g| + eps); with a constant gradient
    every later step is the same (m_hat = g, v_hat = g^2 exactly after bias correction)."""
    rng = np.random.default_rng(10)
    g = rng.normal(size=100) * 10.0 ** rng.uniform(-4, 2, 100)
    p = rng.normal(size=100)
    m, v = np.zeros(100), np.zeros(100)
    q = p.copy()
    for t in (1, 2, 3):
        q, m, v = oracle.adam_step(q, g, m, v, t, lr=1e-2)
        assert np.allclose(q, p - t * 1e-2 * g / (np.abs(g) + 1e-15), rtol=0, atol=1e-12)


def test_raw_gradient_chain_finite_differences():
    """raw_grads against central differences of f(s, o) = sum a s + b o + w L_s through s = exp(l), o = sigmoid(z)."""
    rng = np.random.default_rng(11)
    n, w = 6, 3.0
    ls, z = rng.normal(-1, 0.5, (3, n)), rng.normal(0, 1, n)
    a, b = rng.normal(size=(3, n)), rng.normal(size=n)
    f = lambda ls_, z_: (a * np.exp(ls_)).sum() + (b / (1 + np.exp(-z_))).sum() + w * oracle.flatten_loss(np.exp(ls_))[0]
    gl, gz = oracle.raw_grads(np.exp(ls), 1 / (1 + np.exp(-z)), a, b, w)
    h = 1e-6
    for k in range(3):
        for i in range(n):
            e = np.zeros((3, n)); e[k, i] = h
            assert abs((f(ls + e, z) - f(ls - e, z)) / (2 * h) - gl[k, i]) < 1e-7
    for i in range(n):
        e = np.zeros(n); e[i] = h
        assert abs((f(ls, z + e) - f(ls, z - e)) / (2 * h) - gz[i]) < 1e-7


def test_train_update_rows_and_activations():
    """Row order / learning rates / activations of train_update: with a constant gradient every step
    moves each raw row by exactly -lr sign(g) (Adam, bias-corrected), so the activated values are
    exp / sigmoid of the moved raw values."""
    rng = np.random.default_rng(12)
    n, K3 = 7, 48
    p = dict(mean=rng.normal(size=(3, n)), log_scale=rng.normal(-2, 0.3, (3, n)), rot=rng.normal(size=(4, n)),
             logit_opacity=rng.normal(size=n), sh=rng.normal(size=(K3, n)))
    p["scale"], p["opacity"] = np.exp(p["log_scale"]), 1 / (1 + np.exp(-p["logit_opacity"]))
    g = dict(dmean=rng.normal(size=(3, n)), dscale=rng.normal(size=(3, n)), drot=rng.normal(size=(4, n)),
             dopacity=rng.normal(size=n), dsh=rng.normal(size=(K3, n)))
    hp = dict(lr_mean=1e-3, lr_scale=2e-3, lr_rot=3e-3, lr_opacity=4e-3, lr_sh_dc=5e-3, lr_sh_rest=6e-3,
              beta1=0.9, beta2=0.999, eps=1e-15)
    m, v = np.zeros((11 + K3, n)), np.zeros((11 + K3, n))
    q, m, v, Ls = oracle.train_update(p, g, m, v, 1, hp, flatten_weight=0.0)
    assert abs(Ls - p["scale"].min(axis=0).mean()) < 1e-15
    assert np.allclose(q["mean"], p["mean"] - 1e-3 * np.sign(g["dmean"]), atol=1e-12)
    assert np.allclose(q["log_scale"], p["log_scale"] - 2e-3 * np.sign(g["dscale"]), atol=1e-12)
    assert np.allclose(q["scale"], np.exp(q["log_scale"]), atol=0)
    assert np.allclose(q["rot"], p["rot"] - 3e-3 * np.sign(g["drot"]), atol=1e-12)
    assert np.allclose(q["logit_opacity"], p["logit_opacity"] - 4e-3 * np.sign(g["dopacity"]), atol=1e-12)
    assert np.allclose(q["opacity"], 1 / (1 + np.exp(-q["logit_opacity"])), atol=0)
    assert np.allclose(q["sh"][:3], p["sh"][:3] - 5e-3 * np.sign(g["dsh"][:3]), atol=1e-12)
    assert np.allclose(q["sh"][3:], p["sh"][3:] - 6e-3 * np.sign(g["dsh"][3:]), atol=1e-12)
    assert np.allclose(m, 0.1 * np.vstack([g["dmean"], g["dscale"] * p["scale"], g["drot"],
                                           (g["dopacity"] * p["opacity"] * (1 - p["opacity"]))[None], g["dsh"]]))


# ------------------------------------------------------------ densification (R31)
def test_splitmix64_reference_values():
    """SplitMix64 (Steele, Lea, Flood 2014): the first outputs of the generator seeded with 0 are the
    published 0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F."""
    g = 0x9E3779B97F4A7C15
    outs = [oracle.splitmix64((k * g) & ((1 << 64) - 1)) for k in range(3)]
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_split_normals_moments():
    z = np.array([oracle.split_normals(1677, i, c) for i in range(4000) for c in (0, 1)])
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1) < 0.02
    assert abs(np.corrcoef(z[:, 0], z[:, 1])[0, 1]) < 0.03
    assert not np.array_equal(oracle.split_normals(1, 5, 0), oracle.split_normals(1, 5, 1))


def test_densify_actions_decisions():
    s = np.array([[0.01, 0.5, 0.01, 0.5, 0.02], [0.01, 0.01, 0.01, 0.01, 0.02], [0.01, 0.01, 0.01, 0.01, 0.02]])
    o = np.array([0.5, 0.5, 0.5, 0.5, 0.001])
    acc = np.array([0.0, 0.0, 1.0, 1.0, 1.0])
    cnt = np.array([0.0, 3.0, 2.0, 2.0, 2.0])
    a = oracle.densify_actions(s, o, acc, cnt, grad_threshold=0.4, dense_limit=0.1, min_opacity=0.005)
    assert a.tolist() == [1, 1, 2, 3, 0]
    # the threshold is inclusive and the dense limit exclusive (float32 decisions)
    a = oracle.densify_actions(s[:, 2:4], o[2:4], acc[2:4], cnt[2:4], grad_threshold=0.5, dense_limit=0.5,
                               min_opacity=0.005)
    assert a.tolist() == [2, 2]


def _dens_state(rng, n, K3=12):
    p = dict(mean=rng.normal(size=(3, n)), rot=rng.normal(size=(4, n)), sh=rng.normal(size=(K3, n)),
             log_scale=rng.normal(-2, 0.5, (3, n)), logit_opacity=rng.normal(size=n))
    p["scale"] = np.exp(p["log_scale"]).astype(np.float32).astype(np.float64)
    p["opacity"] = 1 / (1 + np.exp(-p["logit_opacity"]))
    return p, rng.normal(size=(11 + K3, n)), rng.uniform(size=(11 + K3, n))


def test_densify_apply_layout_and_counts():
    rng = np.random.default_rng(13)
    n = 9
    p, m, v = _dens_state(rng, n)
    act = np.array([1, 0, 2, 3, 1, 2, 3, 0, 1], np.uint8)
    q, m2, v2 = oracle.densify_apply(p, m, v, act, seed=7)
    keep, clone, split = [0, 2, 4, 5, 8], [2, 5], [3, 6]
    n2 = len(keep) + len(clone) + 2 * len(split)
    assert q["mean"].shape == (3, n2) and m2.shape == (23, n2)
    for k in ("mean", "rot", "sh", "scale", "opacity", "log_scale", "logit_opacity"):
        assert np.array_equal(q[k][..., :5], np.asarray(p[k])[..., keep])            # kept, source order
        assert np.array_equal(q[k][..., 5:7], np.asarray(p[k])[..., clone])          # clones = copies
    assert np.array_equal(m2[:, :5], m[:, keep]) and (m2[:, 5:] == 0).all() and (v2[:, 5:] == 0).all()
    for j, i in enumerate(split):  # children: scale / 1.6, same rot / opacity / sh
        for c in (0, 1):
            col = 7 + 2 * j + c
            assert np.allclose(q["scale"][:, col], p["scale"][:, i] / 1.6, rtol=1e-7)
            assert np.allclose(q["log_scale"][:, col], np.log(p["scale"][:, i] / 1.6), rtol=1e-6)
            for k in ("rot", "sh", "opacity", "logit_opacity"):
                assert np.array_equal(q[k][..., col], np.asarray(p[k])[..., i])
            R = oracle.quat_to_rot(p["rot"][:, i])
            z = R.T @ (q["mean"][:, col] - p["mean"][:, i]) / p["scale"][:, i]
            assert np.allclose(z, oracle.split_normals(7, int(i), c))


def test_split_children_covariance():
    """Children of one Gaussian are samples of N(mu, R S^2 R^T): empirical covariance over many
    (seeded) splits of the same source matches it within sampling error."""
    rng = np.random.default_rng(14)
    p, m, v = _dens_state(rng, 1)
    p["scale"][:, 0] = [0.5, 0.2, 0.05]
    R = oracle.quat_to_rot(p["rot"][:, 0])
    pts = []
    for seed in range(1500):
        q, _, _ = oracle.densify_apply(p, m, v, np.array([3], np.uint8), seed=seed * 7919)
        pts += [q["mean"][:, 0], q["mean"][:, 1]]
    d = np.array(pts) - p["mean"][:, 0]
    cov = np.cov(d.T)
    ref = R @ np.diag(p["scale"][:, 0] ** 2) @ R.T
    assert np.abs(cov - ref).max() < 0.06 * ref.max()
