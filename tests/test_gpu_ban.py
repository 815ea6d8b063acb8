"""NEXT-2 (boundary band, L_ban with normal-from-depth; Eq. 8; R25-R27)
through the C ABI vs the oracle, on N and Dep rendered by A6, and chained into A7/A8."""
import numpy as np
import pytest
import torch

import oracle
from synth import scenes as S
from tests.gpu_util import KAPPA_MAX, compare_grads, dep_kappa
from tests.helpers import all_pixels
from tests.test_gpu_parity import ragged_scene
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

pytestmark = pytest.mark.gpu

SCENES = {"ragged": ragged_scene, "C2s": lambda: S.config2(n=30000)}


def _render(sc):
    H, W = sc.mask.shape
    g = GaussianTensors.from_numpy(sc.gaussians)
    r = Rasterizer(g.n, W, H, g.sh_degree)
    mask = torch.from_numpy(sc.mask).cuda()
    for t in (r.img_N, r.img_Dep):
        t.zero_()
    r.forward(g, camera_from(sc.camera), mask)
    return g, r, mask


def _oracle_planes(sc, ora0, pix):
    """The oracle's own rendered N (3, H, W) and Dep (H, W) (float build, 0 off the mask)."""
    H, W = sc.mask.shape
    N = np.zeros((3, H * W))
    Dep = np.zeros(H * W)
    N[:, pix] = ora0["N"].T
    Dep[pix] = ora0["Dep"]
    return N.reshape(3, H, W), Dep.reshape(H, W)


def _elementwise(a, b, rel=1e-3, floor=1e-2):
    scale = max(np.abs(b).max(), 1e-30)
    return float((np.abs(a - b) / np.maximum(np.abs(b), floor * scale)).max())


@pytest.mark.parametrize("name", list(SCENES))
@pytest.mark.parametrize("radius", [1, 2, 8, 9])  # 9: the untiled path (r > 8)
def test_boundary_band_bitexact(name, radius):
    sc = SCENES[name]()
    _, r, mask = _render(sc)
    band = r.boundary_band(mask, radius).cpu().numpy()
    np.testing.assert_array_equal(band, oracle.boundary_band(sc.mask, radius))


@pytest.mark.parametrize("name", list(SCENES))
def test_ban_loss_and_gradients(name):
    sc = SCENES[name]()
    _, r, mask = _render(sc)
    band = r.boundary_band(mask, 1)
    H, W = sc.mask.shape
    dN = torch.zeros(3, H, W, device="cuda")
    dD = torch.zeros(H, W, device="cuda")
    lam = 0.01  # Eq. 10's lambda_4
    loss = r.ban_loss(band, lam=lam, dN=dN, dDep=dD).cpu().numpy()
    torch.cuda.synchronize()
    N = r.img_N.cpu().numpy().astype(np.float64)
    Dep = r.img_Dep.cpu().numpy().astype(np.float64)
    s, c, rN, rD = oracle.ban_loss(sc.camera, sc.mask, band.cpu().numpy(), N, Dep, lam=lam, grads=True)
    assert loss[1] == c and c > 100
    assert abs(loss[0] - s) <= 1e-4 * max(1.0, s)
    assert _elementwise(dN.cpu().numpy(), rN) <= 1e-3
    assert _elementwise(dD.cpu().numpy(), rD) <= 1e-3
    assert np.linalg.norm(dD.cpu().numpy() - rD) <= 1e-4 * np.linalg.norm(rD)


@pytest.mark.parametrize("name", list(SCENES))
@pytest.mark.parametrize("one_pass", [False, True])
def test_ban_chained_into_backward(name, one_pass):
    """lambda_4 L_ban as the whole loss: its dN, dDep as A7's upstream; parameter gradients vs the
    oracle backward fed with the oracle's own L_ban gradients (depth upstream dropped where Eq. 4
    is ill-conditioned, R19).  one_pass: the sum-gradient written in one pass (mean = 0) and
    divided by the term count inside A7 (pgsag_image_grad.nd_div)."""
    sc = SCENES[name]()
    g, r, mask = _render(sc)
    band = r.boundary_band(mask, 1)
    H, W = sc.mask.shape
    dN = torch.zeros(3, H, W, device="cuda")
    dD = torch.zeros(H, W, device="cuda")
    loss = r.ban_loss(band, lam=0.01, mean=not one_pass, dN=dN, dDep=dD)
    torch.cuda.synchronize()
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    N = r.img_N.cpu().numpy().astype(np.float64)
    Dep = r.img_Dep.cpu().numpy().astype(np.float64)
    _, _, rN, rD = oracle.ban_loss(sc.camera, sc.mask, band.cpu().numpy(), N, Dep, lam=0.01, grads=True)
    drop = (dep_kappa(ora0, pix, W, sc.camera) > KAPPA_MAX) | ora0["near"].astype(bool)
    rDf = rD.reshape(-1)
    rDf[pix[drop]] = 0.0
    dDg = dD.reshape(-1)
    dDg[torch.from_numpy(pix[drop]).cuda()] = 0.0
    rNf = rN.reshape(3, -1)
    rNf[:, pix[ora0["near"].astype(bool)]] = 0.0
    dNg = dN.reshape(3, -1)
    dNg[:, torch.from_numpy(pix[ora0["near"].astype(bool)]).cuda()] = 0.0
    out = r.backward(dN=dN, dDep=dD, nd_div=loss[1:] if one_pass else None)
    grads = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in out.items()}
    up = np.zeros((len(pix), 10))
    up[:, 3:6] = rN.reshape(3, -1)[:, pix].T
    up[:, 8] = rD.reshape(-1)[pix]
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, upstream=up)
    compare_grads(grads, ora["grads"], sc.gaussians.sh_degree)


@pytest.mark.parametrize("name", list(SCENES))
def test_ban_all_oracle_chain(name):
    """The whole NEXT-2 chain against an all-oracle chain: the GPU's A6 render -> band -> L_ban
    (value and its dN / dDep) vs the oracle's own render -> band -> L_ban.  The loss value is held
    to 1e-4 relative plus the first-order effect of the forward contract (|dN| <= 1e-4,
    |dDep| <= 1e-4 max(1, kappa) |Dep|, R19) on it, sum |dL/dN| 1e-4 + |dL/dDep| |dDep|,
    taken with the oracle's own gradients."""
    sc = SCENES[name]()
    _, r, mask = _render(sc)
    band = r.boundary_band(mask, 1)
    H, W = sc.mask.shape
    dN = torch.zeros(3, H, W, device="cuda")
    dD = torch.zeros(H, W, device="cuda")
    lam = 0.01
    loss = r.ban_loss(band, lam=lam, dN=dN, dDep=dD).cpu().numpy()
    torch.cuda.synchronize()
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    N, Dep = _oracle_planes(sc, ora0, pix)
    band_o = oracle.boundary_band(sc.mask, 1)
    s, c, rN, rD = oracle.ban_loss(sc.camera, sc.mask, band_o, N, Dep, lam=lam, grads=True)
    kap = np.zeros(H * W)
    kap[pix] = np.maximum(1.0, dep_kappa(ora0, pix, W, sc.camera))
    tol = 1e-4 * (np.abs(rN).sum() + (np.abs(rD).reshape(-1) * kap * np.abs(Dep).reshape(-1)).sum())
    print(name, "L gpu", loss[0], "L oracle chain", s, "diff", abs(loss[0] - s), "tol", tol + 1e-4 * max(1.0, s))
    assert loss[1] == c
    assert abs(loss[0] - s) <= 1e-4 * max(1.0, s) + tol


@pytest.mark.parametrize("name", list(SCENES))
def test_ban_all_oracle_chain_backward(name):
    """lambda_4 L_ban as the whole loss, GPU chain A6 -> L_ban -> A7/A8 vs the all-oracle chain
    (oracle render -> oracle L_ban -> oracle backward), depth upstream dropped on both sides where
    Eq. 4 is ill-conditioned or the pixel is near a decision (R18, R19)."""
    sc = SCENES[name]()
    g, r, mask = _render(sc)
    band = r.boundary_band(mask, 1)
    H, W = sc.mask.shape
    dN = torch.zeros(3, H, W, device="cuda")
    dD = torch.zeros(H, W, device="cuda")
    r.ban_loss(band, lam=0.01, dN=dN, dDep=dD)
    torch.cuda.synchronize()
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix)
    N, Dep = _oracle_planes(sc, ora0, pix)
    _, _, rN, rD = oracle.ban_loss(sc.camera, sc.mask, oracle.boundary_band(sc.mask, 1), N, Dep, lam=0.01,
                                   grads=True)
    near = ora0["near"].astype(bool)
    drop = (dep_kappa(ora0, pix, W, sc.camera) > KAPPA_MAX) | near
    rD.reshape(-1)[pix[drop]] = 0.0
    dD.reshape(-1)[torch.from_numpy(pix[drop]).cuda()] = 0.0
    rN.reshape(3, -1)[:, pix[near]] = 0.0
    dN.reshape(3, -1)[:, torch.from_numpy(pix[near]).cuda()] = 0.0
    out = r.backward(dN=dN, dDep=dD)
    grads = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in out.items()}
    up = np.zeros((len(pix), 10))
    up[:, 3:6] = rN.reshape(3, -1)[:, pix].T
    up[:, 8] = rD.reshape(-1)[pix]
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, upstream=up, bound=True)
    rep = compare_grads(grads, ora["grads"], sc.gaussians.sh_degree, bound=ora["bound"])
    print(name, rep)
