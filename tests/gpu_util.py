"""Helpers for the -m gpu parity tests: run the CUDA path (through the C ABI)
and the oracle on the same seeded scene, and compare with the DESIGN.md §6
tolerances."""
import numpy as np
import torch

import oracle
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

# Tolerances (BASELINE.json north_star; DESIGN.md §6 / reading R19)
ABS_IMG = 1e-4        # C, N, D, A, T per masked pixel
REL_DEP = 1e-4        # unbiased depth (a ratio)
NEAR_ABS = 5e-3       # pixels the oracle flags as near a decision threshold (R18)
GRAD_REL = 1e-3       # per element, relative to max(|ref|, 1e-2 * maxabs(class))
GRAD_NORM = 1e-4      # per class ||d||/||ref|| (reading R19)


def run_gpu(scene, bg=(0.0, 0.0, 0.0), capacity=None, upstream=None, counters=True, sync_free=False):
    """sync_free: the launch configuration bench.py times (pgsag_bin_sort_async, no host sync; the
    capacity must then hold M, which is checked after the run)."""
    g = GaussianTensors.from_numpy(scene.gaussians)
    cam = camera_from(scene.camera)
    mask = torch.from_numpy(np.ascontiguousarray(scene.mask)).cuda()
    r = Rasterizer(g.n, scene.camera.width, scene.camera.height, g.sh_degree, capacity=capacity,
                   counters=counters, sync_free=sync_free)
    # sentinel fill so unwritten (masked-out) pixels are detectable
    for t in (r.img_C, r.img_N, r.img_D, r.img_A, r.img_Dep, r.img_T):
        t.fill_(-7.0)
    r.img_g.fill_(-7)
    r.forward(g, cam, mask, bg)
    res = {"r": r}
    if upstream is not None:
        up = {k: torch.from_numpy(v).cuda() for k, v in upstream.items()}
        res["grads"] = {k: v.detach().cpu().numpy().astype(np.float64) for k, v in r.backward(**up).items()}
    torch.cuda.synchronize()
    if sync_free:
        assert r.check_capacity(), "sync-free capacity exceeded"
    res["img"] = {k: v.detach().cpu().numpy() for k, v in dict(
        C=r.img_C, N=r.img_N, D=r.img_D, A=r.img_A, Dep=r.img_Dep, T=r.img_T, g=r.img_g, last=r.img_last).items()}
    res["vals"] = r.vals[:r.M].cpu().numpy().view(np.uint32)
    res["tile_keys"] = r.tile_keys[:r.M].cpu().numpy().view(np.uint32)
    res["ranges"] = r.ranges.cpu().numpy().view(np.uint32).reshape(-1, 2)
    res["stats"] = r.stats()
    return res


KAPPA_MAX = 1e3      # Eq. 4 condition number above which dL/dDep is not compared (reading R19)


def dep_kappa(ora, pix, W, cam):
    """Condition number of Eq. 4's denominator N.r at the listed pixels (from the oracle forward)."""
    i_, j_ = pix % W, pix // W
    r0 = (i_ + 0.5 - cam.cx) / cam.fx
    r1 = (j_ + 0.5 - cam.cy) / cam.fy
    Nn = ora["N"].astype(np.float64)
    den = np.abs(Nn[:, 0] * r0 + Nn[:, 1] * r1 + Nn[:, 2])
    return (np.abs(r0) + np.abs(r1) + 1.0) / np.maximum(den, 1e-30)


def upstream_at(pix, H, W, seed, exclude=None, ora=None, cam=None):
    """Random N(0,1) upstream gradients at the listed flat pixels, 0 elsewhere; returns (planar dict,
    per-listed-pixel (npix, 9) array for the oracle).  exclude: pixels (near a decision threshold,
    R18) with no upstream at all; with ora+cam, dL/dDep is dropped where Eq. 4 is ill-conditioned."""
    rng = np.random.default_rng(seed)
    per = rng.normal(size=(len(pix), 9))
    if exclude is not None:
        per[exclude] = 0.0
    if ora is not None and cam is not None:
        per[dep_kappa(ora, pix, W, cam) > KAPPA_MAX, 8] = 0.0
    planes = {"dC": np.zeros((3, H * W), np.float32), "dN": np.zeros((3, H * W), np.float32),
              "dD": np.zeros(H * W, np.float32), "dA": np.zeros(H * W, np.float32),
              "dDep": np.zeros(H * W, np.float32)}
    per32 = per.astype(np.float32)
    planes["dC"][:, pix] = per32[:, 0:3].T
    planes["dN"][:, pix] = per32[:, 3:6].T
    planes["dD"][pix] = per32[:, 6]
    planes["dA"][pix] = per32[:, 7]
    planes["dDep"][pix] = per32[:, 8]
    planes = {k: np.ascontiguousarray(v.reshape((3, H, W) if v.ndim == 2 else (H, W))) for k, v in planes.items()}
    return planes, per32.astype(np.float64)


def near_scale(proj):
    """Per output class, S = max(1, max |x| over live Gaussians) for the quantity x each blend
    carries (rgb, n_cam, dist; 1 for A and T).  One flipped decision at an R18-flagged pixel
    moves an output by at most 1e-2 * S: an alpha-threshold flip adds or drops a weight
    w <= T/255 and rescales the remainder by (1 - alpha) (2/255 S in all), a T-stop flip drops
    w = alpha*T < 1e-4/(1 - alpha) <= 1e-2 (alpha <= 0.99)."""
    live = (proj["flags"] & 15) == 15
    m = lambda a: max(1.0, float(np.abs(a[live]).max())) if live.any() else 1.0
    return {"C": m(proj["rgb"]), "N": m(proj["ncam"]), "D": m(proj["dist"]), "A": 1.0, "T": 1.0}


def compare_pixels(gpu_img, ora, pix, W, vals, cam=None, proj=None):
    """Element-wise forward parity on the listed pixels. Returns dict of max errors; asserts.
    With proj (oracle.project of the scene), R18-flagged pixels are held to the derived bound
    1e-2 * near_scale(proj)[class] instead of the flat NEAR_ABS."""
    near = ora["near"].astype(bool)
    flat = lambda a: a.reshape(a.shape[0], -1) if a.ndim == 3 else a.reshape(-1)
    C = flat(gpu_img["C"])[:, pix].T
    N = flat(gpu_img["N"])[:, pix].T
    D, A, Dep, T = (flat(gpu_img[k])[pix] for k in ("D", "A", "Dep", "T"))
    g, last = flat(gpu_img["g"])[pix], flat(gpu_img["last"])[pix]
    ok = ~near
    errs = {}
    nsc = near_scale(proj) if proj is not None else None
    for k, a, b in (("C", C, ora["C"]), ("N", N, ora["N"]), ("D", D, ora["D"]), ("A", A, ora["A"]),
                    ("T", T, ora["T"])):
        e = np.abs(a.astype(np.float64) - b.astype(np.float64))
        if k == "D":  # plane distance is in scene units (metres): 1e-4 of max(1, |D|) (reading R19)
            e = e / np.maximum(1.0, np.abs(b.astype(np.float64)))
        e = e.max(axis=1) if e.ndim == 2 else e
        errs[k] = float(e[ok].max()) if ok.any() else 0.0
        assert errs[k] <= ABS_IMG, (k, errs[k], np.argmax(np.where(ok, e, 0)))
        if near.any():
            if nsc is None:
                assert float(e[near].max()) <= NEAR_ABS, (k, "near", float(e[near].max()))
            else:
                en = np.abs(a.astype(np.float64) - b.astype(np.float64))
                en = en.max(axis=1) if en.ndim == 2 else en
                assert float(en[near].max()) <= 1e-2 * nsc[k], (k, "near", float(en[near].max()), nsc[k])
    # Eq. 4 divides by N.r; its relative error is amplified by the condition number of that
    # dot product, kappa = (|r0| + |r1| + 1) / |N.r| (each |n_i| = 1, sum w_i <= 1), so the 1e-4
    # relative bar is applied as 1e-4 * max(1, kappa) (reading R19).
    dv = (ora["Dep"] != 0) & ok
    i_, j_ = pix % W, pix // W
    de =np.abs(Dep[dv].astype(np.float64) - ora["Dep"][dv]) / np.maximum(np.abs(ora["Dep"][dv]), 1e-6)
    if cam is not None:
        r0 = (i_ + 0.5 - cam.cx) / cam.fx
        r1 = (j_ + 0.5 - cam.cy) / cam.fy
        Nn = ora["N"].astype(np.float64)
        den = np.abs(Nn[:, 0] * r0 + Nn[:, 1] * r1 + Nn[:, 2])
        kappa = (np.abs(r0) + np.abs(r1) + 1.0) / np.maximum(den, 1e-12)
        de = de / np.maximum(1.0, kappa[dv])
    errs["Dep"] = float(de.max()) if de.size else 0.0
    assert errs["Dep"] <= REL_DEP, errs["Dep"]
    assert np.array_equal((Dep != 0)[ok], (ora["Dep"] != 0)[ok])
    assert np.array_equal(g[ok], ora["g"][ok]), int((g[ok] != ora["g"][ok]).sum())
    has = ok & (ora["last"] >= 0)
    assert np.array_equal(vals[last[has]], ora["last"][has].astype(np.uint32))
    assert (last[ok & (ora["last"] < 0)] == -1).all()
    errs["n_near"] = int(near.sum())
    return errs


def compare_grads(gpu, ref, deg, bound=None):
    """Per-class gradient parity (reading R19).  bound: the oracle's R19b + R19c bound
    (59, n) on what float32 accumulation and float32 evaluation of the same per-pixel terms can
    cost each element (derived in oracle.cpp eval_bound / DESIGN.md); it is added to the element
    tolerance, and its norm to the class norm tolerance (|d| <= tol + bound elementwise gives
    ||d|| <= ||tol|| + ||bound||)."""
    K3 = (deg + 1) ** 2 * 3
    classes = {"dmean": (gpu["dmean"], ref[0:3]), "dscale": (gpu["dscale"], ref[3:6]),
               "drot": (gpu["drot"], ref[6:10]), "dopacity": (gpu["dopacity"], ref[10]),
               "dsh": (gpu["dsh"][:K3], ref[11:11 + K3])}
    report = {}
    rows = {"dmean": slice(0, 3), "dscale": slice(3, 6), "drot": slice(6, 10), "dopacity": 10,
            "dsh": slice(11, 11 + K3)}
    for k, (a, b) in classes.items():
        a = np.asarray(a, np.float64)
        scale = max(np.abs(b).max(), 1e-30)
        den = np.maximum(np.abs(b), 1e-2 * scale)
        nb = 0.0
        if bound is not None:  # R19b + R19c, in units of the relative tolerance
            den = den + bound[rows[k]] / GRAD_REL
            nb = float(np.linalg.norm(bound[rows[k]]) / max(np.linalg.norm(b), 1e-30))
        el = float((np.abs(a - b) / den).max())
        nrm = float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
        report[k] = (el, nrm)
        assert el <= GRAD_REL, (k, el)
        assert nrm <= GRAD_NORM + nb, (k, nrm, nb)
    return report
