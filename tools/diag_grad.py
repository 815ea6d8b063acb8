"""Diagnose a fuzz gradient mismatch: the gradients are linear in the upstream, so bisect the
mask pixels (upstream zeroed outside the half) down to the pixel whose contribution carries the
GPU-vs-oracle error, then print that pixel's decisions (float64 recompute) near any threshold.

    python tools/diag_grad.py SEED [CLASS]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from tests.test_gpu_fuzz import _scene
from tests.gpu_util import run_gpu, upstream_at
from tests.helpers import all_pixels

seed = int(sys.argv[1])
sc, bg = _scene(seed)
H, W = sc.mask.shape
pix = all_pixels(sc.mask)
ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
planes, per = upstream_at(pix, H, W, seed=seed, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
deg = sc.gaussians.sh_degree
K3 = (deg + 1) ** 2 * 3
rows = {"dmean": slice(0, 3), "dscale": slice(3, 6), "drot": slice(6, 10), "dopacity": slice(10, 11),
        "dsh": slice(11, 11 + K3)}


def errs(sel):
    pl = {k: np.zeros_like(v) for k, v in planes.items()}
    p2 = np.zeros_like(per)
    p2[sel] = per[sel]
    q = pix[sel]
    for k, v in planes.items():
        if v.ndim == 3:
            pl[k].reshape(3, -1)[:, q] = v.reshape(3, -1)[:, q]
        else:
            pl[k].reshape(-1)[q] = v.reshape(-1)[q]
    res = run_gpu(sc, bg=bg, upstream=pl, counters=False)
    ref = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=p2)["grads"]
    out = {}
    for k, s in rows.items():
        a = np.asarray(res["grads"][k], np.float64).reshape(-1, sc.gaussians.n)[: s.stop - s.start]
        b = ref[s]
        out[k] = (float(np.linalg.norm(a - b)), float(np.linalg.norm(b)))
    return out


full = errs(np.arange(len(pix)))
print("W H n deg", W, H, sc.gaussians.n, deg, "near", int(ora0["near"].sum()))
for k, (d, b) in full.items():
    print(f"  {k}: |d| {d:.3e} |ref| {b:.3e} rel {d / max(b, 1e-30):.3e}")
cls = sys.argv[2] if len(sys.argv) > 2 else max(full, key=lambda k: full[k][0] / max(full[k][1], 1e-30))
sel = np.arange(len(pix))
while sel.size > 1:
    a, b = sel[: sel.size // 2], sel[sel.size // 2:]
    ea, eb = errs(a)[cls][0], errs(b)[cls][0]
    print(f"  bisect {sel.size}: halves {ea:.3e} {eb:.3e}")
    sel = a if ea >= eb else b
q = int(pix[sel[0]])
i, j = q % W, q // W
print("pixel", i, j, "upstream", per[sel[0]], "ora g", ora0["g"][sel[0]], "T", ora0["T"][sel[0]])
p = oracle.project(sc.gaussians, sc.camera, sc.mask)
live = np.flatnonzero((p["flags"] & 15) == 15)
order = live[np.lexsort((live, p["depth"][live]))]
T = 1.0
for k in order:
    u, v = p["mean2d"][k].astype(np.float64)
    ca, cb, cc, o = p["conic_o"][k].astype(np.float64)
    dx, dy = i + 0.5 - u, j + 0.5 - v
    pw = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy
    mag = 0.5 * (abs(ca) * dx * dx + abs(cc) * dy * dy) + abs(cb * dx * dy)
    if pw > 0:
        continue
    a = o * np.exp(pw)
    if a < 1 / 255:
        continue
    print(f"   blend {k} alpha {min(a, 0.99):.6f} o*rho {a:.6f} T {T:.3e} power {pw:.4f} mag {mag:.3e} "
          f"conic {ca:.4g} {cb:.4g} {cc:.4g} det {ca * cc - cb * cb:.3e}")
    Tn = T * (1 - min(a, 0.99))
    if Tn < 1e-4:
        print("   stop", k, Tn)
        break
    T = Tn
