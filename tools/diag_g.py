"""Diagnose a blend-count mismatch for a fuzz seed: per pixel, recompute every pair's decision
quantities in float64 from the oracle's projection and show those near the thresholds."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from tests.test_gpu_fuzz import _scene
from tests.gpu_util import run_gpu
from tests.helpers import all_pixels
seed = int(sys.argv[1])
sc, bg = _scene(seed)
H, W = sc.mask.shape
pix = all_pixels(sc.mask)
ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
res = run_gpu(sc, bg=bg)
g = res["img"]["g"].reshape(-1)[pix]
bad = np.flatnonzero((g != ora["g"]) & (ora["near"] == 0))
print("W H n", W, H, sc.gaussians.n, "bad pixels", bad.size)
p = oracle.project(sc.gaussians, sc.camera, sc.mask)
for b in bad[:3]:
    q = pix[b]; i, j = q % W, q // W
    print("pixel", i, j, "gpu g", g[b], "ora g", ora["g"][b], "gpu last", res["img"]["last"].reshape(-1)[q],
          "ora last id", ora["last"][b], "T gpu/ora", res["img"]["T"].reshape(-1)[q], ora["T"][b])
    live = np.flatnonzero((p["flags"] & 15) == 15)
    order = live[np.lexsort((live, p["depth"][live]))]
    T = 1.0
    blends = []
    gid = res["vals"][res["img"]["last"].reshape(-1)[q]]
    print("  gpu last gaussian id", gid)
    for k in order:
        u, v = p["mean2d"][k]
        ca, cb, cc, o = p["conic_o"][k].astype(np.float64)
        dx, dy = i + 0.5 - u, j + 0.5 - v
        pw = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy
        if pw > 0:
            if pw < 1e-4: print("  near power>0", k, pw)
            continue
        a = min(0.99, o * np.exp(pw))
        if a < 1 / 255:
            if a > (1 / 255) * (1 - 1e-4): print("  near alpha", k, a, a * 255 - 1)
            continue
        Tn = T * (1 - a)
        blends.append((k, a, pw, T))
        if abs(Tn - 1e-4) < 1e-6: print("  near T", k, Tn)
        if Tn < 1e-4:
            print("  stop at", k, "T", T, "Tn", Tn)
            break
        T = Tn
    print("  n blends (f64 recompute)", len(blends))
    for (k, a, pw, TT) in blends[-4:]:
        print("   blend", k, "alpha", a, "alpha*255-1", a * 255 - 1, "power", pw, "T", TT)

# emulate A6's exact block cull (alpha.cuh stage_gaussian<8, 8>) in float32 for the pixel's block
f = np.float32
def cull_hits(u, v, co, tile_x0, tile_y0, bw=8, bh=8):
    ca, cb, cc, o = [f(x) for x in co]
    l2o = f(np.log2(f(255.0) * o))
    bb = cb * cb
    det = (ca * cc - bb) - (cb * cb - bb)
    k2 = f(2.0) * (f(max(l2o, 0.0)) * f(0.6931472) + f(0.01)) * f(1.05)
    kd = k2 / det
    rx = f(np.sqrt(kd * cc)) + f(0.5)
    ry = f(np.sqrt(kd * ca)) + f(0.5)
    k2m = k2 + f(0.05)
    out = []
    for kb in range((16 // bw) * (16 // bh)):
        xlo = f(tile_x0 + (kb % (16 // bw)) * bw + 0.5); xhi = xlo + f(bw - 1)
        ylo = f(tile_y0 + (kb // (16 // bw)) * bh + 0.5); yhi = ylo + f(bh - 1)
        hit = (u + rx >= xlo) and (u - rx <= xhi) and (v + ry >= ylo) and (v - ry <= yhi)
        if hit and not (xlo <= u <= xhi and ylo <= v <= yhi):
            def em(dfix, lo, hi, fixx):
                t = -cb * dfix / cc if fixx else -cb * dfix / ca
                t = min(max(t, lo), hi)
                dx, dy = (dfix, t) if fixx else (t, dfix)
                a_, b_, c_ = ca * dx * dx, f(2) * cb * dx * dy, cc * dy * dy
                return a_ + b_ + c_, abs(a_) + abs(b_) + abs(c_)
            qs = [em(xlo - u, ylo - v, yhi - v, True), em(xhi - u, ylo - v, yhi - v, True),
                  em(ylo - v, xlo - u, xhi - u, False), em(yhi - v, xlo - u, xhi - u, False)]
            hit = any(q - f(1e-5) * e <= k2m for q, e in qs)
        out.append(hit)
    return out
for b in bad[:1]:
    q = pix[b]; i, j = q % W, q // W
    tx0, ty0 = (i // 16) * 16, (j // 16) * 16
    kb = ((j % 16) // 8) * 2 + (i % 16) // 8
    for (k, a, pw, TT) in blends:
        u, v = [f(x) for x in p["mean2d"][k]]
        hits = cull_hits(u, v, p["conic_o"][k], tx0, ty0)
        if not hits[kb]:
            print("  CULLED blended gaussian", k, "alpha", a, "block", kb, "u v", u, v, "conic_o", p["conic_o"][k])
