import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, oracle
from tests.test_gpu_parity import _tiny
from tests.gpu_util import run_gpu, upstream_at
from tests.helpers import all_pixels
for deg_case in ("single",):
    sc = _tiny(1)
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    planes, per = upstream_at(pix, H, W, seed=1)
    res = run_gpu(sc, bg=(0.5, 0.25, 0.125), upstream=planes)
    r = res["r"]; r.export_grad2d(True)
    ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=(0.5, 0.25, 0.125), upstream=per)
    G = ora["grads"]
    print("flags", r.flags.cpu().numpy()[:1], "conic", r.conic_o.cpu().numpy()[:1], "mean2d", r.mean2d.cpu().numpy()[:1])
    print("dmean gpu", res["grads"]["dmean"][:, 0], "ref", G[0:3, 0])
    print("dscale gpu", res["grads"]["dscale"][:, 0], "ref", G[3:6, 0])
    print("g2d ref", G[59:73, 0])
    print("blended", int(ora["g"].sum()), "near", int(ora["near"].sum()))
