"""Per fuzz seed and gradient class: GPU-vs-oracle(float build) error against the oracle's own
float-vs-double build gap (the spread float32 evaluation causes), norm-wise and element-wise.

    python tools/diag_gap.py SEED [SEED ...]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from tests.test_gpu_fuzz import _scene
from tests.gpu_util import run_gpu, upstream_at
from tests.helpers import all_pixels

for seed in [int(s) for s in sys.argv[1:]]:
    sc, bg = _scene(seed)
    H, W = sc.mask.shape
    pix = all_pixels(sc.mask)
    ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
    planes, per = upstream_at(pix, H, W, seed=seed, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
    res = run_gpu(sc, bg=bg, upstream=planes, counters=False)
    o32 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per, bound=True)
    o64 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per, dtype=np.float64)
    K3 = (sc.gaussians.sh_degree + 1) ** 2 * 3
    line = [f"{seed:5d} n={sc.gaussians.n:3d}"]
    for k, s in (("dmean", slice(0, 3)), ("dscale", slice(3, 6)), ("drot", slice(6, 10)),
                 ("dopacity", slice(10, 11)), ("dsh", slice(11, 11 + K3))):
        a = np.asarray(res["grads"][k], np.float64).reshape(-1, sc.gaussians.n)[: s.stop - s.start]
        b, c = o32["grads"][s], o64["grads"][s]
        nb = max(np.linalg.norm(b), 1e-30)
        gap = np.abs(b - c)
        den = 1e-3 * np.maximum(np.abs(b), 1e-2 * np.abs(b).max()) + o32["bound"][s]
        el = np.abs(a - b) / (den + 4 * gap)
        line.append(f"{k}: err {np.linalg.norm(a - b) / nb:.1e} gap {np.linalg.norm(gap) / nb:.1e} el {el.max():.2f}")
    print(" | ".join(line), flush=True)
