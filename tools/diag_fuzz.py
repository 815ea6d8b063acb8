"""Diagnose a fuzz seed: worst gradient element, its Gaussian, and the A7 2D gradients of it."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from tests.test_gpu_fuzz import _scene
from tests.gpu_util import upstream_at
from tests.helpers import all_pixels
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
seed = int(sys.argv[1])
sc, bg = _scene(seed)
H, W = sc.mask.shape
pix = all_pixels(sc.mask)
ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
planes, per = upstream_at(pix, H, W, seed=seed, exclude=ora0["near"].astype(bool), ora=ora0, cam=sc.camera)
ref = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per)["grads"]
g = GaussianTensors.from_numpy(sc.gaussians)
r = Rasterizer(g.n, W, H, g.sh_degree, absgrad=True)
r.export_grad2d(True)
r.forward(g, camera_from(sc.camera), torch.from_numpy(np.ascontiguousarray(sc.mask)).cuda(), bg)
out = r.backward(**{k: torch.from_numpy(v).cuda() for k, v in planes.items()})
torch.cuda.synchronize()
drot = out["drot"].cpu().numpy().astype(np.float64)
b = ref[6:10]
scale = np.abs(b).max()
err = np.abs(drot - b) / np.maximum(np.abs(b), 1e-2 * scale)
k, i = np.unravel_index(np.argmax(err), err.shape)
print("W,H,n,deg", W, H, g.n, g.sh_degree, "worst drot", k, i, err[k, i], drot[k, i], b[k, i], "scale", scale)
print("rot", sc.gaussians.rot[:, i], "scale", sc.gaussians.scale[:, i], "op", sc.gaussians.opacity[i],
      "mean", sc.gaussians.mean[:, i])
g2 = r.grad2d.cpu().numpy().astype(np.float64)[:, i]
print("grad2d gpu", g2)
print("grad2d ora", ref[59:73, i])
print("rel 2d", np.abs(g2 - ref[59:73, i]) / np.maximum(np.abs(ref[59:73, i]), 1e-30))
print("norm rel drot", np.linalg.norm(drot - b) / np.linalg.norm(b))
print("dscale gpu/ora", out["dscale"].cpu().numpy()[:, i], ref[3:6, i])
