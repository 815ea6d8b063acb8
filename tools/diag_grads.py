"""Dump GPU vs oracle gradients (incl. A7 2D grads) for a scene into gpurun_out/diag_grads.npz."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from tests.gpu_util import upstream_at
from tests.test_gpu_parity import ragged_scene

sc = ragged_scene()
H, W = sc.mask.shape
bg = (0.3, 0.1, 0.2)
pix = np.flatnonzero(sc.mask.reshape(-1))
ora0 = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg)
planes, per = upstream_at(pix, H, W, seed=3, exclude=ora0["near"].astype(bool))
g = GaussianTensors.from_numpy(sc.gaussians)
r = Rasterizer(g.n, W, H, g.sh_degree)
r.export_grad2d(True)
r.forward(g, camera_from(sc.camera), torch.from_numpy(sc.mask).cuda(), bg)
out = r.backward(**{k: torch.from_numpy(v).cuda() for k, v in planes.items()})
torch.cuda.synchronize()
ora = oracle.render(sc.gaussians, sc.camera, sc.mask, pix, bg=bg, upstream=per)
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/diag_grads.npz", ref=ora["grads"], **{k: v.cpu().numpy() for k, v in out.items()})
print("saved")
