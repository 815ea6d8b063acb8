"""Experiment (debug build with -DPGSAG_HIST): histogram of contributing lanes / pixels per
(warp, candidate) in A7 on one C4 view."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from synth import scenes as S
from paper_2501_01677_b200 import shard
sub = S.subregion(shard.weak_region(0), n_views=1)
cam = sub["cameras"][0]
mask = torch.from_numpy(S.ray_cast_mask(cam, sub["boxes"], device="cuda")).cuda()
g = GaussianTensors.from_numpy(sub["gaussians"])
r = Rasterizer(g.n, cam.width, cam.height, g.sh_degree, capacity=24 * g.n, sat=False)
cnt = torch.zeros(80, dtype=torch.int64, device="cuda")
r.counters = cnt
r._img.counters = cnt.data_ptr()
r.forward(g, camera_from(cam), mask)
H, W = mask.shape
up = {k: torch.randn(*s, device="cuda") for k, s in (("dC", (3, H, W)), ("dN", (3, H, W)), ("dD", (H, W)),
                                                      ("dA", (H, W)), ("dDep", (H, W)))}
r.backward(**up)
torch.cuda.synchronize()
c = cnt.cpu().numpy()
lanes = c[4:37]
pix = c[40:73]
tot = lanes.sum()
print("warp-candidates with work:", tot, " E", c[0], "B", c[1], "V", c[2])
print("lanes hist (frac):", " ".join(f"{k}:{lanes[k]/tot:.3f}" for k in range(33) if lanes[k]))
print("mean lanes", (np.arange(33) * lanes).sum() / tot)
print("px/4 hist:", " ".join(f"{4*k}:{pix[k]/tot:.3f}" for k in range(33) if pix[k]))
print("cum lanes<=4:", lanes[:5].sum()/tot, "<=8:", lanes[:9].sum()/tot, "<=16:", lanes[:17].sum()/tot)
