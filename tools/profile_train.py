"""Run a few NEXT-3 training iterations on one C4 view (for ncu captures of the N* kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from paper_2501_01677_b200.train import Trainer

dev = torch.device("cuda", 0)
sub = S.subregion(0, n_views=1)
cam = sub["cameras"][0]
mask = torch.from_numpy(S.ray_cast_mask(cam, sub["boxes"], device=dev)).to(dev)
g = GaussianTensors.from_numpy(sub["gaussians"], dev)
H, W = mask.shape
r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
tr = Trainer(r, g)
gen = torch.Generator(device=dev); gen.manual_seed(0)
tgt = torch.rand(3, H, W, device=dev, generator=gen)
gc_w, band = r.gc_weights(tgt, mask), r.boundary_band(mask, 1)
for _ in range(2):
    tr.step(camera_from(cam), mask, tgt, gc_w=gc_w, band=band)
torch.cuda.synchronize()
print("done", tr.losses())
