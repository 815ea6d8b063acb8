"""pgsag_ban_loss (one pass: loss sums + gradient scatter) alone on a C4 view's A6 outputs: mean device ms."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200 import _lib as L
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

dev = torch.device("cuda", 0)
sub = S.subregion(0, n_views=1)
cam = sub["cameras"][0]
mask = torch.from_numpy(S.ray_cast_mask(cam, sub["boxes"], device=dev)).to(dev)
g = GaussianTensors.from_numpy(sub["gaussians"], dev)
H, W = mask.shape
r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
r.forward(g, camera_from(cam), mask)
band = r.boundary_band(mask, 1)
dN = torch.zeros(3, H, W, device=dev)
dDep = torch.zeros(H, W, device=dev)
call = lambda: r.ban_loss(band, lam=0.01, bw=0.1, mean=False, dN=dN, dDep=dDep)
for _ in range(3):
    call()
L.timing_enable(True)
L.timing_collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    call()
e1.record()
torch.cuda.synchronize()
L.timing_enable(False)
tk = L.timing_collect()
print("BAN", round(e0.elapsed_time(e1) / 20, 4), {k: round(v[0] / 20, 4) for k, v in tk.items()})
