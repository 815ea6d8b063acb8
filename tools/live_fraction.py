"""Diagnostic: fraction of Gaussians that emit entries (flags LIVE) per C4 view, and M per view."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
dev = torch.device("cuda", 0)
for region in range(3):
    sub = S.subregion(region, n_views=2)
    g = GaussianTensors.from_numpy(sub["gaussians"], dev)
    for c in sub["cameras"]:
        m = torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=dev)).to(dev)
        H, W = m.shape
        r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
        r.forward(g, camera_from(c), m)
        fl = r.flags[:g.n].view(torch.int32)
        live = ((fl & 15) == 15).sum().item()
        vis = ((fl & 1) == 1).sum().item()
        print(f"region {region}: n {g.n} visible {vis} live {live} ({100 * live / g.n:.1f} %) M {r.M}")
        del r
