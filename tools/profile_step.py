"""Run the C4 hot path for a few views (for ncu / nsys-style profiling)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--config", default="c4")
a = ap.parse_args()
dev = torch.device("cuda", 0)
if a.config == "c4":
    sub = S.subregion(0, n_views=2)
    gnp, cams = sub["gaussians"], sub["cameras"]
    masks = [torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=dev)).to(dev) for c in cams]
else:
    sc = {"c2": S.config2, "c3": S.config3, "c5": S.config5}[a.config](device=dev)
    gnp, cams, masks = sc.gaussians, [sc.camera], [torch.from_numpy(sc.mask).to(dev)]
g = GaussianTensors.from_numpy(gnp, dev)
H, W = masks[0].shape
r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
gen = torch.Generator(device=dev); gen.manual_seed(0)
up = {"dC": torch.randn(3, H, W, device=dev, generator=gen), "dN": torch.randn(3, H, W, device=dev, generator=gen),
      "dD": torch.randn(H, W, device=dev, generator=gen), "dA": torch.randn(H, W, device=dev, generator=gen),
      "dDep": torch.randn(H, W, device=dev, generator=gen)}
for s in range(a.steps):
    v = s % len(cams)
    r.forward(g, camera_from(cams[v]), masks[v])
    r.backward(**up)
torch.cuda.synchronize()
print("done M=", r.M)
