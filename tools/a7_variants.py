"""A7 time inside Trainer.step on one C4 view with and without the L_GC-load (soft-count) and
L_ban upstream terms, to attribute the training step's A7 cost."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200 import _lib as L
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from paper_2501_01677_b200.train import AdamConfig, Trainer

dev = torch.device("cuda", 0)
sub = S.subregion(0, n_views=1)
cam = sub["cameras"][0]
mask = torch.from_numpy(S.ray_cast_mask(cam, sub["boxes"], device=dev)).to(dev)
g = GaussianTensors.from_numpy(sub["gaussians"], dev)
H, W = mask.shape
r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
tr = Trainer(r, g, AdamConfig(0, 0, 0, 0, 0, 0))  # zero learning rates: the scene stays fixed
gen = torch.Generator(device=dev)
gen.manual_seed(0)
tgt = torch.rand(3, H, W, device=dev, generator=gen)
gc_w, band = r.gc_weights(tgt, mask), r.boundary_band(mask, 1)
cc = camera_from(cam)
for name, kw in (("gc+ban", dict(gc_w=gc_w, band=band)), ("ban", dict(band=band)), ("gc", dict(gc_w=gc_w)),
                 ("rgb only", {}), ("gc+ban again", dict(gc_w=gc_w, band=band))):
    for _ in range(2):
        tr.step(cc, mask, tgt, **kw)
    torch.cuda.synchronize()
    L.timing_enable(True)
    L.timing_collect()
    for _ in range(5):
        tr.step(cc, mask, tgt, **kw)
    torch.cuda.synchronize()
    L.timing_enable(False)
    tk = L.timing_collect()
    print(f"{name:14s}", {k: round(v[0] / 5, 4) for k, v in sorted(tk.items()) if k.startswith(("A6", "A7", "A8"))},
          flush=True)
