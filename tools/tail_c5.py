"""Per-tile backward work on C5 (maxlast - range start over the tile's mask pixels) vs the A7 time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from paper_2501_01677_b200 import _lib as L
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
sc = {"c5": S.config5, "c3": S.config3}[cfg](device="cuda")
g = GaussianTensors.from_numpy(sc.gaussians)
H, W = sc.mask.shape
r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, counters=False, sat=False)
mask = torch.from_numpy(sc.mask).cuda()
cam = camera_from(sc.camera)
up = {k: torch.randn(*s, device="cuda") for k, s in (("dC", (3, H, W)), ("dN", (3, H, W)), ("dD", (H, W)),
                                                      ("dA", (H, W)), ("dDep", (H, W)))}
for _ in range(2):
    r.forward(g, cam, mask); r.backward(**up)
torch.cuda.synchronize()
L.timing_enable(True); L.timing_collect()
r.forward(g, cam, mask); r.backward(**up)
torch.cuda.synchronize()
L.timing_enable(False); kt = L.timing_collect()
last = r.img_last.clone(); last[mask == 0] = -1
pad = lambda t, v: torch.nn.functional.pad(t, (0, (16 - W % 16) % 16, 0, (16 - H % 16) % 16), value=v)
lt = pad(last, -1).reshape((H + 15) // 16, 16, (W + 15) // 16, 16).amax(dim=(1, 3)).reshape(-1)
rg = r.ranges.view(-1, 2).long()
work = torch.where(lt >= 0, lt - rg[:, 0] + 1, torch.zeros_like(lt)).double()
act = work[work > 0]
print("A6 ms", kt["A6_render_fwd"][0], "A7 ms", kt["A7_render_bwd"][0])
print("tiles", act.numel(), "entries to walk: mean", float(act.mean()), "p99", float(torch.quantile(act, 0.99)),
      "max", float(act.max()), "sum", float(act.sum()))
print("raw list len max", int((rg[:, 1] - rg[:, 0]).max()))
# lower bound if the heaviest tile's walk ran at the average per-entry rate of the whole kernel
per_entry_ms = kt["A7_render_bwd"][0] / float(act.sum()) * 1480  # 1480 CTAs in flight
print("tail bound (heaviest tile alone, ms) ~", float(act.max()) * per_entry_ms)
