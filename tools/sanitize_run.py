"""One A0-A8 pass (forward + backward) on C1 and on a C2-shaped scene (30k Gaussians, 1080p), plus
one training iteration (NEXT-rows) on C1, for compute-sanitizer (memcheck / racecheck / synccheck,
SURVEY §5): every pgsag kernel of the path runs at least once, in both the synchronising and the
sync-free sort configuration, then exits 0."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from paper_2501_01677_b200.train import Trainer

dev = torch.device("cuda", 0)
for name, sc in (("C1", S.config1()), ("C2s", S.config2(n=30000))):
    H, W = sc.mask.shape
    g = GaussianTensors.from_numpy(sc.gaussians, dev)
    mask = torch.from_numpy(np.ascontiguousarray(sc.mask)).to(dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    up = {"dC": torch.randn(3, H, W, device=dev, generator=gen), "dN": torch.randn(3, H, W, device=dev, generator=gen),
          "dD": torch.randn(H, W, device=dev, generator=gen), "dA": torch.randn(H, W, device=dev, generator=gen),
          "dDep": torch.randn(H, W, device=dev, generator=gen)}
    for sync_free in (False, True):
        r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, counters=True, sync_free=sync_free, absgrad=True)
        r.export_grad2d(True)
        r.forward(g, camera_from(sc.camera), mask, (0.1, 0.2, 0.3))
        r.backward(**up)
        torch.cuda.synchronize()
        assert r.check_capacity()
    if name == "C1":
        tgt = torch.from_numpy(S.reference_image(H, W, 3)).to(dev)
        r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, sync_free=True)
        tr = Trainer(r, g)
        tr.step_photo(camera_from(sc.camera), mask, tgt)
        tr.losses()
        tr.densify()
        tr.reset_opacity()
        torch.cuda.synchronize()
    print(name, "ok", flush=True)
