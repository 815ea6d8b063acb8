"""Diagnostic (build with -DPGSAG_A7_STATS): A7's tail on C4 views -- per persistent CTA, the time it
finished relative to the kernel start; how long the grid runs with fewer than half / 90 % of its CTAs."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from synth import scenes as S
from paper_2501_01677_b200 import _lib
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

dev = torch.device("cuda", 0)
lib = ctypes.CDLL(_lib.LIB_PATH)
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
if cfg == "c4":
    sub = S.subregion(0, n_views=2)
    items = [(sub["gaussians"], c, S.ray_cast_mask(c, sub["boxes"], device=dev)) for c in sub["cameras"]]
else:
    sc = {"c5": S.config5, "c3": S.config3}[cfg](device=dev)
    items = [(sc.gaussians, sc.camera, sc.mask)]
for gnp, c, mnp in items:
    g = GaussianTensors.from_numpy(gnp, dev)
    m = torch.from_numpy(np.ascontiguousarray(mnp)).to(dev)
    H, W = m.shape
    r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
    gen = torch.Generator(device=dev); gen.manual_seed(0)
    up = dict(dC=torch.randn(3, H, W, device=dev, generator=gen), dN=torch.randn(3, H, W, device=dev, generator=gen),
              dD=torch.randn(H, W, device=dev, generator=gen), dA=torch.randn(H, W, device=dev, generator=gen),
              dDep=torch.randn(H, W, device=dev, generator=gen))
    for _ in range(2):
        r.forward(g, camera_from(c), m)
        r.backward(**up)
    torch.cuda.synchronize()
    n = 148 * 20
    t0 = (ctypes.c_ulonglong * 1)()
    ends = (ctypes.c_ulonglong * n)()
    lib.pgsag_debug_a7_times(t0, ends, n)  # reset
    r.forward(g, camera_from(c), m)
    r.backward(**up)
    torch.cuda.synchronize()
    lib.pgsag_debug_a7_times(t0, ends, n)
    e = (np.array(ends[:n], dtype=np.float64) - t0[0]) / 1e3  # us
    e.sort()
    tot = e[-1]
    print(f"{cfg}: A7 span {tot:.0f} us; CTAs done at p10 {np.percentile(e, 10):.0f} p50 {np.percentile(e, 50):.0f} "
          f"p90 {np.percentile(e, 90):.0f} max {tot:.0f} us; time with < 50 % of CTAs running "
          f"{tot - np.percentile(e, 50):.0f} us ({100 * (tot - np.percentile(e, 50)) / tot:.1f} %)")
    del r
