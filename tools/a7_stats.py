"""Diagnostic: A7 candidate-loop work statistics on C4 views (build with -DPGSAG_A7_STATS)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200 import _lib
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

dev = torch.device("cuda", 0)
lib = ctypes.CDLL(_lib.LIB_PATH)
f = lib.pgsag_debug_a7_stats
buf = (ctypes.c_ulonglong * 32)()
tot = [0] * 32
for region in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    sub = S.subregion(region, n_views=2)
    gnp, cams = sub["gaussians"], sub["cameras"]
    g = GaussianTensors.from_numpy(gnp, dev)
    for c in cams:
        m = torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=dev)).to(dev)
        H, W = m.shape
        r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
        r.forward(g, camera_from(c), m)
        gen = torch.Generator(device=dev); gen.manual_seed(0)
        r.backward(dC=torch.randn(3, H, W, device=dev, generator=gen), dN=torch.randn(3, H, W, device=dev, generator=gen),
                   dD=torch.randn(H, W, device=dev, generator=gen), dA=torch.randn(H, W, device=dev, generator=gen),
                   dDep=torch.randn(H, W, device=dev, generator=gen))
        f(buf, 1)
        tot = [a + b for a, b in zip(tot, buf)]
        del r
names = {0: "visited", 1: "anyc", 2: "pairs_eval", 3: "pairs_contrib", 4: "blended_px"}
for k, n in names.items():
    print(f"{n:14s} {tot[k]:14d}")
print("per anyc entry: blended px %.1f, pairs %.2f" % (tot[4] / tot[1], tot[3] / tot[1]))
print("lanes hist (1,2,<=4,<=8,<=16,<=32):", [round(tot[8 + i] / tot[1], 3) for i in range(6)])
print("blend hist (<=2,4,8,16,32,64,128):", [round(tot[16 + i] / tot[1], 3) for i in range(7)])
