"""Find non-finite values in a C4 training run (bench's train_step setup): after each
Trainer.step, count non-finite gradients / parameters / moments and show the first offenders."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from paper_2501_01677_b200.train import Trainer

dev = torch.device("cuda", 0)
sub = S.subregion(0, n_views=int(sys.argv[1]) if len(sys.argv) > 1 else 6)
cams = sub["cameras"]
masks = [torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=dev)).to(dev) for c in cams]
g = GaussianTensors.from_numpy(sub["gaussians"], dev)
H, W = masks[0].shape
r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=True, sat=False)
tr = Trainer(r, g)
gen = torch.Generator(device=dev)
gen.manual_seed(1677)
tgt = torch.rand(3, H, W, device=dev, generator=gen)
print("init: log_scale finite", bool(torch.isfinite(tr.log_scale).all()), "logit_op finite",
      bool(torch.isfinite(tr.logit_opacity).all()), "min scale", float(g.scale.min()), "op range",
      float(g.opacity.min()), float(g.opacity.max()))
for it, c in enumerate(cams):
    cc = camera_from(c)
    tr.step(cc, masks[it], tgt, gc_w=r.gc_weights(tgt, masks[it]), band=r.boundary_band(masks[it], 1))
    torch.cuda.synchronize()
    rep = {}
    for k in ("dmean", "dscale", "drot", "dopacity"):
        t = getattr(r, k)
        rep[k] = int((~torch.isfinite(t)).sum())
    for k, t in (("scale", tr.g.scale), ("log_scale", tr.log_scale), ("m", tr.m), ("v", tr.v),
                 ("mean", tr.g.mean), ("opacity", tr.g.opacity)):
        rep[k] = int((~torch.isfinite(t)).sum())
    for k, t in (("dC", tr.dC), ("dN", tr.dN), ("dDep", tr.dDep), ("img_N", r.img_N), ("img_Dep", r.img_Dep),
                 ("img_C", r.img_C), ("img_D", r.img_D)):
        rep[k] = int((~torch.isfinite(t)).sum())
    print(it, tr.losses(), rep, flush=True)
    if rep["dN"] or rep["dDep"]:
        bad = (~torch.isfinite(tr.dDep)) | (~torch.isfinite(tr.dN)).any(0)
        ys, xs = bad.nonzero(as_tuple=True)
        y, x = int(ys[0]), int(xs[0])
        print("  bad pixels", int(bad.sum()), "first", x, y)
        sl = (slice(max(y - 1, 0), y + 2), slice(max(x - 1, 0), x + 2))
        print("  Dep", r.img_Dep[sl].tolist())
        print("  N", r.img_N[(slice(None),) + sl].tolist())
        print("  mask", masks[it][sl].tolist(), "band", r.boundary_band(masks[it], 1)[sl].tolist())
        print("  g", r.img_g[sl].tolist(), "T", r.img_T[sl].tolist())
        print("  dN", tr.dN[(slice(None),) + sl].tolist(), "dDep", tr.dDep[sl].tolist())
    for k in ("dscale", "dmean", "drot", "dopacity"):
        t = getattr(r, k).reshape(-1, g.n)
        bad = (~torch.isfinite(t)).any(0).nonzero().flatten()
        if bad.numel():
            i = int(bad[0])
            print("  first bad", k, i, "grad", t[:, i].tolist(), "scale", g.scale[:, i].tolist(), "rot",
                  g.rot[:, i].tolist(), "op", float(g.opacity[i]), "mean", g.mean[:, i].tolist())
            break
    bad = (~torch.isfinite(tr.g.scale)).any(0).nonzero().flatten()
    if bad.numel():
        i = int(bad[0])
        print("  first bad scale", i, tr.g.scale[:, i].tolist(), tr.log_scale[:, i].tolist(), "m", tr.m[3:6, i].tolist(),
              "v", tr.v[3:6, i].tolist())
