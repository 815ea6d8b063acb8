"""Experiment: the 8-region C4 step on one stream (one rasterizer) vs alternating two streams with a
rasterizer each (region r's backward can overlap region r+1's forward / sort).  Device ms per step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from

dev = torch.device("cuda", 0)
regs = []
for k in range(8):
    sub = S.subregion(k, n_views=2)
    regs.append(dict(g=GaussianTensors.from_numpy(sub["gaussians"], dev), cams=[camera_from(c) for c in sub["cameras"]],
                     masks=[torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=dev)).to(dev) for c in sub["cameras"]]))
H, W = regs[0]["masks"][0].shape
gen = torch.Generator(device=dev); gen.manual_seed(1677)
up = {"dC": torch.randn(3, H, W, device=dev, generator=gen), "dN": torch.randn(3, H, W, device=dev, generator=gen),
      "dD": torch.randn(H, W, device=dev, generator=gen), "dA": torch.randn(H, W, device=dev, generator=gen),
      "dDep": torch.randn(H, W, device=dev, generator=gen)}
NS = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rs = [Rasterizer(1500000, W, H, 3, capacity=int(1.15 * 9.5e6), device=dev, counters=False, sat=False) for _ in range(NS)]
for r in rs:
    r.sync_free = True
streams = [torch.cuda.Stream(device=dev) for _ in range(NS)]


def step(s, ns):
    main = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(main)
    for ri in range(8):
        k = ri % ns
        st = streams[k]
        st.wait_event(ev)
        with torch.cuda.stream(st):
            rg = regs[ri]
            v = s % 2
            rs[k].forward(rg["g"], rg["cams"][v], rg["masks"][v])
            rs[k].backward(**up)
    for k in range(ns):
        e = torch.cuda.Event()
        e.record(streams[k])
        main.wait_event(e)


for ns in (1, NS, 1, NS):
    for s in range(3):
        step(s, ns)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(6):
        step(s, ns)
    e1.record()
    torch.cuda.synchronize()
    ok = all(r.check_capacity() for r in rs)
    print(f"streams {ns}: {e0.elapsed_time(e1) / 6:.3f} ms per 8-view step (capacity ok {ok})", flush=True)
