"""Where the e2e training step's time goes on one C4 sub-region: Trainer.step with precomputed Eq. 9
weights / band, Trainer.step_photo on a device-resident photo (weights and band derived each
step on the side stream), and the same plus the 8-bit unpack.  Device ms per iteration."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200 import _lib as L
from paper_2501_01677_b200.raster import GaussianTensors, Rasterizer, camera_from
from paper_2501_01677_b200.train import Trainer

dev = torch.device("cuda", 0)
sub = S.subregion(0, n_views=5)
cams = [camera_from(c) for c in sub["cameras"]]
masks = [torch.from_numpy(S.ray_cast_mask(c, sub["boxes"], device=dev)).to(dev) for c in sub["cameras"]]
g = GaussianTensors.from_numpy(sub["gaussians"], dev)
H, W = masks[0].shape
r = Rasterizer(g.n, W, H, g.sh_degree, capacity=24 * g.n, device=dev, counters=False, sat=False)
tr = Trainer(r, g)
gen = torch.Generator(device=dev)
gen.manual_seed(0)
tgt = torch.rand(3, H, W, device=dev, generator=gen)
t8 = (tgt * 255).round().to(torch.uint8).permute(1, 2, 0).contiguous()
extras = [(r.gc_weights(tgt, m), r.boundary_band(m, 1)) for m in masks]
st = torch.cuda.current_stream().cuda_stream


def timed(fn, k=5):
    for v in range(2):
        fn(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for v in range(k):
        fn(v)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


print("E2E step(precomputed)", round(timed(lambda v: tr.step(cams[v], masks[v], tgt, gc_w=extras[v][0],
                                                            band=extras[v][1])), 3))
print("E2E step_photo(device)", round(timed(lambda v: tr.step_photo(cams[v], masks[v], tgt)), 3))
buf = torch.empty_like(tgt)


def with_unpack(v):
    L.unpack_rgb8(t8.data_ptr(), W, H, buf.data_ptr(), st)
    tr.step_photo(cams[v], masks[v], buf)


print("E2E unpack+step_photo", round(timed(with_unpack), 3))
L.timing_enable(True)
L.timing_collect()
timed(lambda v: tr.step_photo(cams[v], masks[v], tgt))
L.timing_enable(False)
print("E2E kernels", {k: round(v[0] / 7, 4) for k, v in sorted(L.timing_collect().items())})
