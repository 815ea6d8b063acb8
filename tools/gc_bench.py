"""pgsag_gc_weights (Sobel + normalise) alone on a C4-sized image and mask: mean device ms."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200 import _lib as L

dev = torch.device("cuda", 0)
sub = S.subregion(0, n_views=1)
mask = torch.from_numpy(S.ray_cast_mask(sub["cameras"][0], sub["boxes"], device=dev)).to(dev)
H, W = mask.shape
gen = torch.Generator(device=dev)
gen.manual_seed(0)
img = torch.rand(3, H, W, device=dev, generator=gen)
w = torch.empty(H, W, device=dev)
nb = L.workspace_size(0, W, H, 0)
ws = torch.empty(max(nb, 256), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
call = lambda: L.gc_weights(img.data_ptr(), mask.data_ptr(), W, H, w.data_ptr(), ws.data_ptr(), nb, st)
for _ in range(3):
    call()
L.timing_enable(True)
L.timing_collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30):
    call()
e1.record()
torch.cuda.synchronize()
L.timing_enable(False)
print("GC", round(e0.elapsed_time(e1) / 30, 4), {k: round(v[0] / 30, 4) for k, v in L.timing_collect().items()})
