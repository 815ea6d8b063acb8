"""pgsag_boundary_band alone on a C4 view's building mask: mean device ms (r = 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import scenes as S
from paper_2501_01677_b200 import _lib as L

dev = torch.device("cuda", 0)
sub = S.subregion(0, n_views=1)
mask = torch.from_numpy(S.ray_cast_mask(sub["cameras"][0], sub["boxes"], device=dev)).to(dev)
H, W = mask.shape
band = torch.empty_like(mask)
st = torch.cuda.current_stream().cuda_stream
call = lambda: L.boundary_band(mask.data_ptr(), W, H, 1, band.data_ptr(), st)
for _ in range(3):
    call()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    call()
e1.record()
torch.cuda.synchronize()
print("BAND", round(e0.elapsed_time(e1) / 50, 4))
