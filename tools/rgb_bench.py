"""pgsag_rgb_loss (value + gradient) alone on a C4-sized image and building mask: mean device ms."""
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
C, I = torch.rand(3, H, W, device=dev, generator=gen), torch.rand(3, H, W, device=dev, generator=gen)
loss = torch.zeros(6, dtype=torch.float64, device=dev)
dC = torch.empty(3, H, W, device=dev)
nb = L.rgb_loss_workspace_size(W, H)
ws = torch.empty(nb, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
call = lambda: L.rgb_loss(C.data_ptr(), I.data_ptr(), mask.data_ptr(), W, H, 0.59, loss.data_ptr(), dC.data_ptr(),
                          ws.data_ptr(), nb, st)
for _ in range(3):
    call()
L.timing_enable(True)
L.timing_collect()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    call()
e1.record()
torch.cuda.synchronize()
L.timing_enable(False)
tk = L.timing_collect()
print("RGB", round(e0.elapsed_time(e1) / 20, 4), {k: round(v[0] / 20, 4) for k, v in tk.items()})
