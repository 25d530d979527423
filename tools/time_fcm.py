"""Device time of the pointwise FCM step (lambda = xi = 0) on C3 (never a bench value)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from inputs import config_volume
from paper_2002_01981_b200 import Context, IfcmConfig

ctx = Context(0)
vol, _ = config_volume("C3")
nz, ny, nx = vol.shape
x, hist = ctx.normalize_u8(torch.as_tensor(vol, device="cuda:0"))
c0 = ctx.gmm_init(hist, 4).view(1, 4)
U = torch.full((1, nz * ny * nx, 4), 0.25, device="cuda:0")
Uo = torch.empty_like(U)
lx = torch.zeros((1, 2), dtype=torch.float64, device="cuda:0")
st = torch.zeros((1, 4), dtype=torch.float64, device="cuda:0")
cfg = IfcmConfig(C=4, eps=0.0)
for _ in range(3):
    ctx.iterate(x, U, Uo, c0.clone(), lx, cfg, iters=1, stats=st, nx=nx)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ctx.iterate(x, U, Uo, c0.clone(), lx, cfg, iters=1, stats=st, nx=nx)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"pointwise FCM step (incl. launch overheads of iterate): {ms * 1e3:.1f} us, "
      f"{(nz * ny * nx * 36) / (ms * 1e-3) / 1e9:.0f} GB/s")
