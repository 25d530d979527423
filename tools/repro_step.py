import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from inputs import random_state
from paper_2002_01981_b200 import Context, IfcmConfig, to_aos, to_pitched_x
ctx = Context(0)
dev = torch.device("cuda:0")
nx, ny, nz = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
x, U, c = random_state(nx, ny, nz, 4, seed=1)
Ut = to_aos(U, dev).view(1, -1, 4); Uo = torch.empty_like(Ut)
cen = torch.as_tensor(c, device=dev).view(1, 4).clone()
lx = torch.tensor([[0.6, 0.8]], dtype=torch.float64, device=dev)
ctx.iterate(to_pitched_x(x, dev), Ut, Uo, cen, lx, IfcmConfig(C=4), nx=nx)
torch.cuda.synchronize()
print("ok", Uo[0, :3].cpu().numpy())
