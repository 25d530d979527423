"""The check that replaces the label comparison where the final IFCM is ill
conditioned (lambda*, xi* both ~1: the chained map amplifies fp32-vs-fp64
rounding over up to 100 iterations, tests/test_oracle_chaos.py),
so two 100-iteration trajectories need not end in the same labels.  What the
north_star tolerance does fix there is one IFCM step from the same state:
from the GPU's final (U, c) -- deep in the ill-conditioned regime -- the GPU
step and the fp64 oracle step (Eq. 2-8) must agree within 1e-4
on every membership and 1e-4 relative on the centres."""
import numpy as np
import torch

U_TOL, C_TOL = 1e-4, 1e-4


def final_state_step_parity(ctx, orc, vol_t, U, centers, lam, xi, cfg):
    """U: [N, 4] f32 device (the pipeline's final memberships), centers: the
    final centres (C floats).  Returns (max |du|, max rel dc, label agreement
    of the two steps' argmax)."""
    dev = U.device
    nz, ny, nx = vol_t.shape
    x, _ = ctx.normalize(vol_t)
    N = nz * ny * nx
    C = cfg.C
    c4 = torch.zeros((1, 4), dtype=torch.float32, device=dev)
    c4[0, :C] = torch.as_tensor(np.asarray(centers, dtype=np.float32), device=dev)
    Ui = U.reshape(1, N, 4).contiguous()
    Uo = torch.empty_like(Ui)
    lx = torch.tensor([[lam, xi]], dtype=torch.float64, device=dev)
    cin = c4[0, :C].cpu().numpy().astype(np.float64)
    ctx.iterate(x, Ui, Uo, c4, lx, cfg, iters=1, nx=nx)
    xn = x[..., :nx].cpu().numpy().astype(np.float64)
    Un = Ui[0, :, :C].cpu().numpy().astype(np.float64)
    Ur, cr, _, _ = orc.ifcm_step(xn, Un, cin, lam, xi, m=cfg.m, q_mode=cfg.q_mode, v=cfg.v, h=cfg.h)
    Ug = Uo[0, :, :C].cpu().numpy()
    du = float(np.abs(Ug - Ur).max())
    dc = float(np.max(np.abs(c4[0, :C].cpu().numpy() - cr) / np.abs(cr)))
    agree = float((Ug.argmax(1) == Ur.argmax(1)).mean())
    assert du <= U_TOL and dc <= C_TOL, (du, dc, lam, xi)
    return du, dc, agree
