"""Stage-by-stage comparison of pifcm_segment against the oracle (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from inputs import add_noise_u8, cube_phantom
from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig, to_aos, to_pitched_x

ctx = Context(0)
dev = torch.device("cuda:0")
img, _ = cube_phantom(24, 20, 8, (0.1, 0.5, 0.9))
vol = add_noise_u8(img, 7.0, 3)
cfg = IfcmConfig(C=3)
for G in (1, 2, 4):
    pso = PsoConfig(P=4, max_gen=G, patience=0, seed=7)
    labels, U, rep = ctx.segment(torch.as_tensor(vol, device=dev), cfg, pso, want_U=True)
    r = oracle.segment_u8(vol, C=3, P=4, max_gen=G, seed=7)
    Ug = U.cpu().numpy()[:, :3]
    print(f"G={G} agree={(labels.cpu().numpy()==r.labels).mean():.4f} maxdU={np.abs(Ug-r.U).max():.3e}")
    print("  gpu", {k: rep[k] for k in ('lambda','xi','J','fcm_iters','final_iters','c_init','centers')})
    print("  orc", dict(lam=r.lam, xi=r.xi, J=r.J, final_iters=r.final_iters, c_init=r.c_init.tolist(), c=r.c.tolist()))
# final IFCM alone from the same state, iteration by iteration
x = oracle.normalize_u8(vol).astype(np.float32)
Uf, cf, _ = oracle.fcm_run(x, np.array([0.1,0.5,0.9]))
U = Uf.astype(np.float32); c = cf.astype(np.float32)
lam, xi = 1.0, 1.0
Ut = to_aos(U, dev).view(1, -1, 4); Uo = torch.empty_like(Ut)
cen = torch.zeros(1,4, device=dev); cen[0,:3] = torch.as_tensor(c)
lx = torch.tensor([[lam, xi]], dtype=torch.float64, device=dev)
Ug = U.astype(np.float64); co = c.astype(np.float64)
Uo_or = Ug.copy(); c_or = co.copy()
for it in range(30):
    prevU = Ut[0,:,:3].cpu().numpy().astype(np.float64); prevc = cen[0,:3].cpu().numpy().astype(np.float64)
    ctx.iterate(to_pitched_x(x, dev), Ut, Uo, cen, lx, IfcmConfig(C=3), nx=24)
    Us, cs, _, _ = oracle.ifcm_step(x, prevU, prevc, lam, xi)
    Uo_or, c_or, _, _ = oracle.ifcm_step(x, Uo_or, c_or, lam, xi)
    g = Uo[0,:,:3].cpu().numpy()
    print(it, "same-state diff %.2e" % np.abs(g - Us).max(), "chained diff %.2e" % np.abs(g - Uo_or).max(),
          "labels %.4f" % (g.argmax(1)==Uo_or.argmax(1)).mean())
    Ut, Uo = Uo, Ut
