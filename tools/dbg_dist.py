import os, sys, socket
sys.path.insert(0, os.getcwd())
import numpy as np, torch, torch.multiprocessing as mp
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_dist import _case, CFG, PSO, _port

def w(rank, world, port, P, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from dataclasses import replace
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    ctx = Context(0)
    ctx.attach_dist(rank, world, backend="host")
    vol = _case(40)
    a, b = ctx.dist_range(P, world, rank)
    pso = replace(PsoConfig(**dict(PSO, P=P)), p_begin=a, p_end=b)
    G = PSO["max_gen"]
    tf = torch.zeros((G, P), dtype=torch.float64, device="cuda:0"); tp = torch.zeros((G, P, 2), dtype=torch.float64, device="cuda:0"); tg = torch.zeros(G, dtype=torch.int32, device="cuda:0")
    ctx.pso_trace(tf, tp, tg)
    lab, _, rep = ctx.segment(torch.as_tensor(vol, device="cuda:0"), IfcmConfig(**CFG), pso)
    q.put((rank, lab.cpu().numpy(), rep, tf.cpu().numpy(), tg.cpu().numpy()))
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    from paper_2002_01981_b200 import Context, IfcmConfig, PsoConfig
    P, world = 5, 2
    ctx = Context(0)
    vol = _case(40)
    G = PSO["max_gen"]
    tf = torch.zeros((G, P), dtype=torch.float64, device="cuda:0"); tp = torch.zeros((G, P, 2), dtype=torch.float64, device="cuda:0"); tg = torch.zeros(G, dtype=torch.int32, device="cuda:0")
    ctx.pso_trace(tf, tp, tg)
    lab, _, rep = ctx.segment(torch.as_tensor(vol, device="cuda:0"), IfcmConfig(**CFG), PsoConfig(**dict(PSO, P=P)))
    print("single", rep, tf.cpu().numpy(), tg.cpu().numpy())
    cm = mp.get_context("spawn"); q = cm.Queue(); port = _port()
    ps = [cm.Process(target=w, args=(r, world, port, P, q)) for r in range(world)]
    [p.start() for p in ps]
    res = [q.get(timeout=200) for _ in range(world)]
    [p.join() for p in ps]
    for r, l, rp, f, g in res:
        print("rank", r, rp, "labels agree", (l == lab.cpu().numpy()).mean()); print(f, g)
