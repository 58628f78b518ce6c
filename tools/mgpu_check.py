"""Multi-GPU parity check (run under torchrun): the distributed matvec / solve / BIBEE equal the
single-GPU results.  Not a pytest (needs N GPUs); tests/test_gpu_multigpu.py drives it."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
from paper_1007_4591_b200 import Solver
from synth import configs

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
name = sys.argv[1] if len(sys.argv) > 1 else "lyso40"
cfg = {"lyso40": lambda: configs.lysozyme(40, 400), "kirk32": lambda: configs.kirkwood(32),
       "c3": lambda: configs.lysozyme(113)}[name]()
opts = dict(terms=12, leaf_points=32, device=local)
s = Solver.distributed(cfg, **opts)
n = len(cfg["triangles"])
x = np.random.default_rng(3).normal(size=n)
y = s.matvec(torch.tensor(x[s.local_ids], dtype=torch.float32, device="cuda"), "kprime")
torch.cuda.synchronize()
parts = [None] * world
dist.all_gather_object(parts, (s.local_ids, y.cpu().numpy()))
yh = s.matvec_host(x[s.local_ids].astype(np.float32), "kprime")  # plain host-buffer path (N > 1)
host_rel = float(np.linalg.norm(yh - y.cpu().numpy()) / np.linalg.norm(y.cpu().numpy()))
s_st = Solver.distributed(cfg, self_term=1, **opts)  # curvature self-term option (A7) across ranks
y_st = s_st.matvec(torch.tensor(x[s_st.local_ids], dtype=torch.float32, device="cuda"), "A")
torch.cuda.synchronize()
parts_st = [None] * world
dist.all_gather_object(parts_st, (s_st.local_ids, y_st.cpu().numpy(), host_rel))
r = s.solve()
b = s.bibee("cfa")
out = {}
if rank == 0:
    yd = np.empty(n)
    for ids, yy in parts:
        yd[ids] = yy
    s1 = Solver.from_config(cfg, terms=12, leaf_points=32, device=local)
    y1 = s1.to_global(s1.matvec(torch.tensor(s1.to_local(x), dtype=torch.float32, device="cuda"), "kprime").cpu().numpy())
    r1 = s1.solve()
    b1 = s1.bibee("cfa")
    yst = np.empty(n)
    for ids, yy, _ in parts_st:
        yst[ids] = yy
    s1st = Solver.from_config(cfg, self_term=1, terms=12, leaf_points=32, device=local)
    y1st = s1st.to_global(s1st.matvec(torch.tensor(s1st.to_local(x), dtype=torch.float32, device="cuda"),
                                       "A").cpu().numpy())
    out = dict(world=world, n_local=[len(p[0]) for p in parts],
               matvec_rel=float(np.linalg.norm(yd - y1) / np.linalg.norm(y1)),
               self_term_rel=float(np.linalg.norm(yst - y1st) / np.linalg.norm(y1st)),
               host_rel=max(p[2] for p in parts_st),
               solve=(r["dG"], r1["dG"], r["iterations"], r1["iterations"]), bibee=(b["dG"], b1["dG"]))
    print("MGPU", json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
