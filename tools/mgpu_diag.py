"""Developer diagnostic (torchrun): where the distributed K' product differs from the single-GPU
one -- per-rank relative error of the owned rows, the largest differences and whether their panels'
leaves touch a rank boundary; for the FMM product, the near field alone (far field off is not
exposed, so the same with the plain P2P form) and the potential operator."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_1007_4591_b200 import Solver
from synth import configs
from mgpu_check import gather, rel


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.lysozyme(113)
    leaf = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    opts = dict(terms=13, leaf_points=leaf, device=local)
    n = len(cfg["triangles"])
    x = np.random.default_rng(3).normal(size=n)
    s1 = Solver.from_config(cfg, **opts)
    dev = lambda s, v: torch.tensor(v[s.local_ids], dtype=torch.float32, device="cuda")
    s = Solver.distributed(cfg, **opts)
    res = {"env": {k: v for k, v in os.environ.items() if k.startswith("FMMBEM")}, "leaf": leaf}
    for op in ("kprime", "single", "double"):
        y1 = s1.to_global(s1.matvec(dev(s1, x), op).cpu().numpy())
        y = gather(s, s.matvec(dev(s, x), op))
        d = np.abs(y - y1)
        top = np.argsort(-d)[:8]
        res[op] = {"rel": rel(y, y1), "max_abs": float(d.max()), "scale": float(np.abs(y1).max()),
                   "top": [[int(i), float(d[i]), float(y1[i])] for i in top]}
    # which rank owns the top panels
    ids = [None] * world
    dist.all_gather_object(ids, s.local_ids)
    owner = np.empty(n, np.int64)
    for r, ii in enumerate(ids):
        owner[ii] = r
    res["top_owner"] = [int(owner[i]) for i, _, _ in res["kprime"]["top"]]
    if rank == 0:
        print("DIAG", json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
