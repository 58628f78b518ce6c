"""Multi-GPU parity check (run under torchrun): the distributed matvec / solve / BIBEE / reaction
potential equal the single-GPU results, for input_mode 0 (full mesh on every rank) and 1 (every rank
passes only its part of the mesh), with the self-term and analytic near-field options (mode 0).
Not a pytest (needs N GPUs); tests/test_gpu_multigpu.py drives it."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

from paper_1007_4591_b200 import Solver
from synth import configs


def part_of(cfg, rank, world):
    """Rank's contiguous block of triangles with its own (compacted) vertex array: global ids of
    input_mode 1 are then the triangle indices."""
    t = cfg["triangles"]
    n = len(t)
    lo, hi = n * rank // world, n * (rank + 1) // world
    tt = t[lo:hi]
    used, inv = np.unique(tt.reshape(-1), return_inverse=True)
    return dict(cfg, vertices=cfg["vertices"][used], triangles=inv.reshape(-1, 3).astype(np.int32))


def gather(s, y):
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (s.local_ids, y.cpu().numpy()))
    n = sum(len(p[0]) for p in parts)
    out = np.empty(n)
    for ids, yy in parts:
        out[ids] = yy
    return out


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = sys.argv[1] if len(sys.argv) > 1 else "lyso40"
    cfg = {"lyso40": lambda: configs.lysozyme(40, 400), "kirk32": lambda: configs.kirkwood(32),
           "c3": lambda: configs.lysozyme(113)}[name]()
    opts = dict(terms=13, leaf_points=32, device=local)
    n = len(cfg["triangles"])
    x = np.random.default_rng(3).normal(size=n)
    res = {}
    # single-GPU reference (every rank computes it: simple and symmetric)
    s1 = Solver.from_config(cfg, **opts)
    dev = lambda s, v: torch.tensor(v[s.local_ids], dtype=torch.float32, device="cuda")
    y1 = s1.to_global(s1.matvec(dev(s1, x), "kprime").cpu().numpy())
    yd1 = s1.to_global(s1.matvec(dev(s1, x), "double").cpu().numpy())
    r1 = s1.solve()
    b1 = s1.bibee("cfa")
    phi1 = s1.reaction_potential(r1["sigma"])
    for mode in (0, 1, 2):  # 2: input_mode 1 with every triangle on rank 0 (the others pass none)
        if mode == 0:
            c = cfg
        elif mode == 1:
            c = part_of(cfg, rank, world)
        else:
            c = cfg if rank == 0 else dict(cfg, vertices=np.zeros((0, 3)), triangles=np.zeros((0, 3), np.int32))
        s = Solver.distributed(c, input_mode=min(mode, 1), **opts)
        y = gather(s, s.matvec(dev(s, x), "kprime"))
        yd = gather(s, s.matvec(dev(s, x), "double"))  # dipole sources: the halo carries normals
        yh = s.matvec_host(x[s.local_ids].astype(np.float32), "kprime")
        r = s.solve()
        b = s.bibee("cfa")
        sig = gather(s, r["sigma"])
        phi = s.reaction_potential(torch.tensor(sig[s.local_ids], dtype=torch.float32, device="cuda"))
        res[f"mode{mode}"] = dict(n_local=s.n, matvec_rel=rel(y, y1), double_rel=rel(yd, yd1),
                                  host_rel=rel(yh, y[s.local_ids]),
                                  solve=(r["dG"], r1["dG"], r["iterations"], r1["iterations"]),
                                  bibee=(b["dG"], b1["dG"]), phi_rel=rel(phi, phi1),
                                  slots=s.tree_info()["expansion_slots"], n_cells=s.tree_info()["n_cells"])
        s.close()
    # options that need the full mesh (input_mode 0): curvature self-term, analytic near field
    for kw in (dict(self_term=1), dict(near_mode=1, leaf_points=64), dict(quad_points=3)):
        o = dict(opts, **kw)
        sr = Solver.from_config(cfg, **o)
        yr = sr.to_global(sr.matvec(dev(sr, x), "A").cpu().numpy())
        s = Solver.distributed(cfg, **o)
        y = gather(s, s.matvec(dev(s, x), "A"))
        # the matvec, and the charge-FMM (BIBEE energy: E_n / psi of every quadrature variant)
        res["_".join(kw)] = max(rel(y, yr), abs(s.bibee("cfa")["dG"] / sr.bibee("cfa")["dG"] - 1))
        s.close()
        sr.close()
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        print("MGPU", json.dumps(dict(world=world, ranks=allr)), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
