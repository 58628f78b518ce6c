"""Run a few FMM matvecs on one config for profiling (ncu / launch lists); not a benchmark."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1007_4591_b200 import Solver
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--terms", type=int, default=13)
ap.add_argument("--leaf-points", type=int, default=128)
ap.add_argument("--op", default="A")
a = ap.parse_args()
cfg, name = bench.workload(a.config)
s = Solver.from_config(cfg, terms=a.terms, leaf_points=a.leaf_points)
x = torch.tensor(np.random.default_rng(7).normal(size=s.n), dtype=torch.float32, device="cuda")
for _ in range(a.reps):
    y = s.matvec(x, a.op)
torch.cuda.synchronize()
print(name, s.tree_info(), s.timing())
