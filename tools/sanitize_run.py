"""Developer check (not a test): every ABI entry point on small C1 / C2-like inputs, for running
under compute-sanitizer (memcheck): all operators, solve, BIBEE, fields, reaction potential,
host-buffer matvec, quadrature / near-field / self-term options, direct mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1007_4591_b200 import Solver
from synth import configs

for cfg, kw in ((configs.born(8), dict(terms=13, leaf_points=16)),
                (configs.kirkwood(16), dict(terms=13, leaf_points=32)),
                (configs.kirkwood(16), dict(terms=12, leaf_points=32, quad_points=3)),
                (configs.lysozyme(nu=16, n_atoms=60), dict(terms=10, leaf_points=64, near_mode=1)),
                (configs.lysozyme(nu=16, n_atoms=60), dict(terms=13, leaf_points=16, self_term=1)),
                (configs.born(8), dict(direct=1))):
    s = Solver.from_config(cfg, **kw)
    x = torch.tensor(np.random.default_rng(0).normal(size=s.n), dtype=torch.float32, device="cuda")
    for op in ("kprime", "single", "A") + (() if kw.get("near_mode") else ("double",)):
        s.matvec(x, op)
    s.matvec_host(x.cpu().numpy(), "A")
    s.charge_fields()
    r = s.solve()
    s.bibee("cfa")
    s.reset_fields()
    s.bibee("lb")
    s.reaction_potential(r["sigma"])
    torch.cuda.synchronize()
    print("ok", kw, r["dG"], flush=True)
    s.close()
