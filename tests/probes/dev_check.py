"""Developer check: print parity numbers of the CUDA path vs the oracle (not a test)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from paper_1007_4591_b200 import Solver
from oracle import bem
from synth import configs

def run(s, x, op):
    y = s.matvec(torch.tensor(s.to_local(x), dtype=torch.float32, device="cuda"), op)
    torch.cuda.synchronize()
    return s.to_global(y.cpu().numpy().astype(np.float64))

for name, cfg in [("born8", configs.born(8)), ("kirk24", configs.kirkwood(24)), ("lyso20", configs.lysozyme(nu=20, n_atoms=200))]:
    P = bem.Problem(cfg)
    x = np.random.default_rng(1).normal(size=P.pan.n)
    ref = bem.apply_kprime(P.pan, x)
    for kw in (dict(direct=1), dict(terms=4, leaf_points=16), dict(terms=8, leaf_points=16), dict(terms=12, leaf_points=16)):
        try:
            s = Solver.from_config(cfg, **kw)
            y = run(s, x, "kprime")
            print(name, kw, s.tree_info()["levels"], "K' err", bem.rel_l2(y, ref), flush=True)
        except Exception as e:
            print(name, kw, "FAILED", e, flush=True)
    s = Solver.from_config(cfg, terms=12, leaf_points=16)
    En, psi = s.charge_fields()
    print(" En err", bem.rel_l2(s.to_global(En.cpu().numpy()), P.E))
    r = s.solve(); ref_s = P.solve("gmres")
    print(" solve", r["dG"], ref_s["dG"], r["iterations"], ref_s["iterations"])
    print(" cfa", s.bibee("cfa")["dG"], P.bibee("cfa")["dG"])
