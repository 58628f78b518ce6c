"""Developer probe (not a test): K' FMM error vs the FP64 oracle for SMOOTH / physical inputs
(E_n, sigma, x = 1, low-order Y_lm, random) over the expansion order P and the leaf size, on
C2 (Kirkwood, 32,768 panels) and C3 (synthetic lysozyme, 102,152 panels).

Prints one JSON line per (config, P, leaf, x): rel L2 and max|err| / max|ref|.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

from oracle import bem
from paper_1007_4591_b200 import Solver
from synth import configs


def run(s, x, op="kprime"):
    y = s.matvec(torch.tensor(s.to_local(x), dtype=torch.float32, device="cuda"), op)
    torch.cuda.synchronize()
    return s.to_global(y.cpu().numpy().astype(np.float64))


def inputs(P, cfg):
    c = P.pan.centroid
    d = c - c.mean(0)
    r = np.linalg.norm(d, axis=1)
    u = d / r[:, None]
    xs = {"En": P.E.copy(), "one": np.ones(P.pan.n), "y20": 1.5 * u[:, 2] ** 2 - 0.5, "y21": u[:, 0] * u[:, 2],
          "y33": u[:, 0] * (u[:, 0] ** 2 - 3 * u[:, 1] ** 2), "rand": np.random.default_rng(2).normal(size=P.pan.n)}
    t0 = time.time()
    xs["sigma"] = P.solve("gmres")["sigma"]
    print(f"# oracle solve {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
    return xs


def main():
    which = sys.argv[1:] or ["c2", "c3"]
    terms = [int(t) for t in os.environ.get("PROBE_TERMS", "10,12,13,14").split(",")]
    leaves = [int(t) for t in os.environ.get("PROBE_LEAVES", "64,128").split(",")]
    for name in which:
        cfg = configs.kirkwood(64) if name == "c2" else configs.lysozyme(113)
        P = bem.Problem(cfg)
        xs = inputs(P, cfg)
        refs = {k: bem.apply_kprime(P.pan, v) for k, v in xs.items()}
        for p in terms:
            for lf in leaves:
                s = Solver.from_config(cfg, terms=p, leaf_points=lf)
                lv = s.tree_info()["levels"]
                for k, x in xs.items():
                    y = run(s, x)
                    ref = refs[k]
                    e = y - ref
                    print(json.dumps(dict(cfg=name, P=p, leaf=lf, levels=lv, x=k,
                                          rel_l2=float(np.linalg.norm(e) / np.linalg.norm(ref)),
                                          max_rel=float(np.abs(e).max() / np.abs(ref).max()))), flush=True)
                s.close()


if __name__ == "__main__":
    main()
