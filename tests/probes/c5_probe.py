"""Developer probe (not a test): at C5 (102,152,000 panels, leaf_points 128) and each expansion
order P given, time the A = I - f K' matvec (CUDA events, 10 steps) and check K' on a seeded
sample of rows against the FP64 oracle for a random x, the per-molecule E_n field (the physical
GMRES right-hand side, tiled over the 1000 copies) and x = 1.

  python tests/probes/c5_probe.py 12 13 14      (PROBE_ROWS = sampled rows, default 1024)
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


def main():
    orders = [int(a) for a in sys.argv[1:]] or [12]
    nrows = int(os.environ.get("PROBE_ROWS", "1024"))
    base = configs.lysozyme(113)
    cfg = configs.array((10, 10, 10), base=base)
    n = len(cfg["triangles"])
    pb = bem.Problem(base)
    xs = {"rand": np.random.default_rng(23).normal(size=n), "En": np.tile(pb.E, n // pb.pan.n),
          "one": np.ones(n)}
    rows = np.sort(np.random.default_rng(24).choice(n, nrows, replace=False))
    t0 = time.time()
    pan = bem.Panels(cfg["vertices"], cfg["triangles"])
    refs = {k: bem.apply_kprime(pan, x, rows=rows) for k, x in xs.items()}
    print(f"# oracle rows {time.time() - t0:.1f} s", file=sys.stderr, flush=True)
    for P in orders:
        s = Solver.from_config(cfg, terms=P, leaf_points=128)
        out = dict(P=P, levels=s.tree_info()["levels"])
        for k, x in xs.items():
            xd = torch.tensor(s.to_local(x), dtype=torch.float32, device="cuda")
            y = s.to_global(s.matvec(xd, "kprime").cpu().numpy().astype(np.float64))
            e = y[rows] - refs[k]
            out[k] = dict(rel_l2=float(np.linalg.norm(e) / np.linalg.norm(refs[k])),
                          max_rel=float(np.abs(e).max() / np.abs(refs[k]).max()))
        x = torch.tensor(s.to_local(xs["rand"]), dtype=torch.float32, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            s.matvec(x, "A", out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ph = []
        e0.record()
        for _ in range(10):
            s.matvec(x, "A", out=y)
            ph.append(s.timing())
        e1.record()
        torch.cuda.synchronize()
        out["ms"] = e0.elapsed_time(e1) / 10
        out["phases"] = {k: float(np.mean([p[k] for p in ph])) for k in ("upward", "m2l", "p2p", "l2p")}
        out["m2l_pairs"] = int(ph[-1]["m2l_pairs"])
        print(json.dumps(out), flush=True)
        s.close()


if __name__ == "__main__":
    main()
