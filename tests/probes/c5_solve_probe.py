"""Developer probe (not a test): the full BEM solve at C5 (102,152,000 panels, P = 13, leaf 128)
checked by the oracle itself -- the residual ||f E - (I - f K') sigma|| / ||f E|| of the GPU
solution on a seeded sample of rows, with the oracle's K' rows over ALL sources and the oracle's
E_n (an O(N^2) oracle solve at this size is out of reach)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from oracle import bem
from paper_1007_4591_b200 import Solver
from synth import configs


def main():
    nrows = int(os.environ.get("PROBE_ROWS", "2048"))
    cfg = configs.array((10, 10, 10), base=configs.lysozyme(113))
    n = len(cfg["triangles"])
    s = Solver.from_config(cfg, terms=13, leaf_points=128, charge_terms=12)
    r = s.solve()
    sig = s.to_global(r["sigma"].cpu().numpy().astype(np.float64))
    rows = np.sort(np.random.default_rng(41).choice(n, nrows, replace=False))
    t0 = time.time()
    pan = bem.Panels(cfg["vertices"], cfg["triangles"])
    f = 2.0 * (cfg["eps_out"] - cfg["eps_in"]) / (cfg["eps_in"] + cfg["eps_out"])
    kp = bem.apply_kprime(pan, sig, rows=rows)
    E = bem.normal_field(pan, cfg["charge_xyz"], cfg["charge_q"], cfg["eps_in"], rows=rows)
    b = f * E
    res = b - (sig[rows] - f * kp)
    out = {"rows": int(nrows), "iterations": int(r["iterations"]), "gpu_rel_residual": float(r["rel_residual"]),
           "oracle_rel_residual_rows": float(np.linalg.norm(res) / np.linalg.norm(b)),
           "dG_internal": r["dG"], "oracle_s": time.time() - t0}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
