"""Developer probe (not a test): accuracy and time of the charge-FMM (E_n, psi, BIBEE energy) at
each charge_terms order, K' / matvec order fixed at the bench's P = 13, leaf 128.
C3 (102,152 panels): full E_n / psi against the oracle's direct sums and the BIBEE-CFA energy against
the oracle's; C5 (1.02e8 panels): 1,024 seeded rows of E_n / psi against the oracle and the uncached
BIBEE device time (10 calls)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from oracle import bem
from paper_1007_4591_b200 import Solver
from synth import configs

ORDERS = [int(v) for v in (sys.argv[1].split(",") if len(sys.argv) > 1 else "13,12,10,8".split(","))]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def fields(s):
    s.reset_fields()
    En, psi = s.charge_fields()
    return (s.to_global(En.cpu().numpy().astype(np.float64)), s.to_global(psi.cpu().numpy().astype(np.float64)))


c3 = configs.lysozyme(113)
P3 = bem.Problem(c3)
psi3 = bem.charge_potential(P3.pan, c3["charge_xyz"], c3["charge_q"])
e3 = P3.bibee("cfa")["dG"]
for Pc in ORDERS:
    s = Solver.from_config(c3, terms=13, leaf_points=128, charge_terms=Pc)
    En, psi = fields(s)
    d = s.bibee("cfa")["dG"]
    print(json.dumps({"config": "C3", "charge_terms": Pc, "rel_l2_En": rel(En, P3.E), "rel_l2_psi": rel(psi, psi3),
                      "max_rel_En": float(np.abs(En - P3.E).max() / np.abs(P3.E).max()),
                      "bibee_rel": abs(d / e3 - 1)}), flush=True)
    s.close()

c5 = configs.array((10, 10, 10), base=configs.lysozyme(113))
n = len(c5["triangles"])
rows = np.sort(np.random.default_rng(11).choice(n, 1024, replace=False))
ref = None
for Pc in ORDERS:
    s = Solver.from_config(c5, terms=13, leaf_points=128, charge_terms=Pc)
    if ref is None:
        pan5 = bem.Panels(c5["vertices"], c5["triangles"])
        ref = (bem.normal_field(pan5, c5["charge_xyz"], c5["charge_q"], 4.0, rows=rows),
               bem.charge_potential(pan5, c5["charge_xyz"], c5["charge_q"], rows=rows))
    En, psi = fields(s)
    s.bibee("cfa")
    t = []
    for _ in range(10):
        s.reset_fields()
        e = s.bibee("cfa")
        t.append(s.timing())
    print(json.dumps({"config": "C5", "charge_terms": Pc, "rel_l2_En_rows": rel(En[rows], ref[0]),
                      "rel_l2_psi_rows": rel(psi[rows], ref[1]), "dG": e["dG"],
                      "bibee_ms": float(np.mean([x["bibee"] for x in t])),
                      "m2l_ms": float(np.mean([x["m2l"] for x in t])),
                      "upward_ms": float(np.mean([x["upward"] for x in t])),
                      "l2p_ms": float(np.mean([x["l2p"] for x in t]))}), flush=True)
    s.close()
