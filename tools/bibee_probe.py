"""Developer probe (not a test): the uncached BIBEE energy at C5 (charge-FMM + reduction), device time
and phases over 10 calls, with the exact charge-source P2P interaction count."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1007_4591_b200 import Solver
from synth import configs

cfg = configs.array((10, 10, 10), base=configs.lysozyme(113))
s = Solver.from_config(cfg, terms=13, leaf_points=128)
s.bibee("cfa")
ph = []
for _ in range(10):
    s.reset_fields()
    e = s.bibee("cfa")
    ph.append(s.timing())
out = {k: float(np.mean([p[k] for p in ph])) for k in ("bibee", "upward", "m2l", "p2p", "l2p", "total")}
out["p2p_interactions"] = int(ph[-1]["p2p_interactions"])
out["dG"] = e["dG"]
out["chunk_chg"] = os.environ.get("FMMBEM_P2P_CHUNK_CHG", "64")
print(json.dumps(out), flush=True)
