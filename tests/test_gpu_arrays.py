"""Energy parity at array scale (SURVEY 8(d) "energy parity at array scale uses
a 3 x 3 x 3 array"), through the C ABI at the bench launch configuration (P = 13, leaf 128):

* 2 x 2 x 2 array of a coarser synthetic lysozyme (57,600 panels, 8 molecules that see each other):
  full GMRES Delta G and BIBEE-CFA against the oracle's GMRES / BIBEE, <= 1e-3 (north star);
* 3 x 3 x 3 array of C3 (2,758,104 panels, 54,000 charges): BIBEE-CFA against the exact oracle
  energy (E_n of every panel from every charge, then 1/2 q^T C sigma_hat), and the GMRES solution
  checked with the oracle itself -- its residual ||f E - (I - f K') sigma|| on 1,024 seeded rows
  (the oracle's K' rows over all sources) and its energy 1/2 q^T C sigma by the oracle's plain C
  (O8) -- since an O(N^2) oracle GMRES at 2.76 M panels is out of reach of a test.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import bem  # noqa: E402
from synth import configs  # noqa: E402

pytestmark = pytest.mark.gpu
BENCH = dict(terms=13, leaf_points=128)


def solver(cfg, **kw):
    from paper_1007_4591_b200 import Solver
    return Solver.from_config(cfg, **kw)


def test_small_array_gmres_and_bibee_energies():
    cfg = configs.array((2, 2, 2), base=configs.lysozyme(30, 400))
    P = bem.Problem(cfg)
    s = solver(cfg, **BENCH)
    r = s.solve()
    ref = P.solve("gmres")
    assert r["converged"] and abs(r["dG"] / ref["dG"] - 1) < 1e-3, (r["dG"], ref["dG"])
    e, e_ref = s.bibee("cfa")["dG"], P.bibee("cfa")["dG"]
    assert abs(e / e_ref - 1) < 1e-3, (e, e_ref)


def test_c5_small_bibee_exact_and_gmres_checked_by_oracle():
    cfg = configs.array((3, 3, 3), base=configs.lysozyme(113))
    n = len(cfg["triangles"])
    P = bem.Problem(cfg)
    s = solver(cfg, **BENCH)
    # BIBEE-CFA: exact oracle (all panels x all charges, twice)
    e_ref = P.bibee("cfa")["dG"]
    e = s.bibee("cfa")["dG"]
    assert abs(e / e_ref - 1) < 1e-3, (e, e_ref)
    # full solve on the GPU, then the oracle's own residual and energy of that solution
    r = s.solve()
    assert r["converged"]
    sig = s.to_global(r["sigma"].cpu().numpy().astype(np.float64))
    rows = np.sort(np.random.default_rng(41).choice(n, 1024, replace=False))
    kp = bem.apply_kprime(P.pan, sig, rows=rows)
    b = P.f * P.E[rows]
    res = b - (sig[rows] - P.f * kp)
    assert np.linalg.norm(res) / np.linalg.norm(b) < 2e-4  # FMM truncation (<= 1e-4 of K') + GMRES 1e-6
    e_sig = P.energy_of(sig)[0]
    assert abs(r["dG"] / e_sig - 1) < 1e-3, (r["dG"], e_sig)
