"""Parity at the BASELINE.json configurations (full sizes, the bench launch configuration P = 13,
leaf_points = 128), through the C ABI, against the FP64 oracle.

Where the O(N^2) oracle is too slow for every output (C4, C5) it is evaluated on a seeded
sample of rows (each row is the exact oracle sum over ALL sources).

K' bounds: relative L2 <= 1e-4 (north star) and, per element,
max_i |y_i - y_ref_i| <= 1e-3 max_i |y_ref_i| -- for random x and for the smooth / physical inputs
GMRES applies (E_n, sigma, x = 1, low-order Y_lm).  Measured on a B200 at P = 12 the C3 random-x
error is 1.4e-4 (smooth inputs <= 1.4e-5), at P = 13 7.0e-5: the bench order is 13.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import bem, closed_forms as cf  # noqa: E402
from synth import configs  # noqa: E402

pytestmark = pytest.mark.gpu
BENCH = dict(terms=13, leaf_points=128)


def solver(cfg, **kw):
    from paper_1007_4591_b200 import Solver
    return Solver.from_config(cfg, **kw)


def matvec_global(s, x, op):
    y = s.matvec(torch.tensor(s.to_local(x), dtype=torch.float32, device="cuda"), op)
    torch.cuda.synchronize()
    return s.to_global(y.cpu().numpy().astype(np.float64))


def kprime_errors(y, ref):
    e = y - ref
    return float(np.linalg.norm(e) / np.linalg.norm(ref)), float(np.abs(e).max() / np.abs(ref).max())


def input_vectors(P):
    """Random x and the smooth / physical inputs of a K' matvec inside GMRES (rhs E_n, the solution
    sigma, a constant, low-order spherical harmonics of the direction from the centre)."""
    d = P.pan.centroid - P.pan.centroid.mean(0)
    u = d / np.linalg.norm(d, axis=1)[:, None]
    return {"rand": np.random.default_rng(31).normal(size=P.pan.n), "En": P.E.copy(), "one": np.ones(P.pan.n),
            "y20": 1.5 * u[:, 2] ** 2 - 0.5, "y21": u[:, 0] * u[:, 2],
            "y33": u[:, 0] * (u[:, 0] ** 2 - 3 * u[:, 1] ** 2), "sigma": P.solve("gmres")["sigma"]}


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_kprime_smooth_and_physical_inputs(name):
    """the 1e-4 K' bound at the bench configuration for the vectors GMRES
    actually applies, not only for white noise; plus a per-element bound."""
    cfg = configs.kirkwood(64) if name == "c2" else configs.lysozyme(113)
    P = bem.Problem(cfg)
    s = solver(cfg, **BENCH)
    errs = {}
    for k, x in input_vectors(P).items():
        errs[k] = kprime_errors(matvec_global(s, x, "kprime"), bem.apply_kprime(P.pan, x))
    assert all(l2 < 1e-4 and mx < 1e-3 for l2, mx in errs.values()), errs


def test_c1_born_fmm_and_direct():
    cfg = configs.born(8)
    for kw in (dict(direct=1), BENCH):
        r = solver(cfg, **kw).solve()
        assert abs(r["dG"] / -0.00982207 - 1) < 1e-5, (kw, r["dG"])


def test_c2_kirkwood_full():
    cfg = configs.kirkwood(64)  # 32,768 panels
    P = bem.Problem(cfg)
    s = solver(cfg, **BENCH)
    x = np.random.default_rng(21).normal(size=P.pan.n)
    assert bem.rel_l2(matvec_global(s, x, "kprime"), bem.apply_kprime(P.pan, x)) < 1e-4
    r = s.solve()
    ref = P.solve("gmres")
    assert abs(r["dG"] / ref["dG"] - 1) < 1e-3
    series = cf.sphere_series(cfg["charge_xyz"], cfg["charge_q"], 1.0, 4.0, 80.0)
    assert abs(r["dG"] / series - 1) < 0.01  # BASELINE: within 1 % of the analytic sphere value
    cfa_series = cf.sphere_series(cfg["charge_xyz"], cfg["charge_q"], 1.0, 4.0, 80.0, lam=-0.5)
    assert abs(s.bibee("cfa")["dG"] / cfa_series - 1) < 0.01


def test_c3_lysozyme_full():
    cfg = configs.lysozyme(113)  # 102,152 panels, 2,000 atoms
    P = bem.Problem(cfg)
    s = solver(cfg, **BENCH)
    x = np.random.default_rng(22).normal(size=P.pan.n)
    assert bem.rel_l2(matvec_global(s, x, "A"), bem.apply_A(P.pan, x, P.f)) < 1e-5
    assert bem.rel_l2(matvec_global(s, x, "kprime"), bem.apply_kprime(P.pan, x)) < 1e-4
    En, psi = s.charge_fields()
    assert bem.rel_l2(s.to_global(En.cpu().numpy().astype(np.float64)), P.E) < 1e-4
    e, e_ref = s.bibee("cfa")["dG"], P.bibee("cfa")["dG"]
    assert abs(e / e_ref - 1) < 1e-3
    r = s.solve()
    ref = P.solve("gmres")
    assert r["converged"] and abs(r["dG"] / ref["dG"] - 1) < 1e-3, (r["dG"], ref["dG"])


def test_c4_binding_bibee_full_and_bem_scaled():
    b = configs.binding()
    dg = {}
    for k in ("complex", "protein", "ligand"):
        s = solver(b[k], **BENCH)
        dg[k] = (s.bibee("cfa")["dG"], bem.Problem(b[k]).bibee("cfa")["dG"])
    gpu = bem.binding_energy(*(dg[k][0] for k in ("complex", "protein", "ligand")))
    ref = bem.binding_energy(*(dg[k][1] for k in ("complex", "protein", "ligand")))
    for k in dg:
        assert abs(dg[k][0] / dg[k][1] - 1) < 1e-3
    scale = max(abs(dg["protein"][1]), abs(dg["ligand"][1]))
    assert abs(gpu - ref) < 1e-3 * scale
    # full BEM binding on a reduced-resolution copy of the recipe (oracle GMRES affordable)
    b = configs.binding(nu_protein=40, nu_ligand=16)
    g, o = {}, {}
    for k in ("complex", "protein", "ligand"):
        g[k] = solver(b[k], **BENCH).solve()["dG"]
        o[k] = bem.Problem(b[k]).solve("gmres")["dG"]
    gd = bem.binding_energy(g["complex"], g["protein"], g["ligand"])
    od = bem.binding_energy(o["complex"], o["protein"], o["ligand"])
    assert abs(gd - od) < 1e-3 * max(abs(o["protein"]), abs(o["ligand"]))


def test_c5_array_sampled_rows():
    """C5 (102,152,000 panels) at the bench launch configuration: K' on 1,024 seeded rows (each the
    full FP64 sum over all sources) for random x, the per-molecule E_n field tiled over the copies
    (the physical GMRES right-hand side) and x = 1; rel L2 and per-element bounds."""
    base = configs.lysozyme(113)
    cfg = configs.array((10, 10, 10), base=base)  # 102,152,000 panels
    s = solver(cfg, **BENCH)
    n = len(cfg["triangles"])
    pb = bem.Problem(base)
    xs = {"rand": np.random.default_rng(23).normal(size=n), "En": np.tile(pb.E, n // pb.pan.n), "one": np.ones(n)}
    rows = np.sort(np.random.default_rng(24).choice(n, 1024, replace=False))
    pan = bem.Panels(cfg["vertices"], cfg["triangles"])
    errs = {}
    for k, x in xs.items():
        y = matvec_global(s, x, "kprime")
        errs[k] = kprime_errors(y[rows], bem.apply_kprime(pan, x, rows=rows))
        if k == "rand":  # every output finite, deterministic repeat
            assert np.isfinite(y).all()
            assert np.array_equal(y, matvec_global(s, x, "kprime"))
    assert all(l2 < 1e-4 and mx < 1e-3 for l2, mx in errs.values()), errs


def test_charge_terms_fields_energy_and_matvec_unchanged():
    """options.charge_terms (the charge-FMM order, the bench uses 12 under K' order 13): on C3 the
    fields E_n / psi stay within 1e-4 of the oracle at 12 (measured 3.3e-5 / 1.8e-6) and the BIBEE
    energy within 1e-3 at 10 and 12 (measured 2e-6 / 7e-7); the K' matvec does not depend on it."""
    cfg = configs.lysozyme(113)
    P = bem.Problem(cfg)
    psi_ref = bem.charge_potential(P.pan, cfg["charge_xyz"], cfg["charge_q"])
    e_ref = P.bibee("cfa")["dG"]
    x = np.random.default_rng(5).normal(size=P.pan.n)
    y13 = matvec_global(solver(cfg, **BENCH), x, "kprime")
    for ct in (12, 10):
        s = solver(cfg, charge_terms=ct, **BENCH)
        assert np.array_equal(matvec_global(s, x, "kprime"), y13)
        En, psi = s.charge_fields()
        En = s.to_global(En.cpu().numpy().astype(np.float64))
        psi = s.to_global(psi.cpu().numpy().astype(np.float64))
        if ct == 12:
            assert bem.rel_l2(En, P.E) < 1e-4 and bem.rel_l2(psi, psi_ref) < 1e-4
        assert abs(s.bibee("cfa")["dG"] / e_ref - 1) < 1e-3
