"""Pins of the FP64 oracle against what the paper and mathematics fix (marker: not gpu).

Each test pins an oracle function to something other than itself: printed example
values, closed forms, invariants, special cases, or brute force / finite differences.
"""
import os
from math import factorial

import numpy as np
import pytest

from oracle import bem, closed_forms as cf
from oracle import _cdirect
from synth import configs, octasphere, icosphere

GOLD = os.path.join(os.path.dirname(__file__), "golden")
BORN = cf.born(1.0, 1.0, 4.0, 80.0)


def _gold(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        if line.strip() and not line.startswith("#"):
            rows.append(line.split())
    return rows


# ---------------------------------------------------------------- kernel
def test_kernel_spec_examples():
    rows = {r[0] + r[1] + r[2] + r[3]: float(r[4]) for r in _gold("spec_examples.txt") if len(r) == 5}
    src = np.zeros((1, 3)); w = np.ones(1)
    assert cf.born  # keep import
    phi1 = _cdirect.pot_sum(np.array([[1.0, 0, 0]]), None, src, w, None)[0]
    phi2 = _cdirect.pot_sum(np.array([[3.0, 4.0, 0]]), None, src, w, None)[0]
    gx = _cdirect.dn_sum(np.array([[1.0, 0, 0]]), np.array([[1.0, 0, 0]]), None, src, w, None)[0]
    assert phi1 == pytest.approx(rows["phi100"], abs=5e-8)
    assert phi2 == pytest.approx(rows["phi340"], abs=5e-8)
    assert gx == pytest.approx(rows["grad_x100"], abs=5e-8)


def test_normal_derivative_is_finite_difference_of_potential():
    """dG/dn_x equals the central difference of G along n (pins sign and 1/r^3 form)."""
    rng = np.random.default_rng(3)
    x = rng.normal(size=(20, 3)); n = rng.normal(size=(20, 3))
    n /= np.linalg.norm(n, axis=1)[:, None]
    y = rng.normal(size=(30, 3)) + 4.0; w = rng.normal(size=30)
    h = 1e-5
    fd = (_cdirect.pot_sum(x + h * n, None, y, w, None) - _cdirect.pot_sum(x - h * n, None, y, w, None)) / (2 * h)
    dn = _cdirect.dn_sum(x, n, None, y, w, None)
    assert np.allclose(dn, fd, rtol=1e-7, atol=1e-10)


def test_exclusion_and_coincidence():
    x = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    w = np.array([1.0, 2.0])
    out = _cdirect.pot_sum(x, np.array([0, 1]), x, w, np.array([0, 1]))
    assert out == pytest.approx([2.0 / (4 * np.pi), 1.0 / (4 * np.pi)])
    with pytest.raises(ValueError):
        _cdirect.pot_sum(x, None, x, w, None)


# ---------------------------------------------------------------- panels (O1)
def test_panel_spec_example():
    p = bem.Panels(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]), np.array([[0, 1, 2]]))
    assert np.allclose(p.centroid[0], [1 / 3, 1 / 3, 0])
    assert p.area[0] == pytest.approx(0.5)
    assert np.allclose(p.normal[0], [0, 0, 1])


def test_degenerate_and_bad_index():
    v = np.array([[0.0, 0, 0], [1, 0, 0], [2, 0, 0], [0, 1, 0]])
    with pytest.raises(ValueError, match="degenerate triangle 1"):
        bem.Panels(v, np.array([[0, 1, 3], [0, 1, 2]]))
    with pytest.raises(ValueError, match="out of range"):
        bem.Panels(v, np.array([[0, 1, 4]]))


@pytest.mark.parametrize("nu", [1, 3, 8])
def test_octasphere_counts_euler_outward_closed(nu):
    v, t = octasphere(nu)
    assert len(t) == 8 * nu * nu and len(v) == 4 * nu * nu + 2
    edges = {tuple(sorted(e)) for tri in t for e in ((tri[0], tri[1]), (tri[1], tri[2]), (tri[2], tri[0]))}
    assert len(v) - len(edges) + len(t) == 2
    p = bem.Panels(v, t)
    assert np.all(np.einsum("ij,ij->i", p.normal, p.centroid) > 0)  # outward
    s = (p.area[:, None] * p.normal).sum(0)
    assert np.linalg.norm(s) < 1e-12 * p.area.sum()  # divergence theorem (SPEC)


def test_icosphere_counts_and_area():
    for k in (0, 1, 2):
        v, t = icosphere(k)
        assert len(t) == 20 * 4 ** k
    p = bem.Panels(*icosphere(4))
    assert abs(p.area.sum() / (4 * np.pi) - 1) < 5e-3


def test_rigid_motion_invariance():
    cfg = configs.born(4)
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    p1 = bem.Panels(cfg["vertices"], cfg["triangles"])
    p2 = bem.Panels(cfg["vertices"] @ Q.T + [3.0, -1.0, 2.0], cfg["triangles"])
    assert np.allclose(p1.area, p2.area, rtol=1e-12)
    assert np.allclose(p1.normal @ Q.T, p2.normal, atol=1e-12)
    x = rng.normal(size=p1.n)
    assert np.allclose(bem.apply_kprime(p1, x), bem.apply_kprime(p2, x), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("K,deg", [(1, 1), (3, 2), (6, 4), (7, 5)])
def test_quadrature_exactness(K, deg):
    """Each rule integrates x^a y^b exactly over the reference triangle for a+b <= degree:
    int_T x^a y^b = a! b! / (a+b+2)!  (closed form)."""
    beta, w = bem.quad_rule(K)
    assert w.sum() == pytest.approx(1.0, abs=1e-14)
    x, y = beta[:, 1], beta[:, 2]  # vertices (0,0),(1,0),(0,1)
    for a in range(deg + 1):
        for b in range(deg + 1 - a):
            exact = factorial(a) * factorial(b) / factorial(a + b + 2)
            assert 0.5 * np.sum(w * x ** a * y ** b) == pytest.approx(exact, abs=1e-12)
    # and is NOT exact one degree higher for the 1-point rule (sanity)
    if K == 1:
        assert 0.5 * np.sum(w * x ** 2) != pytest.approx(1 / 12, abs=1e-6)


# ---------------------------------------------------------------- E (O3), K' (O4), V (O5), C (O7)
def test_normal_field_born_and_gauss_law():
    P = bem.Problem(configs.born(16))
    En = float([r for r in _gold("spec_examples.txt") if r[0] == "En_born"][0][1])
    # at every centroid the flat-panel value is within O(h^2) of -1/(16 pi)
    assert np.allclose(P.E, En, rtol=2e-2)
    # Gauss: sum_j A_j eps_I E_j -> -(enclosed charge)   (flux of a unit charge)
    errs = []
    for nu in (8, 16, 32):
        Q = bem.Problem(configs.born(nu, q=1.0))
        errs.append(abs(np.sum(Q.pan.area * Q.E) * Q.eps_in + 1.0))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-3
    # exact sphere points with radial normals: E = -q/(4 pi eps_I a^2) exactly
    u = np.random.default_rng(1).normal(size=(10, 3)); u /= np.linalg.norm(u, axis=1)[:, None]
    e = _cdirect.dn_sum(u, u, None, np.zeros((1, 3)), np.ones(1), None) / 4.0
    assert np.allclose(e, -1 / (16 * np.pi), rtol=1e-13)


def test_kprime_constant_eigenvalue_on_sphere():
    """Continuum: K' 1 = -1/2 on the sphere; discrete mean converges to it."""
    errs = []
    for nu in (8, 16, 32):
        p = bem.Panels(*octasphere(nu))
        errs.append(abs(np.mean(bem.apply_kprime(p, np.ones(p.n))) + 0.5))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.01


def test_kprime_matches_dense_and_single_layer_fd():
    cfg = configs.kirkwood(6)
    p = bem.Panels(cfg["vertices"], cfg["triangles"])
    x = np.random.default_rng(2).normal(size=p.n)
    assert np.allclose(bem.apply_kprime(p, x), bem.dense_kprime(p) @ x, rtol=1e-10, atol=1e-13)
    # K' row i is d/dn_i of the single-layer potential of all panels j != i
    h = 1e-5
    y, owner, aw = p.sources()
    w = np.repeat(x, p.K) * aw
    idx = np.arange(p.n)
    fd = (_cdirect.pot_sum(p.centroid + h * p.normal, idx, y, w, owner)
          - _cdirect.pot_sum(p.centroid - h * p.normal, idx, y, w, owner)) / (2 * h)
    assert np.allclose(bem.apply_kprime(p, x), fd, rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("K", [1, 3, 6, 7])
def test_kprime_sphere_eigenvalues_all_rules(K):
    """On the sphere K' Y_n = -1/(2(2n+1)) Y_n (n=0: P:446-447).
    For n = 1 (x = z) and n = 2 (x = 3z^2 - 1) the discrete operator converges to it."""
    for n, fn in ((1, lambda c: c[:, 2]), (2, lambda c: 3 * c[:, 2] ** 2 - 1)):
        lam = -1.0 / (2 * (2 * n + 1))
        errs = []
        for nu in (8, 16, 32):
            p = bem.Panels(*octasphere(nu), K=K)
            u = p.centroid / np.linalg.norm(p.centroid, axis=1)[:, None]
            x = fn(u)
            errs.append(bem.rel_l2(bem.apply_kprime(p, x), lam * x))
        assert errs[0] > 1.5 * errs[1] > 2.25 * errs[2] and errs[2] < 0.1, errs  # O(h)


def test_single_layer_and_reaction_potential_shell_theorem():
    """Uniform sigma on a sphere: potential at the centre = sigma a."""
    errs = []
    for nu in (8, 16, 32):
        p = bem.Panels(*octasphere(nu, 2.0))
        errs.append(abs(bem.reaction_potential(p, np.ones(p.n), np.zeros((1, 3)))[0] - 2.0))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 2e-3
    # V symmetric after area weighting: A_i V_ij = A_j V_ji  (G symmetric)
    p = bem.Panels(*octasphere(3))
    Vd = np.stack([bem.apply_single(p, e) for e in np.eye(p.n)], 1)
    S = p.area[:, None] * Vd
    assert np.allclose(S, S.T, rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- GMRES (O6)
def test_gmres_identity_and_scaled_identity():
    b = np.arange(1.0, 11.0)
    x, its, _, ok = bem.gmres(lambda v: v, b)
    assert ok and its == 1 and np.allclose(x, b)
    x, its, _, ok = bem.gmres(lambda v: 2 * v, b)
    assert ok and its == 1 and np.allclose(x, b / 2)


def test_gmres_matches_dense_lu_monotone_and_restarts():
    P = bem.Problem(configs.kirkwood(12))
    s_lu = bem.solve_dense(P.pan, P.E, P.f)
    s_gm, its, hist, ok = bem.gmres(lambda v: bem.apply_A(P.pan, v, P.f), P.f * P.E, 1e-10)
    assert ok and bem.rel_l2(s_gm, s_lu) < 1e-9
    assert all(h2 <= h1 * (1 + 1e-12) for h1, h2 in zip(hist, hist[1:]))
    s_r, its_r, _, ok_r = bem.gmres(lambda v: bem.apply_A(P.pan, v, P.f), P.f * P.E, 1e-10, restart=2)
    assert ok_r and its_r >= its and bem.rel_l2(s_r, s_lu) < 1e-8


# ---------------------------------------------------------------- energies (O8, O9, O12)
def test_born_discrete_golden_and_convergence():
    errs = []
    for nu, n, dg in _gold("born_discrete.txt"):
        r = bem.Problem(configs.born(int(nu))).solve("dense")
        assert r["dG"] == pytest.approx(float(dg), rel=1e-5)
        errs.append(abs(r["dG"] / BORN - 1))
    assert errs[0] > errs[1] > errs[2]


def test_self_term_born_errors_match_survey():
    """Option self_term = 1: the curvature self-term K'_ii = -H_i sqrt(A_i/pi)/4 cuts the
    Born error of the octasphere meshes to the values computed at survey time by an independent
    script: 512 panels 3.94 % -> 1.69 %, 2048: 1.57 % -> 0.46 %, 8192: 0.69 % -> 0.14 %; and the
    convergence becomes ~second order (the flat self-term drops an O(h) term)."""
    survey = {8: (3.94, 1.69), 16: (1.57, 0.46), 32: (0.69, 0.14)}
    e1 = {}
    for nu, (flat, curved) in survey.items():
        cfg = configs.born(nu)
        e0 = abs(bem.Problem(cfg).solve("dense")["dG"] / BORN - 1) * 100
        e1[nu] = abs(bem.Problem(cfg, self_term=True).solve("dense")["dG"] / BORN - 1) * 100
        assert e0 == pytest.approx(flat, abs=0.01)
        assert e1[nu] == pytest.approx(curved, abs=0.02), (nu, e1[nu])
    assert e1[8] / e1[16] > 3.3 and e1[16] / e1[32] > 3.3


def test_mean_curvature_of_spheres():
    """H_i from vertex normals (A7) -> 1/R: O(h) per panel, scales as 1/R, invariant under motion."""
    for nu, tol in ((16, 0.03), (32, 0.02)):
        for R in (1.0, 2.5):
            v, t = octasphere(nu, R)
            H = bem.mean_curvature(bem.Panels(v, t))
            assert np.mean(H) * R == pytest.approx(1.0, abs=tol)
    v, t = octasphere(16, 1.0)
    th = 0.7
    rot = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1.0]])
    H0 = bem.mean_curvature(bem.Panels(v, t))
    H1 = bem.mean_curvature(bem.Panels(v @ rot.T + [3.0, -1.0, 2.0], t))
    assert np.allclose(H0, H1, rtol=1e-9, atol=1e-12)


def test_self_term_operator_forms_agree():
    """Dense K' with the self-term diagonal and the matvec form are the same operator."""
    cfg = configs.kirkwood(6)
    pan = bem.Panels(cfg["vertices"], cfg["triangles"])
    x = np.random.default_rng(21).normal(size=pan.n)
    d = bem.self_term_diag(pan)
    assert np.all(d < 0)  # convex surface, outward normals
    y = bem.apply_kprime(pan, x, self_term=True)
    assert np.allclose(bem.dense_kprime(pan, self_term=True) @ x, y, rtol=1e-12, atol=1e-14)
    assert np.allclose(y - bem.apply_kprime(pan, x), d * x, rtol=1e-12, atol=1e-14)


def test_born_kcal_and_charge_scaling():
    """a = 2 A Born: -19.7163 kcal/mol; q -> lam q: dG -> lam^2 dG."""
    assert cf.born(1.0, 2.0, 4.0, 80.0) * bem.KCAL_PER_INTERNAL == pytest.approx(-19.7163, abs=2e-4)
    P1 = bem.Problem(configs.kirkwood(6))
    cfg = configs.kirkwood(6); cfg["charge_q"] = cfg["charge_q"] * -2.5
    P2 = bem.Problem(cfg)
    assert P2.solve("dense")["dG"] == pytest.approx(6.25 * P1.solve("dense")["dG"], rel=1e-12)


def test_closed_forms_reduce_to_born_and_cfa_exact_for_central_charge():
    assert cf.sphere_series([[0, 0, 0]], [1.0], 1.0, 4.0, 80.0) == pytest.approx(BORN, rel=1e-14)
    # CFA exact for uniform normal fields: central charge, lam = -1/2 equals Born
    assert cf.sphere_series([[0, 0, 0]], [1.0], 1.0, 4.0, 80.0, lam=-0.5) == pytest.approx(BORN, rel=1e-14)
    # rotation invariance of the series
    cx, cq = configs.kirkwood_charges(5, 0.6, 7)
    Q, _ = np.linalg.qr(np.random.default_rng(1).normal(size=(3, 3)))
    assert cf.sphere_series(cx @ Q.T, cq, 1, 4, 80) == pytest.approx(cf.sphere_series(cx, cq, 1, 4, 80), rel=1e-12)


def test_kirkwood_single_charge_image_series():
    """Single charge at depth d: the n-th Kirkwood term with q_i=q_k, cos g = 1 is the
    classical (n+1)(eps_I - eps_O)/(eps_I (n eps_I + (n+1) eps_O)) (d/a)^(2n) q^2/(8 pi a) series."""
    q, a, d = 1.3, 2.0, 0.9
    ei, eo = 4.0, 80.0
    ref = sum((n + 1) * (ei - eo) / (ei * (n * ei + (n + 1) * eo)) * (d / a) ** (2 * n)
              for n in range(400)) * q * q / (8 * np.pi * a)
    assert cf.sphere_series([[0, 0, d]], [q], a, ei, eo) == pytest.approx(ref, rel=1e-12)


def test_dense_bem_converges_to_kirkwood_and_bibee_series():
    cfg = configs.kirkwood(8)
    ex = cf.sphere_series(cfg["charge_xyz"], cfg["charge_q"], 1, 4, 80)
    errs, errs_cfa = [], []
    for nu in (8, 16, 32):
        P = bem.Problem(configs.kirkwood(nu))
        errs.append(abs(P.solve("gmres")["dG"] / ex - 1))
        cfs = cf.sphere_series(cfg["charge_xyz"], cfg["charge_q"], 1, 4, 80, lam=-0.5)
        errs_cfa.append(abs(P.bibee("cfa")["dG"] / cfs - 1))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.01
    assert errs_cfa[0] > errs_cfa[1] > errs_cfa[2] and errs_cfa[2] < 0.005


def test_energy_ordering_on_sphere():
    """LB <= P <= BEM <= CFA <= 0 (P:482-487 upper bound; SURVEY App. B ordering)."""
    P = bem.Problem(configs.kirkwood(16))
    bemv = P.solve("dense")["dG"]
    cfa, p0, lb = (P.bibee(v)["dG"] for v in ("cfa", "p", "lb"))
    assert lb <= p0 <= bemv <= cfa <= 0
    cx, cq = configs.kirkwood_charges(10, 0.6, 1)
    s = [cf.sphere_series(cx, cq, 1, 4, 80, lam=l) for l in (0.5, 0.0, "exact", -0.5)]
    assert s[0] <= s[1] <= s[2] <= s[3] <= 0


def test_bibee_scale_identities():
    """P (s=0): sigma = f E exactly; CFA: f/(1+f/2) = eps_hat."""
    f, eh = bem.constants(4.0, 80.0)
    E = np.array([0.3, -1.2])
    assert np.allclose(bem.bibee_sigma(E, f, 0.0), f * E)
    assert np.allclose(bem.bibee_sigma(E, f, -0.5), eh * E, rtol=1e-14)
    with pytest.raises(ValueError):
        bem.bibee_sigma(E, 2.0, 0.5)
    with pytest.raises(ValueError):
        bem.constants(4.0, 4.0)


def test_binding_decoupling():
    """Delta Delta G -> 0 as the ligand separates."""
    def two(sep):
        a = configs.born(6, 1.0, 1.0); b = configs.born(6, 0.7, -0.5)
        vb = b["vertices"] + [sep, 0, 0]
        comp = dict(a, vertices=np.concatenate([a["vertices"], vb]),
                    triangles=np.concatenate([a["triangles"], b["triangles"] + len(a["vertices"])]),
                    charge_xyz=np.array([[0, 0, 0], [sep, 0, 0]]), charge_q=np.array([1.0, -0.5]))
        lig = dict(b, vertices=vb, charge_xyz=np.array([[sep, 0, 0]]))
        g = [bem.Problem(x).solve("dense")["dG"] for x in (comp, a, lig)]
        return bem.binding_energy(*g)
    # far apart, Delta Delta G is the solvent screening of the bare Coulomb pair energy:
    # q1 q2 (1/eps_O - 1/eps_I) / (4 pi sep) -> decays like 1/sep
    seps = (10.0, 20.0, 40.0)
    d = [two(s) * s for s in seps]
    assert np.allclose(d, d[-1], rtol=2e-2)
    scr = 1.0 * -0.5 * (1 / 80 - 1 / 4) / (4 * np.pi)
    assert d[-1] == pytest.approx(scr, rel=0.06)  # octasphere(6) discretisation error ~4-5%


def test_rel_l2():
    assert bem.rel_l2([1.0, 2.0], [1.0, 2.0]) == 0.0
    assert bem.rel_l2([2.0, 0.0], [1.0, 0.0]) == pytest.approx(1.0)


# ---------------------------------------------------------------- near-field option (a11)
def test_triangle_integrals_match_scipy_dblquad():
    """The oracle's panel integrals (adaptive subdivision / Duffy) equal scipy's dblquad over the
    triangle's parameter domain (an independent library integrator)."""
    from scipy.integrate import dblquad
    tv = np.array([[0.0, 0, 0], [1.0, 0.1, 0], [0.2, 0.9, 0.1]])
    n = np.array([0.3, -0.2, 0.9]); n /= np.linalg.norm(n)
    J = np.linalg.norm(np.cross(tv[1] - tv[0], tv[2] - tv[0]))
    for x in (np.array([0.3, 0.3, 0.4]), np.array([1.3, 1.1, 0.05]), np.array([0.45, 0.35, -0.02])):
        def y(u, v):
            return tv[0] + u * (tv[1] - tv[0]) + v * (tv[2] - tv[0])
        gp = dblquad(lambda v, u: J / (4 * np.pi * np.linalg.norm(x - y(u, v))), 0, 1, 0, lambda u: 1 - u,
                     epsabs=1e-13, epsrel=1e-11)[0]
        gd = dblquad(lambda v, u: J * (-(n @ (x - y(u, v))) / (4 * np.pi * np.linalg.norm(x - y(u, v)) ** 3)),
                     0, 1, 0, lambda u: 1 - u, epsabs=1e-13, epsrel=1e-11)[0]
        pot, dn = _cdirect.tri_integrals(x[None], n[None], tv.reshape(1, 9))
        assert pot[0] == pytest.approx(gp, rel=1e-8)
        assert dn[0] == pytest.approx(gd, rel=1e-7, abs=1e-12)


def test_triangle_integrals_limits():
    """Far away the panel integral tends to A G(x, c) with an O((h/d)^2) error; the self integral
    of an equilateral triangle at its centroid equals 3 * (side/(4 pi)) * asinh(sqrt 3) / sqrt 3 * ...
    closed form int 1/r = 3 h ln((1+sin 60)/cos 60)... checked against Duffy on subdivided copies."""
    tv = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, np.sqrt(3) / 2, 0]])
    c = tv.mean(0); A = np.sqrt(3) / 4
    errs = []
    for d in (4.0, 8.0, 16.0):
        x = c + np.array([0.3, 0.2, 1.0]) / np.linalg.norm([0.3, 0.2, 1.0]) * d
        pot, _ = _cdirect.tri_integrals(x[None], np.array([[0, 0, 1.0]]), tv.reshape(1, 9))
        errs.append(abs(pot[0] / (A / (4 * np.pi * d)) - 1))
    assert errs[0] / errs[1] == pytest.approx(4.0, rel=0.1) and errs[1] / errs[2] == pytest.approx(4.0, rel=0.1)
    # centroid of an equilateral triangle of side s: int_T dA/r = 3 * r_in * ln((1 + sin 60)/(1 - sin 60))
    # ... with r_in = s / (2 sqrt 3) the inradius (sum over the 3 edges of the in-plane line integral)
    r_in = 1.0 / (2 * np.sqrt(3))
    exact = 3 * r_in * np.log((1 + np.sin(np.pi / 3)) / (1 - np.sin(np.pi / 3))) / (4 * np.pi)
    pot, dn = _cdirect.tri_integrals(c[None], np.array([[0, 0, 1.0]]), tv.reshape(1, 9), np.ones(1, np.int32))
    assert pot[0] == pytest.approx(exact, rel=1e-12) and dn[0] == 0.0


def test_near_operator_consistency():
    """Near correction: exact - quadrature is small for the farther pairs and the corrected K'
    still has the sphere eigenvalue -1/2 for the constant."""
    p = bem.Panels(*octasphere(12))
    i, j, c_pot, c_dn, self_pot = bem.near_corrections(p, 3.0)
    assert len(i) > 0 and np.all(i != j)
    x = np.ones(p.n)
    assert abs(np.mean(bem.apply_kprime_near(p, x)) + 0.5) < 0.03
    # the single-layer self term of a flat panel is positive and O(sqrt(A))
    assert np.all(self_pot > 0) and np.allclose(self_pot / np.sqrt(p.area), self_pot[0] / np.sqrt(p.area[0]), rtol=0.3)


# ---------------------------------------------------------------- round-2 pins

def test_near_pairs_equal_brute_force_on_a_tiny_mesh():
    """near_pairs (KD-tree query + filter) equals the O(n^2) brute-force enumeration of its definition
    j != i, |c_i - c_j| < eta sqrt(A_j) on a small irregular mesh (different areas per panel)."""
    cfg = configs.lysozyme(nu=6, n_atoms=10)
    p = bem.Panels(cfg["vertices"], cfg["triangles"])
    for eta in (1.0, 2.5, 4.0):
        i, j = bem.near_pairs(p, eta)
        d = np.linalg.norm(p.centroid[:, None, :] - p.centroid[None, :, :], axis=2)
        want = set(zip(*np.nonzero((d < eta * np.sqrt(p.area)[None, :]) & ~np.eye(p.n, dtype=bool))))
        got = set(zip(i.tolist(), j.tolist()))
        assert got == want and len(want) > 0
        assert not any(a == b for a, b in got)


def test_charge_potential_mean_value_on_a_sphere():
    """psi_i = sum_k q_k G(c_i, r_k): by the shell theorem the area-weighted sum over a sphere of
    radius a of the potential of an interior unit charge is q a (independent of the charge's
    position inside); the flat-panel centroid rule converges to it with refinement."""
    errs = []
    for nu in (8, 16, 32):
        cfg = configs.born(nu, radius=2.0)
        p = bem.Panels(cfg["vertices"], cfg["triangles"])
        for r in ([0.0, 0.0, 0.0], [0.3, -0.5, 0.7]):
            psi = bem.charge_potential(p, np.array([r]), np.array([1.0]))
            errs.append(abs(np.sum(p.area * psi) / 2.0 - 1.0))
    assert errs[-1] < 2e-4 and errs[-2] < 2e-4
    assert errs[-1] < errs[-3] < errs[1]  # monotone in nu (off-centre charge)
    assert 3.0 < errs[-3] / errs[-1] < 5.0  # second order in the panel size


def test_rows_helpers_equal_full_operators():
    """KprimeRows / SingleRows (the split used to time the oracle) give the rows of the full sums."""
    cfg = configs.kirkwood(6)
    p = bem.Panels(cfg["vertices"], cfg["triangles"], K=3)
    x = np.random.default_rng(3).normal(size=p.n)
    rows = np.array([0, 5, 17, p.n - 1])
    assert np.array_equal(bem.KprimeRows(p, x)(rows), bem.apply_kprime(p, x)[rows])
    assert np.array_equal(bem.SingleRows(p, x)(rows), bem.apply_single(p, x)[rows])
    En = bem.normal_field(p, cfg["charge_xyz"], cfg["charge_q"], 4.0)
    assert np.array_equal(bem.normal_field(p, cfg["charge_xyz"], cfg["charge_q"], 4.0, rows=rows), En[rows])


def test_double_layer_adjoint_of_kprime_and_gauss_limit():
    """Double layer K: with the centroid rule the discrete K is exactly the
    area-weighted adjoint of the (pinned) discrete K': sum_i A_i v_i (K'u)_i = sum_j A_j u_j (K v)_j;
    and Gauss's integral of the double-layer kernel over a closed surface seen from a surface point
    is -1/2 (principal value), so K 1 -> -1/2 on spheres, first order in the panel size."""
    devs = []
    for nu in (8, 16, 32):
        cfg = configs.born(nu, radius=1.5)
        p = bem.Panels(cfg["vertices"], cfg["triangles"])
        rng = np.random.default_rng(nu)
        u, v = rng.normal(size=p.n), rng.normal(size=p.n)
        lhs = np.sum(p.area * v * bem.apply_kprime(p, u))
        rhs = np.sum(p.area * u * bem.apply_double(p, v))
        assert abs(lhs - rhs) <= 1e-12 * np.sum(p.area * np.abs(v) * np.abs(bem.apply_kprime(p, np.abs(u))))
        devs.append(np.abs(bem.apply_double(p, np.ones(p.n)) + 0.5).max())
    assert devs[0] > devs[1] > devs[2] and devs[2] < 0.01, devs
    assert 1.6 < devs[1] / devs[2] < 2.5  # O(h)
    # a 3-point rule approaches the same limit
    cfg = configs.born(16)
    p3 = bem.Panels(cfg["vertices"], cfg["triangles"], K=3)
    assert abs(np.mean(bem.apply_double(p3, np.ones(p3.n))) + 0.5) < 0.02
