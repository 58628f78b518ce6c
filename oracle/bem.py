"""FP64 oracle of the discrete BEM / BIBEE method -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this package.  It shares no code with paper_1007_4591_b200/ (the CUDA
path) and is written from PAPER.md (arXiv 1007.4591) with the readings of SURVEY.md
Sec. 8(c) (A1-A22), listed again in DESIGN.md.  Every operator is the plain definition
(direct O(N^2) sums / dense LU / textbook GMRES); nothing here is an FMM.

Notation (Sec. 2.1):
  panels j: centroid c_j, unit outward normal n_j, area A_j
  quadrature points y_jg with weights w_g, sum_g w_g = 1 (K = 1: the centroid)
  G(x,y) = 1/(4 pi |x-y|);  dG/dn_x = -n_x.(x-y)/(4 pi |x-y|^3)   (Eq. 4-5, explicit 1/4pi)
  f = 2(eps_II - eps_I)/(eps_I + eps_II), eps_hat = 1 - eps_I/eps_II  (reading A1)
"""
from __future__ import annotations

import numpy as np

from . import _cdirect

KCAL_PER_INTERNAL = 4.0 * np.pi * 332.0637  # SPEC.md S:409/S:455, SURVEY A13

# Appendix C quadrature rules (barycentric beta_g, weight w_g), SURVEY.md App. C.
# K = 1 is the paper's rule: "a single point, located at the center of the triangle".
_QUAD = {
    1: ([(1 / 3, 1 / 3, 1 / 3)], [1.0]),
    3: ([(2 / 3, 1 / 6, 1 / 6), (1 / 6, 2 / 3, 1 / 6), (1 / 6, 1 / 6, 2 / 3)], [1 / 3] * 3),
    6: ([(0.108103018168070, 0.445948490915965, 0.445948490915965),
         (0.445948490915965, 0.108103018168070, 0.445948490915965),
         (0.445948490915965, 0.445948490915965, 0.108103018168070),
         (0.816847572980459, 0.091576213509771, 0.091576213509771),
         (0.091576213509771, 0.816847572980459, 0.091576213509771),
         (0.091576213509771, 0.091576213509771, 0.816847572980459)],
        [0.223381589678011] * 3 + [0.109951743655322] * 3),
    7: ([(1 / 3, 1 / 3, 1 / 3),
         (0.059715871789770, 0.470142064105115, 0.470142064105115),
         (0.470142064105115, 0.059715871789770, 0.470142064105115),
         (0.470142064105115, 0.470142064105115, 0.059715871789770),
         (0.797426985353087, 0.101286507323456, 0.101286507323456),
         (0.101286507323456, 0.797426985353087, 0.101286507323456),
         (0.101286507323456, 0.101286507323456, 0.797426985353087)],
        [0.225] + [0.132394152788506] * 3 + [0.125939180544827] * 3),
}


def quad_rule(K: int):
    """(beta [K,3], w [K]) of the K-point rule."""
    if K not in _QUAD:
        raise ValueError(f"quad_points must be one of {sorted(_QUAD)}")
    b, w = _QUAD[K]
    return np.array(b, np.float64), np.array(w, np.float64)


class Panels:
    """O1: panel centroid, normal, area.

    centroid = mean of the 3 vertices; normal = normalised cross((v1-v0),(v2-v0))
    (orientation from the winding); area = |cross|/2.  A triangle with index out of
    range or area < 1e-14 * bbox_diag^2 is a hard error.
    """

    def __init__(self, vertices, triangles, K: int = 1):
        v = np.asarray(vertices, np.float64)
        t = np.asarray(triangles, np.int64)
        if t.size and (t.min() < 0 or t.max() >= len(v)):
            raise ValueError("triangle index out of range")
        v0, v1, v2 = v[t[:, 0]], v[t[:, 1]], v[t[:, 2]]
        self.tri_v = np.stack([v0, v1, v2], 1)  # [n, 3 vertices, 3]
        cr = np.cross(v1 - v0, v2 - v0)
        nrm = np.linalg.norm(cr, axis=1)
        scale2 = float(np.sum((v.max(0) - v.min(0)) ** 2)) if len(v) else 1.0
        bad = np.nonzero(0.5 * nrm < 1e-14 * scale2)[0]
        if bad.size:
            raise ValueError(f"degenerate triangle {int(bad[0])}")
        self.centroid = (v0 + v1 + v2) / 3.0
        self.normal = cr / nrm[:, None]
        self.area = 0.5 * nrm
        beta, w = quad_rule(K)
        self.K = K
        self.wq = w
        # y_jg = sum_a beta_ga v_{j,a}
        self.qpts = (beta[None, :, 0, None] * v0[:, None, :] + beta[None, :, 1, None] * v1[:, None, :]
                     + beta[None, :, 2, None] * v2[:, None, :])
        self.n = len(t)
        self._v, self._t = v, t  # kept for the curvature self-term option (vertex normals)

    # flattened quadrature sources: position, owner panel, weight factor A_j w_g
    def sources(self):
        y = self.qpts.reshape(-1, 3)
        owner = np.repeat(np.arange(self.n, dtype=np.int64), self.K)
        aw = (self.area[:, None] * self.wq[None, :]).reshape(-1)
        return y, owner, aw


def constants(eps_in: float, eps_out: float):
    """O2: f = 2(eps_II-eps_I)/(eps_I+eps_II), eps_hat = 1 - eps_I/eps_II (A1)."""
    if eps_in <= 0 or eps_out <= 0 or eps_in == eps_out:
        raise ValueError("need eps > 0 and eps_in != eps_out (SPEC S:40)")
    return 2.0 * (eps_out - eps_in) / (eps_in + eps_out), 1.0 - eps_in / eps_out


def normal_field(pan: Panels, cxyz, cq, eps_in: float, rows=None):
    """O3: E_i = (1/eps_I) sum_k q_k dG/dn_i(c_i, r_k)  (Eq. 1's 1/eps_I; Eq. 4; A2)."""
    idx = np.arange(pan.n, dtype=np.int64) if rows is None else np.asarray(rows, np.int64)
    if len(cq) == 0:
        return np.zeros(len(idx))
    return _cdirect.dn_sum(pan.centroid[idx], pan.normal[idx], None, cxyz, cq, None) / eps_in


def charge_potential(pan: Panels, cxyz, cq, rows=None):
    """psi_i = sum_k q_k G(c_i, r_k) at the centroids (K = 1): the charges' Coulomb potential whose
    area-weighted sum with sigma gives Delta G = 1/2 q^T C sigma (A20; Eq. 5-6)."""
    idx = np.arange(pan.n, dtype=np.int64) if rows is None else np.asarray(rows, np.int64)
    if len(cq) == 0:
        return np.zeros(len(idx))
    return _cdirect.pot_sum(pan.centroid[idx], None, np.asarray(cxyz, np.float64), np.asarray(cq, np.float64), None)


def mean_curvature(pan: Panels):
    """Per-panel mean curvature for the self_term = 1 option ("from vertex normals").

    Vertex normal n_a = normalised sum of the incident faces' area-weighted normals.  The normal
    curvature of the surface along the chord from the centroid c_i to vertex a is estimated by
    (n_a - n_i).(v_a - c_i) / |v_a - c_i|^2 (on a sphere of radius R, n(v) = (v - o)/R makes this
    1/R up to O(h)); the mean over the three chords estimates H_i.  Convex outward surface: H > 0.
    """
    v, t = pan._v, pan._t
    acc = np.zeros_like(v)
    for a in range(3):  # area-weighted face normals summed at each vertex
        np.add.at(acc, t[:, a], pan.normal * pan.area[:, None])
    nv = acc / np.linalg.norm(acc, axis=1)[:, None]
    H = np.zeros(pan.n)
    for a in range(3):
        d = v[t[:, a]] - pan.centroid
        H += np.einsum("ij,ij->i", nv[t[:, a]] - pan.normal, d) / np.einsum("ij,ij->i", d, d)
    return H / 3.0


def self_term_diag(pan: Panels):
    """K'_ii = -H_i sqrt(A_i/pi) / 4: the principal-value integral of dG/dn_i over the
    curved panel, modelled as a spherical cap of curvature H_i and area A_i.  On a sphere
    dG/dn_x(x, y) = -1/(8 pi R |x - y|) for x, y on the surface, and the integral of 1/|x - y| over
    a disc of radius a = sqrt(A/pi) is 2 pi a, giving -a/(4R)."""
    return -mean_curvature(pan) * np.sqrt(pan.area / np.pi) / 4.0


class KprimeRows:
    """O4 split in two: the source weights x_j A_j w_g (once per x) and then any rows i of
    (K'x)_i = sum_{j!=i} x_j A_j sum_g w_g dG/dn_i(c_i, y_jg) -- the same sums
    as apply_kprime, so that a timing of rows measures the direct sums only."""

    def __init__(self, pan: Panels, x):
        self.pan = pan
        self.y, self.owner, aw = pan.sources()
        self.w = np.repeat(np.asarray(x, np.float64), pan.K) * aw
        self.y = np.ascontiguousarray(self.y)

    def __call__(self, rows):
        idx = np.asarray(rows, np.int64)
        return _cdirect.dn_sum(self.pan.centroid[idx], self.pan.normal[idx], idx, self.y, self.w, self.owner)


def apply_kprime(pan: Panels, x, rows=None, self_term: bool = False):
    """O4: (K'x)_i = sum_{j!=i} x_j A_j sum_g w_g dG/dn_i(c_i, y_jg); K'_ii = 0,
    or K'_ii = self_term_diag (option self_term = 1)."""
    idx = np.arange(pan.n, dtype=np.int64) if rows is None else np.asarray(rows, np.int64)
    out = KprimeRows(pan, x)(idx)
    if self_term:
        out = out + self_term_diag(pan)[idx] * np.asarray(x, np.float64)[idx]
    return out


class SingleRows(KprimeRows):
    """O5 split like KprimeRows: (Vx)_i = sum_{j!=i} x_j A_j sum_g w_g G(c_i, y_jg) for any rows."""

    def __call__(self, rows):
        idx = np.asarray(rows, np.int64)
        return _cdirect.pot_sum(self.pan.centroid[idx], idx, self.y, self.w, self.owner)


def apply_double(pan: Panels, x, rows=None):
    """Double layer: (Kx)_i = sum_{j!=i} x_j A_j sum_g w_g dG/dn_y(c_i, y_jg), n_y = n_j --
    the continuum adjoint of K' (Eq. 4, P:326 uses K'); K_ii = 0 for a flat panel (c_i lies in its plane)."""
    y, owner, aw = pan.sources()
    w = np.repeat(np.asarray(x, np.float64), pan.K) * aw
    m = np.repeat(pan.normal, pan.K, axis=0)
    idx = np.arange(pan.n, dtype=np.int64) if rows is None else np.asarray(rows, np.int64)
    return _cdirect.dipole_sum(pan.centroid[idx], idx, y, m, w, owner)


def apply_single(pan: Panels, x, rows=None):
    """O5: (Vx)_i = sum_{j!=i} x_j A_j sum_g w_g G(c_i, y_jg)  (Eq. 5)."""
    idx = np.arange(pan.n, dtype=np.int64) if rows is None else np.asarray(rows, np.int64)
    return SingleRows(pan, x)(idx)


def near_pairs(pan: Panels, eta: float):
    """Near pairs of the analytic option: j != i with |c_i - c_j| < eta sqrt(A_j)."""
    from scipy.spatial import cKDTree
    rmax = eta * np.sqrt(pan.area.max())
    pr = cKDTree(pan.centroid).query_pairs(rmax, output_type="ndarray")
    if len(pr) == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    both = np.concatenate([pr, pr[:, ::-1]])
    i, j = both[:, 0].astype(np.int64), both[:, 1].astype(np.int64)
    keep = np.linalg.norm(pan.centroid[i] - pan.centroid[j], axis=1) < eta * np.sqrt(pan.area[j])
    o = np.lexsort((j[keep], i[keep]))
    return i[keep][o], j[keep][o]


def near_corrections(pan: Panels, eta: float):
    """For near_mode = 1: per near pair, (exact panel integral) - (K-point quadrature) of
    G and of dG/dn_i, and the single-layer self integrals int_{T_i} G(c_i, y) dA.  The exact
    integrals are done numerically (oracle/direct.c: adaptive subdivision / Duffy), never by the
    closed forms the CUDA path uses."""
    key = ("near", eta)
    if key in pan.__dict__:
        return pan.__dict__[key]
    i, j = near_pairs(pan, eta)
    ex_pot, ex_dn = _cdirect.tri_integrals(pan.centroid[i], pan.normal[i], pan.tri_v[j])
    q_pot, q_dn = np.zeros(len(i)), np.zeros(len(i))
    for g in range(pan.K):
        d = pan.centroid[i] - pan.qpts[j, g, :]
        r = np.linalg.norm(d, axis=1)
        q_pot += pan.wq[g] * pan.area[j] / (4 * np.pi * r)
        q_dn += pan.wq[g] * pan.area[j] * (-np.einsum("ij,ij->i", pan.normal[i], d) / (4 * np.pi * r ** 3))
    self_pot, _ = _cdirect.tri_integrals(pan.centroid, pan.normal, pan.tri_v, np.ones(pan.n, np.int32))
    out = (i, j, ex_pot - q_pot, ex_dn - q_dn, self_pot)
    pan.__dict__[key] = out
    return out


def apply_kprime_near(pan: Panels, x, eta: float = 3.0):
    """O4 with near_mode = 1: K' with the exact flat-panel integral for the near pairs."""
    i, j, _, c_dn, _ = near_corrections(pan, eta)
    x = np.asarray(x, np.float64)
    return apply_kprime(pan, x) + np.bincount(i, weights=c_dn * x[j], minlength=pan.n)


def apply_single_near(pan: Panels, x, eta: float = 3.0):
    """O5 with near_mode = 1: V with exact near-pair integrals and the analytic self term (A7)."""
    i, j, c_pot, _, self_pot = near_corrections(pan, eta)
    x = np.asarray(x, np.float64)
    return apply_single(pan, x) + np.bincount(i, weights=c_pot * x[j], minlength=pan.n) + self_pot * x


def apply_A(pan: Panels, x, f: float, self_term: bool = False):
    """GMRES operator (I - f K') x  ("A x = B q")."""
    return np.asarray(x, np.float64) - f * apply_kprime(pan, x, self_term=self_term)


def reaction_potential(pan: Panels, sigma, cxyz):
    """O7: (C sigma)_k = sum_j sigma_j A_j sum_g w_g G(r_k, y_jg)  (Eq. 5)."""
    y, owner, aw = pan.sources()
    w = np.repeat(np.asarray(sigma, np.float64), pan.K) * aw
    return _cdirect.pot_sum(np.asarray(cxyz, np.float64), None, y, w, None)


def solvation_energy(cq, phi_reac):
    """O8: Delta G = 1/2 sum_k q_k phi_reac(r_k)  (Eq. 6).  Returns (internal, kcal/mol)."""
    e = 0.5 * float(np.dot(np.asarray(cq, np.float64), phi_reac))
    return e, e * KCAL_PER_INTERNAL


def dense_kprime(pan: Panels, self_term: bool = False):
    """Dense K' (n_p <= ~10^4): column j = K' e_j, assembled entry by entry as in O4."""
    n = pan.n
    c, nr = pan.centroid, pan.normal
    Kp = np.zeros((n, n))
    for g in range(pan.K):
        y = pan.qpts[:, g, :]
        d = c[:, None, :] - y[None, :, :]
        r2 = np.einsum("ijk,ijk->ij", d, d)
        np.fill_diagonal(r2, 1.0)
        nd = np.einsum("ik,ijk->ij", nr, d)
        blk = -nd / (4.0 * np.pi * r2 * np.sqrt(r2)) * (pan.area * pan.wq[g])[None, :]
        np.fill_diagonal(blk, 0.0)
        Kp += blk
    if self_term:
        Kp[np.diag_indices(n)] = self_term_diag(pan)
    return Kp


def solve_dense(pan: Panels, E, f: float, self_term: bool = False):
    """O6 (direct): (I - f K') sigma = f E by dense LU."""
    A = np.eye(pan.n) - f * dense_kprime(pan, self_term)
    return np.linalg.solve(A, f * np.asarray(E))


def gmres(matvec, b, tol=1e-6, restart=30, max_iters=200):
    """O6 (iterative): restarted GMRES(m) of Saad & Schultz, FP64.

    Zero initial guess; modified Gram-Schmidt Arnoldi; Givens rotations; stops when the
    relative residual ||b - A x|| / ||b|| <= tol.  Returns
    (x, iterations, residual history [relative], converged).
    """
    b = np.asarray(b, np.float64)
    n = len(b)
    x = np.zeros(n)
    bn = np.linalg.norm(b)
    hist = [1.0]
    if bn == 0.0:
        return x, 0, hist, True
    its = 0
    while its < max_iters:
        r = b - matvec(x) if its else b.copy()
        beta = np.linalg.norm(r)
        if beta / bn <= tol:
            return x, its, hist, True
        m = min(restart, max_iters - its)
        V = np.zeros((m + 1, n))
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k_done = 0
        for k in range(m):
            w = matvec(V[k])
            for i in range(k + 1):
                H[i, k] = np.dot(V[i], w)
                w = w - H[i, k] * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            if H[k + 1, k] > 0:
                V[k + 1] = w / H[k + 1, k]
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            den = np.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = H[k, k] / den, H[k + 1, k] / den
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            its += 1
            k_done = k + 1
            hist.append(abs(g[k + 1]) / bn)
            if abs(g[k + 1]) / bn <= tol:
                break
        yk = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done])
        x = x + V[:k_done].T @ yk
        if hist[-1] <= tol:
            return x, its, hist, True
    return x, its, hist, False


def bibee_sigma(E, f: float, s: float):
    """O9: sigma_hat = f E / (1 - f s), s in {-1/2 (CFA), 0 (P), +1/2 (LB)} (A3, A4)."""
    d = 1.0 - f * s
    if d == 0.0:
        raise ValueError("1 - f s == 0 (SPEC S:383)")
    return f * np.asarray(E) / d


BIBEE_SCALE = {"cfa": -0.5, "p": 0.0, "lb": 0.5}


class Problem:
    """A molecule: mesh + charges + dielectrics; the full oracle pipeline (O1-O9)."""

    def __init__(self, cfg, K: int = 1, near_eta=None, self_term: bool = False):
        self.pan = Panels(cfg["vertices"], cfg["triangles"], K)
        self.near_eta = near_eta  # None: paper's quadrature only; else the analytic near-field option
        self.self_term = self_term  # True: curvature self-term K'_ii (option self_term = 1, A7)
        self.cxyz = np.asarray(cfg["charge_xyz"], np.float64).reshape(-1, 3)
        self.cq = np.asarray(cfg["charge_q"], np.float64).reshape(-1)
        self.eps_in, self.eps_out = float(cfg["eps_in"]), float(cfg["eps_out"])
        self.f, self.eps_hat = constants(self.eps_in, self.eps_out)
        self._E = None

    @property
    def E(self):
        if self._E is None:
            self._E = normal_field(self.pan, self.cxyz, self.cq, self.eps_in)
        return self._E

    def energy_of(self, sigma):
        return solvation_energy(self.cq, reaction_potential(self.pan, sigma, self.cxyz))

    def solve(self, method="dense", tol=1e-6, restart=30, max_iters=200):
        if method == "dense":
            sigma = solve_dense(self.pan, self.E, self.f, self.self_term)
            info = dict(iterations=0, converged=True)
        else:
            if self.near_eta is None:
                op = lambda v: apply_A(self.pan, v, self.f, self.self_term)  # noqa: E731
            else:
                op = lambda v: np.asarray(v) - self.f * apply_kprime_near(self.pan, v, self.near_eta)  # noqa: E731
            sigma, its, hist, conv = gmres(op, self.f * self.E, tol, restart, max_iters)
            info = dict(iterations=its, converged=conv, history=hist)
        e, kcal = self.energy_of(sigma)
        return dict(sigma=sigma, dG=e, dG_kcal=kcal, **info)

    def bibee(self, variant="cfa"):
        sig = bibee_sigma(self.E, self.f, BIBEE_SCALE[variant])
        e, kcal = self.energy_of(sig)
        return dict(sigma=sig, dG=e, dG_kcal=kcal)


def binding_energy(dg_complex: float, dg_protein: float, dg_ligand: float) -> float:
    """O10: Delta Delta G = G_complex - G_protein - G_ligand (Eq. 10)."""
    return dg_complex - dg_protein - dg_ligand


def rel_l2(y, y_ref) -> float:
    """O11: ||y - y_ref||_2 / ||y_ref||_2 (P:580-587 'L2-norm of the relative error')."""
    y = np.asarray(y, np.float64); y_ref = np.asarray(y_ref, np.float64)
    return float(np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref))
