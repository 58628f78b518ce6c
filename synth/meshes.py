"""Seeded synthetic geometry shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no panel centroids/normals/areas,
no kernels, no quadrature): it only produces closed triangle meshes
(vertices f64 [n_v,3], triangles i32 [n_t,3], outward winding) and point charges
(xyz f64 [n_c,3], q f64 [n_c]).  Recipes follow SURVEY.md Sec. 8(d) and Appendix A:

* octasphere(nu): octahedron faces flat-subdivided into nu^2 triangles, vertices
  projected radially; 8 nu^2 faces, 4 nu^2 + 2 vertices (the
  "512-triangle icosphere" of BASELINE config 1 is the octasphere nu = 8).
* icosphere(k): 20 * 4^k faces, midpoint subdivision normalised every level.
* star_molecule(...): star-shaped "lysozyme-like" surface over an octasphere
  (SURVEY Sec. 8(d) C3 recipe) with interior atoms.
* replicate_grid(...): nx*ny*nz randomly rotated copies (Sec. 4.5
  "randomly oriented lysozyme molecules arranged on a regular Cartesian grid",
  P:807-831; SPEC.md replicate_grid S:84-92).
"""
from __future__ import annotations

import numpy as np

# Octahedron faces, SURVEY.md Appendix A (each (A, B, C) has cross(B-A, C-A) outward).
_EX, _EY, _EZ = np.eye(3, dtype=np.int64)
_OCTA_FACES = [
    (_EX, _EY, _EZ), (_EY, -_EX, _EZ), (-_EX, -_EY, _EZ), (-_EY, _EX, _EZ),
    (_EY, _EX, -_EZ), (-_EX, _EY, -_EZ), (-_EY, -_EX, -_EZ), (_EX, -_EY, -_EZ),
]


def octasphere(nu: int, radius: float = 1.0):
    """Octasphere with 8*nu^2 triangles; returns (vertices f64 [V,3], tri i32 [F,3])."""
    if nu < 1:
        raise ValueError("nu must be >= 1")
    pts, tris = [], []
    base = 0
    for A, B, C in _OCTA_FACES:
        ii, jj = np.meshgrid(np.arange(nu + 1), np.arange(nu + 1), indexing="ij")
        keep = ii + jj <= nu
        i, j = ii[keep], jj[keep]
        # integer lattice point nu*p = nu*A + (B-A) i + (C-A) j  (exact)
        p = nu * A[None, :] + np.outer(i, B - A) + np.outer(j, C - A)
        local = -np.ones((nu + 1, nu + 1), dtype=np.int64)
        local[i, j] = np.arange(i.size)
        pts.append(p)
        ci, cj = np.meshgrid(np.arange(nu), np.arange(nu), indexing="ij")
        up = ci + cj < nu
        a, b = ci[up], cj[up]
        tris.append(base + np.stack([local[a, b], local[a + 1, b], local[a, b + 1]], 1))
        dn = ci + cj < nu - 1
        a, b = ci[dn], cj[dn]
        tris.append(base + np.stack([local[a + 1, b], local[a + 1, b + 1], local[a, b + 1]], 1))
        base += i.size
    pts = np.concatenate(pts)
    tris = np.concatenate(tris)
    uniq, inv = np.unique(pts, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    v = uniq.astype(np.float64)
    v /= np.linalg.norm(v, axis=1)[:, None]
    v *= radius
    t = inv[tris].astype(np.int32)
    return v, t


def icosphere(k: int, radius: float = 1.0):
    """Icosphere with 20*4^k faces (midpoint subdivision, normalised every level)."""
    g = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array([[-1, g, 0], [1, g, 0], [-1, -g, 0], [1, -g, 0], [0, -1, g], [0, 1, g],
                  [0, -1, -g], [0, 1, -g], [g, 0, -1], [g, 0, 1], [-g, 0, -1], [-g, 0, 1]],
                 dtype=np.float64)
    v /= np.linalg.norm(v, axis=1)[:, None]
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9],
                  [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2],
                  [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5], [2, 4, 11], [6, 2, 10],
                  [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    verts = [tuple(x) for x in v]
    for _ in range(k):
        cache = {}
        vl = verts

        def mid(a, b):
            key = (a, b) if a < b else (b, a)
            if key not in cache:
                m = (np.array(vl[a]) + np.array(vl[b])) / 2.0
                m /= np.linalg.norm(m)
                vl.append(tuple(m))
                cache[key] = len(vl) - 1
            return cache[key]

        nf = []
        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [[a, ab, ca], [b, bc, ab], [c, ca, bc], [ab, bc, ca]]
        f = np.array(nf, dtype=np.int64)
    v = np.array(verts, dtype=np.float64) * radius
    return v, f.astype(np.int32)


def _real_sph_harm(l: int, m: int, theta, phi):
    """Real spherical harmonic (scipy's complex Y_l^m, real/imag parts); geometry only."""
    from scipy.special import sph_harm_y
    y = sph_harm_y(l, abs(m), theta, phi)
    if m > 0:
        return np.sqrt(2.0) * y.real
    if m < 0:
        return np.sqrt(2.0) * y.imag
    return y.real


def star_radius(u, semi_axes, alm):
    """rho(u) = rho_ell(u) * (1 + sum a_lm Y_lm(u)), clipped at 0.7 rho_ell."""
    a, b, c = semi_axes
    rho_ell = 1.0 / np.sqrt(u[:, 0] ** 2 / a ** 2 + u[:, 1] ** 2 / b ** 2 + u[:, 2] ** 2 / c ** 2)
    theta = np.arccos(np.clip(u[:, 2], -1.0, 1.0))
    phi = np.arctan2(u[:, 1], u[:, 0])
    pert = np.ones(len(u))
    for (l, m), coef in alm.items():
        pert += coef * _real_sph_harm(l, m, theta, phi)
    return np.maximum(rho_ell * pert, 0.7 * rho_ell)


def star_molecule(nu: int, semi_axes=(22.5, 15.0, 15.0), n_atoms: int = 2000, seed: int = 2,
                  qsum: float = 8.0, depth: float = 1.4, min_sep: float = 1.0):
    """Synthetic lysozyme-like molecule (SURVEY.md Sec. 8(d) C3 recipe).

    Surface x(u) = rho(u) u over the octasphere(nu) directions; atoms sampled uniformly
    inside rho(u) - depth with pairwise separation >= min_sep; q ~ N(0, 0.3^2) shifted so
    sum(q) = qsum.  Returns (vertices, triangles, charge_xyz, charge_q).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    alm = {}
    for l in range(2, 7):
        for m in range(-l, l + 1):
            alm[(l, m)] = rng.normal(0.0, 0.06 / l)
    u, tri = octasphere(nu, 1.0)
    v = u * star_radius(u, semi_axes, alm)[:, None]
    # atoms: rejection sampling in the bounding box
    amax = max(semi_axes) * 1.5
    acc = []
    grid = {}
    while len(acc) < n_atoms:
        cand = rng.uniform(-amax, amax, size=(4096, 3))
        r = np.linalg.norm(cand, axis=1)
        uu = cand / np.maximum(r, 1e-300)[:, None]
        ok = r < star_radius(uu, semi_axes, alm) - depth
        for p in cand[ok]:
            key = np.floor(p / min_sep).astype(int)
            near = [qn for dx in (-1, 0, 1) for dy in (-1, 0, 1) for dz in (-1, 0, 1)
                    for qn in grid.get((key[0] + dx, key[1] + dy, key[2] + dz), ())]
            if near and np.min(np.sum((np.array(near) - p) ** 2, axis=1)) < min_sep ** 2:
                continue
            grid.setdefault(tuple(key), []).append(p)
            acc.append(p)
            if len(acc) >= n_atoms:
                break
    acc = np.array(acc).reshape(-1, 3)
    q = rng.normal(0.0, 0.3, size=n_atoms)
    q += (qsum - q.sum()) / n_atoms
    return v, tri, acc.astype(np.float64), q.astype(np.float64)


def random_rotations(n: int, rng):
    """Uniform random rotation matrices via Shoemake's quaternion method."""
    u1, u2, u3 = rng.random(n), rng.random(n), rng.random(n)
    qw = np.sqrt(1 - u1) * np.sin(2 * np.pi * u2)
    qx = np.sqrt(1 - u1) * np.cos(2 * np.pi * u2)
    qy = np.sqrt(u1) * np.sin(2 * np.pi * u3)
    qz = np.sqrt(u1) * np.cos(2 * np.pi * u3)
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (qy * qy + qz * qz)
    R[:, 0, 1] = 2 * (qx * qy - qz * qw)
    R[:, 0, 2] = 2 * (qx * qz + qy * qw)
    R[:, 1, 0] = 2 * (qx * qy + qz * qw)
    R[:, 1, 1] = 1 - 2 * (qx * qx + qz * qz)
    R[:, 1, 2] = 2 * (qy * qz - qx * qw)
    R[:, 2, 0] = 2 * (qx * qz - qy * qw)
    R[:, 2, 1] = 2 * (qy * qz + qx * qw)
    R[:, 2, 2] = 1 - 2 * (qx * qx + qy * qy)
    return R


def replicate_grid(v, tri, cxyz, cq, n=(10, 10, 10), spacing=60.0, seed=5, jitter=0.0, copies=None,
                   charges=True):
    """n[0]*n[1]*n[2] randomly rotated copies on a grid.

    Each copy is rotated about the origin (the molecule's frame) by an independent
    uniform random rotation and translated to its grid point (+ optional uniform
    jitter of +-jitter Angstrom, "quasi-scattered").  `copies` = (first, count)
    materialises only that contiguous block of copies (the same rotations and positions as
    the full array: a rank's part for input_mode 1); `charges` = False skips the charges.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    nx, ny, nz = n
    nc = nx * ny * nz
    rad = np.linalg.norm(v, axis=1).max()
    if spacing <= 2 * rad + 2 * jitter:
        raise ValueError(f"spacing too small: need > {2 * rad + 2 * jitter:.3f}")
    R = random_rotations(nc, rng)
    gi = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1)
    shift = gi.reshape(-1, 3).astype(np.float64) * spacing
    if jitter > 0:
        shift += rng.uniform(-jitter, jitter, size=shift.shape)
    c0, cn = (0, nc) if copies is None else copies
    nv, nt, ncg = len(v), len(tri), len(cxyz)
    V = np.empty((cn, nv, 3))
    for i in range(cn):  # per-copy rotation keeps peak memory at one copy of temporaries
        np.matmul(v, R[c0 + i].T, out=V[i])
        V[i] += shift[c0 + i]
    C = np.empty((nc if charges else 0, ncg, 3))
    for c in range(len(C)):
        if ncg:
            np.matmul(cxyz, R[c].T, out=C[c])
            C[c] += shift[c]
    T = (tri[None, :, :].astype(np.int64) + (np.arange(cn, dtype=np.int64) * nv)[:, None, None])
    return (V.reshape(-1, 3), T.reshape(-1, 3).astype(np.int32), C.reshape(-1, 3),
            np.tile(cq, len(C)))
