"""The five BASELINE.json workloads as seeded synthetic inputs.

Every function returns a plain dict of numpy arrays:
  vertices f64 [n_v,3] (Angstrom), triangles i32 [n_p,3] (0-based, outward winding),
  charge_xyz f64 [n_c,3], charge_q f64 [n_c], eps_in, eps_out (4 / 80).
No arithmetic of the method lives here.
"""
from __future__ import annotations

import numpy as np

from .meshes import octasphere, icosphere, star_molecule, replicate_grid

EPS_IN, EPS_OUT = 4.0, 80.0  # PAPER.md P:653 "epsilon_I = 4 and epsilon_II = 80"


def _pack(v, t, cx, cq, name):
    return dict(name=name, vertices=np.ascontiguousarray(v, np.float64),
                triangles=np.ascontiguousarray(t, np.int32),
                charge_xyz=np.ascontiguousarray(np.asarray(cx, np.float64).reshape(-1, 3)),
                charge_q=np.ascontiguousarray(np.asarray(cq, np.float64).reshape(-1)),
                eps_in=EPS_IN, eps_out=EPS_OUT)


def born(nu: int = 8, radius: float = 1.0, q: float = 1.0):
    """C1: octasphere(nu) (nu=8 -> 512 panels), one charge at the centre."""
    v, t = octasphere(nu, radius)
    return _pack(v, t, [[0.0, 0.0, 0.0]], [q], f"born_octa{nu}")


def born_ico(k: int, radius: float = 1.0, q: float = 1.0):
    v, t = icosphere(k, radius)
    return _pack(v, t, [[0.0, 0.0, 0.0]], [q], f"born_ico{k}")


def kirkwood_charges(n: int = 10, rmax: float = 0.6, seed: int = 1):
    """r = rmax*U^(1/3), direction = normalised N(0,I3), q = +-1 by a fair coin."""
    rng = np.random.Generator(np.random.PCG64(seed))
    r = rmax * rng.random(n) ** (1.0 / 3.0)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    q = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return d * r[:, None], q


def kirkwood(nu: int = 64, n_charges: int = 10, seed: int = 1, radius: float = 1.0):
    """C2: octasphere nu=64 (32,768 panels), 10 off-centre charges at r <= 0.6 a."""
    v, t = octasphere(nu, radius)
    cx, cq = kirkwood_charges(n_charges, 0.6 * radius, seed)
    return _pack(v, t, cx, cq, f"kirkwood_octa{nu}")


def lysozyme(nu: int = 113, n_atoms: int = 2000, seed: int = 2, semi_axes=(22.5, 15.0, 15.0)):
    """C3: star-shaped synthetic lysozyme, nu=113 -> 102,152 panels, 2,000 atoms."""
    v, t, cx, cq = star_molecule(nu, semi_axes, n_atoms, seed)
    return _pack(v, t, cx, cq, f"lysozyme_nu{nu}")


def binding(nu_protein: int = 187, nu_ligand: int = 50, gap: float = 1.0):
    """C4: protein (26,22,20) A nu=187 + ligand (5,3.5,2.5) A nu=50 on +x, 1 A surface gap.

    Returns dict(complex=..., protein=..., ligand=...) (Eq. 10).
    """
    pv, pt, pcx, pcq = star_molecule(nu_protein, (26.0, 22.0, 20.0), 4800, seed=3)
    lv, lt, lcx, lcq = star_molecule(nu_ligand, (5.0, 3.5, 2.5), 40, seed=4, qsum=0.0,
                                     depth=1.0, min_sep=0.8)
    from scipy.spatial import cKDTree
    tree = cKDTree(pv)
    # slide the ligand along +x: smallest shift with min vertex distance >= gap
    lo = float(pv[:, 0].max() - lv[:, 0].min() - 3.0)
    hi = lo + 20.0
    for _ in range(50):
        mid = 0.5 * (lo + hi)
        d, _ = tree.query(lv + np.array([mid, 0.0, 0.0]))
        if d.min() < gap:
            lo = mid
        else:
            hi = mid
    shift = np.array([hi, 0.0, 0.0])
    lv2, lcx2 = lv + shift, lcx + shift
    cv = np.concatenate([pv, lv2])
    ct = np.concatenate([pt, lt + len(pv)]).astype(np.int32)
    return dict(protein=_pack(pv, pt, pcx, pcq, "protein"),
                ligand=_pack(lv2, lt, lcx2, lcq, "ligand"),
                complex=_pack(cv, ct, np.concatenate([pcx, lcx2]), np.concatenate([pcq, lcq]),
                              "complex"))


def array(n=(10, 10, 10), nu: int = 113, spacing: float = 60.0, seed: int = 5,
          jitter: float = 0.0, base=None):
    """C5: n copies of C3 on a grid, random rotations (seed 5): 102,152,000 panels at 10^3."""
    if base is None:
        base = lysozyme(nu)
    V, T, C, Q = replicate_grid(base["vertices"], base["triangles"], base["charge_xyz"],
                                base["charge_q"], n, spacing, seed, jitter)
    return _pack(V, T, C, Q, f"array_{n[0]}x{n[1]}x{n[2]}_nu{nu}")


def array_part(n=(10, 10, 10), rank: int = 0, world: int = 1, nu: int = 113, spacing: float = 60.0,
               seed: int = 5, jitter: float = 0.0, base=None):
    """Rank `rank`'s part of the C5-style array for input_mode 1: the contiguous block of copies
    [C r / world, C (r + 1) / world) (same rotations as `array`), ALL charges.  Concatenated in rank
    order the parts are `array(...)`, so the library's global ids are the array's triangle indices."""
    if base is None:
        base = lysozyme(nu)
    nc = n[0] * n[1] * n[2]
    c0, c1 = nc * rank // world, nc * (rank + 1) // world
    V, T, C, Q = replicate_grid(base["vertices"], base["triangles"], base["charge_xyz"], base["charge_q"], n,
                                spacing, seed, jitter, copies=(c0, c1 - c0))
    out = _pack(V, T, C, Q, f"array_{n[0]}x{n[1]}x{n[2]}_nu{nu}_part{rank}of{world}")
    out["first_panel"] = c0 * len(base["triangles"])
    out["n_panels_total"] = nc * len(base["triangles"])
    return out


def random_cube(n: int, seed: int = 0, width: float = 1.0):
    """Uniform random points in a cube (the paper's scaling control); points only."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.random((n, 3)) * width, rng.uniform(-1.0, 1.0, n)


def cube_panels(n: int, seed: int = 0, width: float = 100.0, eps: float = 1e-4):
    """The random-cube control ("N = 10^8 ... randomly distributed in a cube") as a
    panel set the library accepts: one tiny right triangle (legs eps, far below the ~0.2 A mean
    point spacing at 1e8 points in a 100 A cube) per uniform random point p, vertices
    (p, p + eps e_x, p + eps e_y).  With the centroid rule a panel is a point source of weight
    A_j x_j; `charge_per_area` = 1/A_j turns unit charges into x.  No charges."""
    rng = np.random.Generator(np.random.PCG64(seed))
    p = rng.random((n, 3)) * width
    v = np.empty((n, 3, 3))
    v[:, 0] = p
    v[:, 1] = p
    v[:, 1, 0] += eps
    v[:, 2] = p
    v[:, 2, 1] += eps
    t = np.arange(3 * n, dtype=np.int64).reshape(n, 3)
    out = _pack(v.reshape(-1, 3), t.astype(np.int32), np.zeros((0, 3)), np.zeros(0), f"random_cube_{n}")
    out["charge_per_area"] = 2.0 / (eps * eps)
    return out
