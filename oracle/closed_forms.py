"""Closed-form sphere energies (oracle O12) -- TEST INFRASTRUCTURE ONLY.

Sphere of radius a, charges q_i at r_i (|r_i| < a), eps_I inside, eps_O outside,
internal units with explicit 1/(4 pi) (Eq. 4-6).

  Delta G = 1/(8 pi) sum_i sum_k q_i q_k sum_{n>=0} c_n (|r_i||r_k|)^n / a^(2n+1) P_n(cos g_ik)
  c_n(lam) = -(n+1) f / (eps_I (2n+1) (1 - f lam))

lam = lam_n = -1/(2(2n+1)) (the K' eigenvalues on the sphere) gives the exact
Kirkwood solution, c_n = -(eps_O-eps_I)(n+1)/(eps_I(n eps_I + (n+1) eps_O)), whose n = 0
term is the Born energy (q^2/(8 pi a))(1/eps_O - 1/eps_I).
lam = s gives BIBEE with scale s (Eq. 7 and P:455-457, reading A3).
"""
from __future__ import annotations

import numpy as np


def born(q: float, a: float, eps_in: float, eps_out: float) -> float:
    """Born ion: (q^2/(8 pi a)) (1/eps_O - 1/eps_I)."""
    return q * q / (8.0 * np.pi * a) * (1.0 / eps_out - 1.0 / eps_in)


def sphere_series(cxyz, cq, a, eps_in, eps_out, lam="exact", terms=200):
    """Delta G of the sphere for lam in {'exact'} or a BIBEE scale s (float)."""
    cxyz = np.asarray(cxyz, np.float64).reshape(-1, 3)
    cq = np.asarray(cq, np.float64).reshape(-1)
    f = 2.0 * (eps_out - eps_in) / (eps_in + eps_out)
    n = np.arange(terms, dtype=np.float64)
    if lam == "exact":
        lamn = -1.0 / (2.0 * (2.0 * n + 1.0))
    else:
        lamn = np.full(terms, float(lam))
    c = -(n + 1.0) * f / (eps_in * (2.0 * n + 1.0) * (1.0 - f * lamn))
    r = np.linalg.norm(cxyz, axis=1)
    tot = 0.0
    for i in range(len(cq)):
        for k in range(len(cq)):
            if r[i] == 0.0 or r[k] == 0.0:
                cosg = 1.0
            else:
                cosg = float(np.dot(cxyz[i], cxyz[k]) / (r[i] * r[k]))
            t = r[i] * r[k] / (a * a)
            # sum_n c_n t^n P_n(cosg) / a
            pm1, p = 1.0, cosg
            s = c[0]
            tn = 1.0
            for m in range(1, terms):
                tn *= t
                if tn == 0.0:
                    break
                s += c[m] * tn * p
                pm1, p = p, ((2 * m + 1) * cosg * p - m * pm1) / (m + 1)
            tot += cq[i] * cq[k] * s / a
    return tot / (8.0 * np.pi)
