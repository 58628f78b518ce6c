"""ctypes loader for oracle/direct.c (TEST INFRASTRUCTURE ONLY).

The shared object is compiled by `build_oracle()` (called from __graft_entry__.build()
and lazily on first use) with plain `gcc -O2 -fopenmp` (no fast-math).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "direct.c")
_SO = os.path.join(_HERE, "_direct.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = ctypes.CDLL(_SO)
        d = ctypes.POINTER(ctypes.c_double)
        i = ctypes.POINTER(ctypes.c_int64)
        L.oracle_dn_sum.argtypes = [ctypes.c_int64, d, d, i, ctypes.c_int64, d, d, i, d]
        L.oracle_dn_sum.restype = ctypes.c_int
        L.oracle_pot_sum.argtypes = [ctypes.c_int64, d, i, ctypes.c_int64, d, d, i, d]
        L.oracle_pot_sum.restype = ctypes.c_int
        L.oracle_dipole_sum.argtypes = [ctypes.c_int64, d, i, ctypes.c_int64, d, d, d, i, d]
        L.oracle_dipole_sum.restype = ctypes.c_int
        L.oracle_threads.restype = ctypes.c_int
        L.oracle_tri_integrals.argtypes = [ctypes.c_int64, d, d, d, ctypes.POINTER(ctypes.c_int32), d, d]
        L.oracle_tri_integrals.restype = None
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def threads() -> int:
    return int(lib().oracle_threads())


def dn_sum(x, n, tid, y, w, owner):
    x = np.ascontiguousarray(x, np.float64); n = np.ascontiguousarray(n, np.float64)
    y = np.ascontiguousarray(y, np.float64); w = np.ascontiguousarray(w, np.float64)
    tid = None if tid is None else np.ascontiguousarray(tid, np.int64)
    owner = None if owner is None else np.ascontiguousarray(owner, np.int64)
    out = np.zeros(len(x))
    bad = lib().oracle_dn_sum(len(x), _dp(x), _dp(n), _ip(tid), len(y), _dp(y), _dp(w),
                              _ip(owner), _dp(out))
    if bad:
        raise ValueError("coincident target/source pair (SURVEY A14)")
    return out


def dipole_sum(x, tid, y, m, w, owner):
    """out[i] = sum_j w[j] m_j . (x_i - y_j) / (4 pi |x_i - y_j|^3)  (source-normal derivative of G)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64); m = np.ascontiguousarray(m, np.float64)
    w = np.ascontiguousarray(w, np.float64)
    tid = None if tid is None else np.ascontiguousarray(tid, np.int64)
    owner = None if owner is None else np.ascontiguousarray(owner, np.int64)
    out = np.zeros(len(x))
    bad = lib().oracle_dipole_sum(len(x), _dp(x), _ip(tid), len(y), _dp(y), _dp(m), _dp(w), _ip(owner), _dp(out))
    if bad:
        raise ValueError("coincident target/source pair (SURVEY A14)")
    return out


def pot_sum(x, tid, y, w, owner):
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64); w = np.ascontiguousarray(w, np.float64)
    tid = None if tid is None else np.ascontiguousarray(tid, np.int64)
    owner = None if owner is None else np.ascontiguousarray(owner, np.int64)
    out = np.zeros(len(x))
    bad = lib().oracle_pot_sum(len(x), _dp(x), _ip(tid), len(y), _dp(y), _dp(w), _ip(owner),
                               _dp(out))
    if bad:
        raise ValueError("coincident target/source pair (SURVEY A14)")
    return out


def tri_integrals(x, n, tv, self_flags=None):
    """Per row k: (int_T G(x_k, y) dA, int_T dG/dn_x(x_k, y) dA) over triangle tv[k] (3x3)."""
    x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
    n = np.ascontiguousarray(n, np.float64).reshape(-1, 3)
    tv = np.ascontiguousarray(tv, np.float64).reshape(-1, 9)
    sf = None if self_flags is None else np.ascontiguousarray(self_flags, np.int32)
    pot, dn = np.zeros(len(x)), np.zeros(len(x))
    lib().oracle_tri_integrals(len(x), _dp(x), _dp(n), _dp(tv),
                               None if sf is None else sf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                               _dp(pot), _dp(dn))
    return pot, dn
