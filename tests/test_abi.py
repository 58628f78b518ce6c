"""The C-ABI library loads and exports every symbol include/fmmbem.h declares (no GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fmmbem.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fmmbem_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_1007_4591_b200 import _build
    _build.build()
    from paper_1007_4591_b200 import _lib
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s


def test_binding_covers_header(lib):
    from paper_1007_4591_b200 import _lib
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_default_options_and_struct_sizes(lib):
    from paper_1007_4591_b200 import _lib
    o = _lib.Options()
    assert lib.fmmbem_default_options(ctypes.byref(o)) == 0
    assert o.struct_size == ctypes.sizeof(_lib.Options)
    assert (o.terms, o.leaf_points, o.quad_points, o.nranks) == (10, 64, 1, 1)
    assert lib.fmmbem_default_options(None) == _lib.E_INVALID


def test_create_rejects_bad_input_without_touching_gpu(lib):
    from paper_1007_4591_b200 import _lib
    h = ctypes.c_void_p(1)
    # null mesh -> E_INVALID and *out = NULL
    assert lib.fmmbem_create(None, None, 4.0, 80.0, None, ctypes.byref(h)) == _lib.E_INVALID
    assert h.value is None
    assert b"null" in lib.fmmbem_last_error()
    lib.fmmbem_destroy(None)  # NULL-safe
    # option validation happens before any CUDA call: charge_terms must be 0 or a rotation order <= terms
    import numpy as np
    v = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], np.float64)
    t = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.int32)
    mesh = _lib.Mesh(len(v), v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(t),
                     t.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    for ct, terms in ((11, 13), (14, 13), (-1, 13), (9, 10)):
        o = _lib.Options()
        lib.fmmbem_default_options(ctypes.byref(o))
        o.terms, o.charge_terms = terms, ct
        assert lib.fmmbem_create(ctypes.byref(mesh), None, 4.0, 80.0, ctypes.byref(o), ctypes.byref(h)) == _lib.E_INVALID
        assert b"charge_terms" in lib.fmmbem_last_error()


def test_sm100a_code_in_library():
    import subprocess
    from paper_1007_4591_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1007_4591_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).replace("oracle keeps", ""), f
