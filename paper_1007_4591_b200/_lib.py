"""ctypes binding of libfmmbem.so (argument marshalling only; include/fmmbem.h).

The library is required: importing this module raises ImportError when the in-tree
shared object is missing or cannot be loaded -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FMMBEM_LIB") or os.path.join(HERE, "libfmmbem.so")  # override: A/B builds

OK, NOT_CONVERGED = 0, 1
E_INVALID, E_DEGENERATE, E_COINCIDENT, E_CUDA, E_NOMEM, E_NCCL = -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "OK", 1: "NOT_CONVERGED", -1: "E_INVALID", -2: "E_DEGENERATE", -3: "E_COINCIDENT",
                -4: "E_CUDA", -5: "E_NOMEM", -6: "E_NCCL"}
OP_KPRIME, OP_SINGLE, OP_A, OP_DOUBLE = 0, 1, 2, 3
BIBEE_CFA, BIBEE_P, BIBEE_LB = 0, 1, 2


class Mesh(C.Structure):
    _fields_ = [("n_vertices", C.c_int64), ("xyz", C.POINTER(C.c_double)),
                ("n_triangles", C.c_int64), ("tri", C.POINTER(C.c_int32))]


class Charges(C.Structure):
    _fields_ = [("n", C.c_int64), ("xyz", C.POINTER(C.c_double)), ("q", C.POINTER(C.c_double))]


class Options(C.Structure):
    _fields_ = [("struct_size", C.c_int32), ("terms", C.c_int32), ("leaf_points", C.c_int32),
                ("quad_points", C.c_int32), ("near_mode", C.c_int32), ("near_radius", C.c_float),
                ("self_term", C.c_int32), ("direct", C.c_int32), ("deterministic", C.c_int32),
                ("device", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_id", C.c_void_p), ("input_mode", C.c_int32), ("charge_terms", C.c_int32)]


class SolveOptions(C.Structure):
    _fields_ = [("tol", C.c_double), ("restart", C.c_int32), ("max_iters", C.c_int32),
                ("x0_dev", C.c_void_p)]


class Energy(C.Structure):
    _fields_ = [("dG_internal", C.c_double), ("dG_kcal_mol", C.c_double), ("iterations", C.c_int32),
                ("rel_residual", C.c_double)]


class Timing(C.Structure):
    _fields_ = [(k, C.c_double) for k in ("tree", "upward", "m2l", "p2p", "l2p", "near", "comm", "gmres",
                                          "total")] + [("p2p_interactions", C.c_int64), ("m2l_pairs", C.c_int64)] + \
        [(k, C.c_double) for k in ("p2m", "m2m", "l2l", "leaf_l2p", "bibee")]


class TreeInfo(C.Structure):
    _fields_ = [("levels", C.c_int32), ("n_leaves", C.c_int64), ("n_cells", C.c_int64),
                ("n_panels", C.c_int64), ("n_charges", C.c_int64), ("nbr_pairs", C.c_int64),
                ("m2l_pairs", C.c_int64), ("root_width", C.c_double), ("root_origin", C.c_double * 3),
                ("expansion_slots", C.c_int64), ("let_send_peers", C.c_int32), ("let_recv_peers", C.c_int32),
                ("let_cells_sent", C.c_int64), ("let_cells_recv", C.c_int64), ("let_shared_cells", C.c_int64),
                ("halo_panels_sent", C.c_int64), ("halo_panels_recv", C.c_int64)]


# symbol -> (restype, argtypes); every entry point declared in include/fmmbem.h
ABI_VERSION = 3  # include/fmmbem.h FMMBEM_ABI_VERSION this binding is written for

SIGNATURES = {
    "fmmbem_abi_version": (C.c_int32, []),
    "fmmbem_struct_size": (C.c_int64, [C.c_char_p]),
    "fmmbem_default_options": (C.c_int, [C.POINTER(Options)]),
    "fmmbem_get_unique_id": (C.c_int, [C.c_void_p]),
    "fmmbem_split_costs": (C.c_int, [C.POINTER(C.c_double), C.c_int64, C.c_int32, C.POINTER(C.c_int64)]),
    "fmmbem_create": (C.c_int, [C.POINTER(Mesh), C.POINTER(Charges), C.c_double, C.c_double,
                                C.POINTER(Options), C.POINTER(C.c_void_p)]),
    "fmmbem_destroy": (None, [C.c_void_p]),
    "fmmbem_num_local_panels": (C.c_int64, [C.c_void_p]),
    "fmmbem_local_panel_ids": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "fmmbem_matvec": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "fmmbem_matvec_host": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "fmmbem_solve": (C.c_int, [C.c_void_p, C.POINTER(SolveOptions), C.c_void_p,
                               C.POINTER(C.c_double), C.POINTER(Energy)]),
    "fmmbem_bibee_energy": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.POINTER(Energy)]),
    "fmmbem_charge_fields": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "fmmbem_reset_fields": (C.c_int, [C.c_void_p]),
    "fmmbem_reaction_potential": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]),
    "fmmbem_last_timing": (C.c_int, [C.c_void_p, C.POINTER(Timing)]),
    "fmmbem_tree_info_get": (C.c_int, [C.c_void_p, C.POINTER(TreeInfo)]),
    "fmmbem_last_error": (C.c_char_p, []),
    "fmmbem_plan_create": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int64,
                                     C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "fmmbem_plan_destroy": (None, [C.c_void_p]),
    "fmmbem_plan_list": (C.c_int64, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
}

_lib = None


def load():
    """Load the in-tree libfmmbem.so (raises ImportError when it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fmmbem_abi_version() != ABI_VERSION:
        raise ImportError(f"{LIB_PATH}: ABI version {lib.fmmbem_abi_version()}, binding expects {ABI_VERSION}")
    for nm, st in (("options", Options), ("timing", Timing), ("energy", Energy), ("tree_info", TreeInfo),
                   ("solve_options", SolveOptions)):
        if lib.fmmbem_struct_size(nm.encode()) != C.sizeof(st):
            raise ImportError(f"{LIB_PATH}: sizeof({nm}) differs from the binding's ctypes struct")
    _lib = lib
    return lib


class FmmbemError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def check(code):
    if code < 0:
        raise FmmbemError(code, load().fmmbem_last_error().decode())
    return code
