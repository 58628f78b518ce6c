"""Thin Python wrapper of the C ABI (include/fmmbem.h): argument marshalling only.

Every step of the hot path runs in libfmmbem.so's CUDA kernels; PyTorch is used for
device tensors and streams.  Vectors are in the library's LOCAL (Morton) order; use
`local_ids` / `to_local` / `to_global` to map from / to the caller's triangle order.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

BIBEE = {"cfa": L.BIBEE_CFA, "p": L.BIBEE_P, "lb": L.BIBEE_LB}
OPS = {"kprime": L.OP_KPRIME, "single": L.OP_SINGLE, "A": L.OP_A, "double": L.OP_DOUBLE}


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def get_unique_id() -> bytes:
    """128-byte NCCL unique id for a multi-GPU Solver (call on rank 0, broadcast the bytes)."""
    buf = C.create_string_buffer(128)
    L.check(L.load().fmmbem_get_unique_id(buf))
    return buf.raw


def split_costs(costs, parts):
    """Contiguous equal-cost split used by the domain decomposition (pure host code)."""
    c = np.ascontiguousarray(costs, np.float64)
    b = np.empty(parts + 1, np.int64)
    L.check(L.load().fmmbem_split_costs(c.ctypes.data_as(C.POINTER(C.c_double)), len(c), parts,
                                        b.ctypes.data_as(C.POINTER(C.c_int64))))
    return b


def default_options(**kw):
    lib = L.load()
    o = L.Options()
    L.check(lib.fmmbem_default_options(C.byref(o)))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, v)
    return o


class Solver:
    """One molecule: fmmbem_create(...) + the calls of the C ABI."""

    def __init__(self, vertices, triangles, charge_xyz=None, charge_q=None, eps_in=4.0, eps_out=80.0,
                 **options):
        import torch
        self._torch = torch
        self.lib = L.load()
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
        t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
        cx = np.ascontiguousarray(np.zeros((0, 3)) if charge_xyz is None else charge_xyz, np.float64).reshape(-1, 3)
        cq = np.ascontiguousarray(np.zeros(0) if charge_q is None else charge_q, np.float64).reshape(-1)
        if len(cx) != len(cq):
            raise ValueError("charge_xyz and charge_q differ in length")
        nccl_id = options.pop("nccl_id", None)
        self.options = default_options(**options)
        self.device = int(self.options.device)
        self._id_buf = None
        if self.options.nranks > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nranks > 1 needs the 128-byte nccl_id of rank 0")
            self._id_buf = C.create_string_buffer(bytes(nccl_id), 128)
            self.options.nccl_id = C.cast(self._id_buf, C.c_void_p)
        mesh = L.Mesh(len(v), _dp(v), len(t), t.ctypes.data_as(C.POINTER(C.c_int32)))
        chg = L.Charges(len(cq), _dp(cx) if len(cq) else None, _dp(cq) if len(cq) else None)
        h = C.c_void_p()
        L.check(self.lib.fmmbem_create(C.byref(mesh), C.byref(chg), float(eps_in), float(eps_out),
                                       C.byref(self.options), C.byref(h)))
        self._h = h
        self.n = int(self.lib.fmmbem_num_local_panels(h))
        ids = np.empty(self.n, np.int64)
        L.check(self.lib.fmmbem_local_panel_ids(h, ids.ctypes.data_as(C.POINTER(C.c_int64))))
        self.local_ids = ids
        self.n_charges = len(cq)
        self.eps_in, self.eps_out = float(eps_in), float(eps_out)

    @classmethod
    def from_config(cls, cfg, **options):
        return cls(cfg["vertices"], cfg["triangles"], cfg["charge_xyz"], cfg["charge_q"], cfg["eps_in"],
                   cfg["eps_out"], **options)

    @classmethod
    def distributed(cls, cfg, group=None, **options):
        """One rank of a multi-GPU solver; torch.distributed must be initialised.  Rank 0 draws the
        NCCL id and torch.distributed broadcasts it.  input_mode 0 (default): every rank passes the
        full problem; input_mode=1: `cfg` holds only this rank's part of the mesh (all charges), see
        include/fmmbem.h."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [get_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls.from_config(cfg, rank=rank, nranks=world, nccl_id=obj[0], **options)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.fmmbem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- order helpers
    def to_local(self, x_global):
        return np.asarray(x_global)[self.local_ids]

    def to_global(self, x_local):
        x_local = np.asarray(x_local)
        out = np.empty_like(x_local)
        out[self.local_ids] = x_local
        return out

    def _dev(self):
        return self._torch.device("cuda", self.device)

    def _vec(self, x):
        torch = self._torch
        if not isinstance(x, torch.Tensor):
            x = torch.as_tensor(np.asarray(x, np.float32))
        x = x.to(device=self._dev(), dtype=torch.float32).contiguous()
        if x.numel() != self.n:
            raise ValueError(f"vector of {x.numel()} entries, expected {self.n}")
        return x

    def _check_dev(self, t, what):
        """A caller-provided device buffer the library writes or reads in place: float32,
        contiguous, n entries, on this ctx's device (the ABI takes a raw pointer)."""
        torch = self._torch
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{what} must be a torch tensor")
        if t.dtype != torch.float32 or not t.is_contiguous() or t.numel() != self.n or t.device != self._dev():
            raise ValueError(f"{what} must be a contiguous float32 tensor of {self.n} entries on {self._dev()}")
        return t

    def _sync_current(self):
        # blocking ABI calls run on the library's own stream: finish the caller's pending work on
        # the buffers they read or write first (include/fmmbem.h "Ordering")
        self._torch.cuda.current_stream(self._dev()).synchronize()

    # ---- ABI calls
    def matvec(self, x, op="kprime", out=None, stream=None):
        """y = op(x) on the GPU (local order); x: torch CUDA float32 tensor or array."""
        torch = self._torch
        x = self._vec(x)
        y = torch.empty_like(x) if out is None else self._check_dev(out, "out")
        cur = torch.cuda.current_stream(self._dev())
        st = cur if stream is None else stream
        if st != cur:  # the kernels read x / write y on st: keep the allocator from recycling them early
            st.wait_stream(cur)
            x.record_stream(st)
            y.record_stream(st)
        L.check(self.lib.fmmbem_matvec(self._h, OPS[op], C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                       C.c_void_p(st.cuda_stream)))
        return y

    def matvec_host(self, x_host, op="kprime", y_host=None):
        """End-to-end product with host buffers (copies inside the library)."""
        x = np.ascontiguousarray(x_host, np.float32)
        if x.size != self.n:
            raise ValueError(f"x_host has {x.size} entries, expected {self.n}")
        if y_host is None:
            y = np.empty_like(x)
        else:
            y = y_host
            if not (isinstance(y, np.ndarray) and y.dtype == np.float32 and y.flags.c_contiguous
                    and y.size == self.n and y.flags.writeable):
                raise ValueError(f"y_host must be a writeable contiguous float32 array of {self.n} entries")
        L.check(self.lib.fmmbem_matvec_host(self._h, OPS[op], C.c_void_p(x.ctypes.data),
                                            C.c_void_p(y.ctypes.data)))
        return y

    def charge_fields(self):
        torch = self._torch
        En = torch.empty(self.n, device=self._dev(), dtype=torch.float32)
        psi = torch.empty_like(En)
        self._sync_current()
        L.check(self.lib.fmmbem_charge_fields(self._h, C.c_void_p(En.data_ptr()), C.c_void_p(psi.data_ptr())))
        return En, psi

    def reset_fields(self):
        """Drop the cached charge-FMM fields (the next bibee / solve recomputes E_n and psi)."""
        L.check(self.lib.fmmbem_reset_fields(self._h))

    def bibee(self, variant="cfa", want_sigma=False):
        torch = self._torch
        e = L.Energy()
        sig = torch.empty(self.n, device=self._dev(), dtype=torch.float32) if want_sigma else None
        self._sync_current()
        L.check(self.lib.fmmbem_bibee_energy(self._h, BIBEE[variant],
                                             C.c_void_p(sig.data_ptr()) if sig is not None else None, C.byref(e)))
        out = dict(dG=e.dG_internal, dG_kcal=e.dG_kcal_mol)
        if sig is not None:
            out["sigma"] = sig
        return out

    def solve(self, tol=1e-6, restart=30, max_iters=200, x0=None):
        torch = self._torch
        if x0 is not None:
            x0 = self._check_dev(x0, "x0")
        so = L.SolveOptions(tol, restart, max_iters, C.c_void_p(x0.data_ptr()) if x0 is not None else None)
        sig = torch.empty(self.n, device=self._dev(), dtype=torch.float32)
        hist = np.empty(max_iters + 1, np.float64)
        e = L.Energy()
        self._sync_current()
        code = L.check(self.lib.fmmbem_solve(self._h, C.byref(so), C.c_void_p(sig.data_ptr()),
                                             hist.ctypes.data_as(C.POINTER(C.c_double)), C.byref(e)))
        return dict(sigma=sig, dG=e.dG_internal, dG_kcal=e.dG_kcal_mol, iterations=e.iterations,
                    rel_residual=e.rel_residual, converged=(code == L.OK), history=hist[hist >= 0])

    def reaction_potential(self, sigma):
        sigma = self._vec(sigma)
        phi = np.empty(self.n_charges, np.float64)
        self._sync_current()
        L.check(self.lib.fmmbem_reaction_potential(self._h, C.c_void_p(sigma.data_ptr()), _dp(phi)))
        return phi

    def timing(self):
        t = L.Timing()
        L.check(self.lib.fmmbem_last_timing(self._h, C.byref(t)))
        return {k: getattr(t, k) for k, _ in L.Timing._fields_}

    def tree_info(self):
        t = L.TreeInfo()
        L.check(self.lib.fmmbem_tree_info_get(self._h, C.byref(t)))
        d = {k: getattr(t, k) for k, _ in L.TreeInfo._fields_}
        d["root_origin"] = list(t.root_origin)
        return d
