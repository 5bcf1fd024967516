"""Thin Python binding of the C ABI in include/rm.h (argument marshalling only).

Every step of the sweep runs in librm.so (host setup in C++, the sweep in sm_100a kernels).
There is no CPU fallback: importing this package fails loudly when the library is missing,
and every call checks that its vectors are fp64 CUDA tensors of the layout's length.

    ctx = rm_setup(nx, ny, nz, p, space, alpha, beta, gamma_d, coords=None, decomposition=RM_PAFW,
                   factorization=RM_CHOL, patch_entities=RM_ALL_ENTITIES, potential_shift=1e-3)
    rm_apply(ctx, u, v); rm_residual(ctx, f, u, r); rm_relax(ctx, f, u_in, u_out, omega)
    rm_precondition(ctx, r, z); rm_relax_host(ctx, f_np, u_np, out_np, omega)
    iters, rel = rm_pcg(ctx, f, u, rtol, maxit)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librm.so")

RM_HGRAD, RM_HCURL, RM_HDIV = 0, 1, 2
RM_PAFW, RM_PH, RM_SC_PAFW, RM_SC_PH = 0, 1, 2, 3
RM_CHOL, RM_ICC_SC = 0, 1
RM_ALL_ENTITIES, RM_INTERIOR_ONLY = 0, 1
RM_SETUP_HOST, RM_SETUP_DEVICE = 0, 1
RM_OK, RM_NOT_CONVERGED = 0, 1
RM_NPHASE = 8   # entries of rm_timing_read (include/rm.h)
STATUS = {0: "RM_OK", 1: "RM_NOT_CONVERGED", -1: "RM_EINVAL", -2: "RM_ENOMEM", -3: "RM_ENUMERIC",
          -4: "RM_ECUDA", -5: "RM_ENCCL"}


class RmError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class rm_mesh(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("coords", ctypes.POINTER(ctypes.c_double)), ("z_begin", ctypes.c_int32), ("z_end", ctypes.c_int32)]


class rm_options(ctypes.Structure):
    _fields_ = [("decomposition", ctypes.c_int32), ("factorization", ctypes.c_int32),
                ("patch_entities", ctypes.c_int32), ("potential_shift", ctypes.c_double),
                ("coarse", ctypes.c_int32), ("stream", ctypes.c_void_p), ("nccl_id", ctypes.c_void_p),
                ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("device", ctypes.c_int32),
                ("setup", ctypes.c_int32)]


class rm_partition_info(ctypes.Structure):
    _fields_ = [("z_cell0", ctypes.c_int32), ("nz_local", ctypes.c_int32), ("ghost_lo", ctypes.c_int32),
                ("v_lo", ctypes.c_int32), ("v_hi", ctypes.c_int32), ("own_lo", ctypes.c_int32),
                ("own_hi", ctypes.c_int32), ("fwd_recv_lo", ctypes.c_int32 * 2), ("fwd_send_lo", ctypes.c_int32 * 2),
                ("fwd_recv_hi", ctypes.c_int32 * 2), ("fwd_send_hi", ctypes.c_int32 * 2),
                ("rev_send_lo", ctypes.c_int32 * 2), ("rev_recv_hi", ctypes.c_int32 * 2),
                ("gamma_local", ctypes.c_uint32), ("plane_len", ctypes.c_int64),
                ("dp_own_lo", ctypes.c_int32), ("dp_own_hi", ctypes.c_int32),
                ("dp_fwd_recv_lo", ctypes.c_int32 * 2), ("dp_fwd_send_hi", ctypes.c_int32 * 2),
                ("dp_rev_send_lo", ctypes.c_int32 * 2), ("dp_rev_recv_hi", ctypes.c_int32 * 2)]

    def as_dict(self):
        d = {}
        for name, _ in self._fields_:
            v = getattr(self, name)
            d[name] = tuple(v) if hasattr(v, "__len__") else v
        return d


class rm_info(ctypes.Structure):
    _fields_ = [("n_local", ctypes.c_int64), ("n_free", ctypes.c_int64), ("n_patches", ctypes.c_int64),
                ("n_patches_potential", ctypes.c_int64), ("n_factor_blocks", ctypes.c_int64),
                ("factor_bytes", ctypes.c_int64), ("sweep_bytes", ctypes.c_int64), ("n_colors", ctypes.c_int32),
                ("n_classes", ctypes.c_int32), ("icc_sigma_max", ctypes.c_double), ("setup_seconds", ctypes.c_double),
                ("factor_nnz", ctypes.c_int64), ("factor_nnz_primary", ctypes.c_int64),
                ("factor_unique_bytes", ctypes.c_int64), ("comm_nranks", ctypes.c_int32), ("coarse", ctypes.c_int32),
                ("coarse_ndof", ctypes.c_int64), ("batched_families", ctypes.c_int32),
                ("batch_width", ctypes.c_int32), ("setup_on_device", ctypes.c_int32),
                ("setup_host_family_seconds", ctypes.c_double), ("setup_device_numeric_seconds", ctypes.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python paper_2211_14284_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, D, I32, I64, U32 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    lib.rm_default_options.argtypes = [ctypes.POINTER(rm_options)]
    lib.rm_default_options.restype = None
    lib.rm_setup.argtypes = [ctypes.POINTER(P), ctypes.POINTER(rm_mesh), I32, I32, ctypes.POINTER(D), I64,
                             ctypes.POINTER(D), I64, U32, ctypes.POINTER(rm_options)]
    lib.rm_layout.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64), ctypes.POINTER(I32 * 9)]
    lib.rm_info_get.argtypes = [P, ctypes.POINTER(rm_info)]
    lib.rm_constrained_mask.argtypes = [P, ctypes.POINTER(ctypes.c_uint8)]
    lib.rm_apply.argtypes = [P, P, P]
    lib.rm_residual.argtypes = [P, P, P, P]
    lib.rm_relax.argtypes = [P, P, P, P, D]
    lib.rm_precondition.argtypes = [P, P, P]
    lib.rm_relax_host.argtypes = [P, P, P, P, D]
    lib.rm_relax_begin.argtypes = [P, P, P, P]
    lib.rm_relax_end.argtypes = [P, P, P, P, D]
    lib.rm_partition.argtypes = [ctypes.POINTER(rm_mesh), I32, I32, U32, I32, I32, ctypes.POINTER(rm_partition_info)]
    lib.rm_nccl_unique_id.argtypes = [P]
    lib.rm_nccl_check.argtypes = [I32]
    lib.rm_pcg.argtypes = [P, P, P, D, I32, ctypes.POINTER(I32), ctypes.POINTER(D)]
    lib.rm_timing_enable.argtypes = [P, I32]
    lib.rm_timing_read.argtypes = [P, ctypes.POINTER(D * RM_NPHASE), ctypes.POINTER(I64 * RM_NPHASE)]
    lib.rm_destroy.argtypes = [P]
    lib.rm_destroy.restype = None
    lib.rm_last_error.restype = ctypes.c_char_p
    for f in ("rm_setup", "rm_layout", "rm_info_get", "rm_constrained_mask", "rm_apply", "rm_residual",
              "rm_relax", "rm_precondition", "rm_relax_host", "rm_pcg", "rm_timing_enable", "rm_timing_read",
              "rm_relax_begin", "rm_relax_end", "rm_partition", "rm_nccl_unique_id", "rm_nccl_check"):
        getattr(lib, f).restype = ctypes.c_int
    return lib


_lib = _load()


def _check(st):
    if st not in (RM_OK, RM_NOT_CONVERGED):
        raise RmError(st, _lib.rm_last_error().decode())
    return st


class RmContext:
    """Owns an rm_ctx handle (rm_destroy on close / garbage collection)."""

    def __init__(self, handle, stream):
        self.h = handle
        self.stream = stream
        n = ctypes.c_int64()
        nf = ctypes.c_int64()
        shp = (ctypes.c_int32 * 9)()
        _check(_lib.rm_layout(self.h, ctypes.byref(n), ctypes.byref(nf), ctypes.byref(shp)))
        self.n_local = n.value
        self.n_free = nf.value
        self.shapes = [tuple(shp[3 * m:3 * m + 3]) for m in range(3) if shp[3 * m] > 0]

    def close(self):
        if self.h:
            _lib.rm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = rm_info()
        _check(_lib.rm_info_get(self.h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in rm_info._fields_}

    def constrained_mask(self) -> np.ndarray:
        m = np.zeros(self.n_local, dtype=np.uint8)
        _check(_lib.rm_constrained_mask(self.h, m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return m.astype(bool)

    def _vec(self, t, name):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64:
            raise TypeError(f"{name}: expected a float64 CUDA tensor")
        if not t.is_contiguous() or t.numel() != self.n_local:
            raise ValueError(f"{name}: expected a contiguous tensor of {self.n_local} elements")
        return ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    if stream is None:
        import torch
        if not torch.cuda.is_available():
            return 0      # rm_setup will report the missing device as RM_ECUDA
        return torch.cuda.current_stream().cuda_stream
    return int(stream)


def rm_partition(nx, ny, nz, p, space, gamma_d, rank, nranks, z_begin, z_end) -> dict:
    """Z-slab partition of rank `rank` owning cell layers [z_begin, z_end) (include/rm.h):
    local mesh, owned planes / patches, halo plane ranges.  Host arithmetic only."""
    mesh = rm_mesh(nx, ny, nz, None, z_begin, z_end)
    info = rm_partition_info()
    _check(_lib.rm_partition(ctypes.byref(mesh), p, space, gamma_d, rank, nranks, ctypes.byref(info)))
    return info.as_dict()


def rm_nccl_check(device=0):
    """Diagnostic of the NCCL transport on one device (include/rm.h)."""
    _check(_lib.rm_nccl_check(int(device)))


def rm_nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId (rank 0 creates it; broadcast it with torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.rm_nccl_unique_id(buf))
    return buf.raw


def rm_setup(nx, ny, nz, p, space, alpha, beta, gamma_d, coords=None, decomposition=RM_PAFW,
             factorization=RM_CHOL, patch_entities=RM_ALL_ENTITIES, potential_shift=1e-3, stream=None,
             device=0, rank=0, nranks=1, z_begin=0, z_end=None, nccl_id=None, coarse=0,
             setup=None) -> RmContext:
    """coords / alpha / beta describe the GLOBAL mesh; with nranks > 1 the context holds the local
    problem of the cell layers [z_begin, z_end) (rm_partition) and its vectors are local.
    setup: RM_SETUP_DEVICE (default: numeric setup on the GPU) or RM_SETUP_HOST."""
    alpha = np.ascontiguousarray(np.atleast_1d(np.asarray(alpha, dtype=np.float64)).ravel())
    beta = np.ascontiguousarray(np.atleast_1d(np.asarray(beta, dtype=np.float64)).ravel())
    mesh = rm_mesh(nx, ny, nz, None, z_begin, nz if z_end is None else z_end)
    keep = None
    if coords is not None:
        keep = np.ascontiguousarray(np.asarray(coords, dtype=np.float64))
        if keep.size != (nx + 1) * (ny + 1) * (nz + 1) * 3:
            raise ValueError("coords must have (nz+1)(ny+1)(nx+1)*3 entries")
        mesh.coords = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    opt = rm_options()
    _lib.rm_default_options(ctypes.byref(opt))
    opt.decomposition = decomposition
    opt.factorization = factorization
    opt.patch_entities = patch_entities
    opt.potential_shift = potential_shift
    opt.coarse = int(coarse)
    if setup is not None:
        opt.setup = int(setup)
    sp = _stream_ptr(stream)
    opt.stream = ctypes.c_void_p(sp)
    opt.device = device
    opt.rank = rank
    opt.nranks = nranks
    idbuf = None
    if nccl_id is not None:
        if len(nccl_id) != 128:
            raise ValueError("nccl_id must be 128 bytes")
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        opt.nccl_id = ctypes.cast(idbuf, ctypes.c_void_p)
    h = ctypes.c_void_p()
    _check(_lib.rm_setup(ctypes.byref(h), ctypes.byref(mesh), p, space,
                         alpha.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), alpha.size,
                         beta.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), beta.size, gamma_d, ctypes.byref(opt)))
    return RmContext(h, sp)


def rm_apply(ctx: RmContext, u, v):
    _check(_lib.rm_apply(ctx.h, ctx._vec(u, "u"), ctx._vec(v, "v")))


def rm_residual(ctx: RmContext, f, u, r):
    _check(_lib.rm_residual(ctx.h, ctx._vec(f, "f"), ctx._vec(u, "u"), ctx._vec(r, "r")))


def rm_relax(ctx: RmContext, f, u_in, u_out, omega=1.0):
    _check(_lib.rm_relax(ctx.h, ctx._vec(f, "f"), ctx._vec(u_in, "u_in"), ctx._vec(u_out, "u_out"), float(omega)))


def rm_relax_begin(ctx: RmContext, f, u_in, c):
    """Multi-rank stage 1 (halos of f, u_in filled by the caller): c = local patch correction."""
    _check(_lib.rm_relax_begin(ctx.h, ctx._vec(f, "f"), ctx._vec(u_in, "u_in"), ctx._vec(c, "c")))


def rm_relax_end(ctx: RmContext, u_in, c, u_out, omega=1.0):
    """Multi-rank stage 2 (c reverse-added by the caller): u_out = u_in + omega c."""
    _check(_lib.rm_relax_end(ctx.h, ctx._vec(u_in, "u_in"), ctx._vec(c, "c"), ctx._vec(u_out, "u_out"), float(omega)))


def rm_precondition(ctx: RmContext, r, z):
    _check(_lib.rm_precondition(ctx.h, ctx._vec(r, "r"), ctx._vec(z, "z")))


def rm_relax_host(ctx: RmContext, f, u_in, u_out, omega=1.0):
    """Host (numpy or pinned CPU torch) buffers; copies happen inside the call."""
    def ptr(a, name, write=False):
        if isinstance(a, np.ndarray):
            if a.dtype != np.float64 or not a.flags.c_contiguous or a.size != ctx.n_local:
                raise ValueError(f"{name}: expected contiguous float64 array of {ctx.n_local}")
            return ctypes.c_void_p(a.ctypes.data)
        import torch
        if isinstance(a, torch.Tensor) and not a.is_cuda and a.dtype == torch.float64 and a.is_contiguous() \
                and a.numel() == ctx.n_local:
            return ctypes.c_void_p(a.data_ptr())
        raise TypeError(f"{name}: expected a host float64 buffer")
    _check(_lib.rm_relax_host(ctx.h, ptr(f, "f"), ptr(u_in, "u_in"), ptr(u_out, "u_out", True), float(omega)))


def rm_pcg(ctx: RmContext, f, u, rtol=1e-8, maxit=500):
    it = ctypes.c_int32()
    rel = ctypes.c_double()
    st = _check(_lib.rm_pcg(ctx.h, ctx._vec(f, "f"), ctx._vec(u, "u"), float(rtol), int(maxit),
                            ctypes.byref(it), ctypes.byref(rel)))
    return it.value, rel.value, st == RM_OK


def rm_timing_enable(ctx: RmContext, on=True):
    _check(_lib.rm_timing_enable(ctx.h, 1 if on else 0))


def rm_timing_read(ctx: RmContext):
    """-> (ms[RM_NPHASE], launches[RM_NPHASE]) accumulated per entry (include/rm.h): residual,
    primary patch stage, potential stage, other, patch kernel alone, apply kernel alone."""
    ms = (ctypes.c_double * RM_NPHASE)()
    nl = (ctypes.c_int64 * RM_NPHASE)()
    _check(_lib.rm_timing_read(ctx.h, ctypes.byref(ms), ctypes.byref(nl)))
    return list(ms), list(nl)


def exported_symbols():
    """Function names declared in include/rm.h (for the symbol-export test)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "rm.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"^\s*(?:rm_status|void|const char \*)\s*(rm_\w+)\s*\(", src, re.M)))
