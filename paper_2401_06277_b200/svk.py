"""Thin ctypes binding of libsvk (include/svk.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels of ``libsvk.so``.  PyTorch supplies device memory (float64 CUDA
tensors in the pitched layout of ``svk_level_info``) and the current stream.
There is no CPU fallback: if ``libsvk.so`` is missing or no CUDA device is
present, construction fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SVK_LIBRARY") or os.path.join(_PKG, "libsvk.so")  # SVK_LIBRARY: dev builds

SVK_OK, SVK_NOT_CONVERGED = 0, 1
PROBLEMS = {"zero": 0, "mms_paper": 1, "mms_inspace": 2, "cavity": 3}
WEIGHTING = {"mult": 0, "scalar": 1}
COARSE = {"exact": 0, "sweeps3": 1}
SWEEP = {"fused": 0, "unfused": 1, "simple": 2}
ORTH = {"adaptive": 0, "cgs2": 1}
TRANSPORT = {"none": 0, "nccl": 1, "emulated": 2}
RELAX = {"vanka": 0, "bs": 1, "su": 2}
PRECOND = {"mg": 0, "bt": 1}
# comparator defaults: (t, omega_r, jacobi_omega, jacobi_sweeps)
RELAX_DEFAULTS = {"bs": (1.0, 1.0, 0.8, 3), "su": (1.0, 1.0, 0.4, 1)}


class SvkError(RuntimeError):
    pass


class Config(C.Structure):
    _fields_ = [("n_elem", C.c_int32), ("n_coarse", C.c_int32), ("nu", C.c_double), ("omega_v", C.c_double),
                ("weighting", C.c_int32), ("nu_pre", C.c_int32), ("nu_post", C.c_int32), ("coarse", C.c_int32),
                ("sweep_impl", C.c_int32), ("device", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("transport", C.c_int32), ("agglom_rows", C.c_int32), ("emul_group", C.c_int32),
                ("orth", C.c_int32), ("relax", C.c_int32), ("jacobi_sweeps", C.c_int32), ("nccl_id", C.c_uint8 * 128),
                ("relax_t", C.c_double), ("relax_omega", C.c_double), ("jacobi_omega", C.c_double),
                ("precond", C.c_int32), ("bt_cycles", C.c_int32), ("bt_nu", C.c_int32), ("validate", C.c_int32),
                ("bt_omega_u", C.c_double), ("bt_omega_p", C.c_double), ("krylov_store_z", C.c_int32),
                ("reserved0", C.c_int32), ("alloc_fn", C.c_void_p), ("free_fn", C.c_void_p),
                ("alloc_user", C.c_void_p)]

# svk_config.alloc_fn / free_fn
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p)


def torch_allocator_callbacks():
    """(alloc_fn, free_fn) routing svk workspaces through torch's CUDA caching
    allocator (torch.cuda.caching_allocator_alloc / _delete, on the device's
    current stream); keep the returned objects alive as long as the context."""
    import torch

    def _alloc(nbytes, device, user):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), device)
        except Exception:   # NULL -> SVK_ERR_CUDA from the calling entry point
            return None

    def _free(ptr, nbytes, device, user):
        torch.cuda.caching_allocator_delete(ptr)

    return ALLOC_FN(_alloc), FREE_FN(_free)


class LevelInfo(C.Structure):
    _fields_ = [("N", C.c_int32), ("lat", C.c_int32), ("vec_len", C.c_int64), ("off_ux", C.c_int64),
                ("off_uy", C.c_int64), ("off_p", C.c_int64), ("pitch_u", C.c_int64), ("pitch_p", C.c_int64),
                ("n_dof", C.c_int64), ("n_patch", C.c_int64), ("row0", C.c_int32), ("row1", C.c_int32),
                ("distributed", C.c_int32), ("halo_rows", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32), ("n_reorth", C.c_int32),
                ("rel_residual", C.c_double), ("t_total_s", C.c_double), ("t_vcycle_s", C.c_double),
                ("t_orth_s", C.c_double), ("t_setup_s", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


_lib = None

# every symbol declared in include/svk.h (tests check the export table against this)
EXPORTS = {
    "svk_config_default": (C.c_int, [C.POINTER(Config), C.c_int32]),
    "svk_create": (C.c_int, [C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "svk_destroy": (C.c_int, [C.c_void_p]),
    "svk_num_levels": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "svk_level_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(LevelInfo)]),
    "svk_set_problem": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_residual": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_matvec": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_vanka_sweep": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "svk_relax_sweep": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_precond_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_restrict": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_prolong_add": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_residual_restrict": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_coarse_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_vcycle": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_fgmres": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int32, C.c_void_p,
                             C.POINTER(Report), C.c_void_p]),
    "svk_solve_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                                 C.POINTER(Report), C.c_void_p]),
    "svk_solve_host_batch": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                       C.POINTER(C.c_void_p), C.c_double, C.c_int32, C.POINTER(Report), C.c_void_p]),
    "svk_patch_inverse": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_int32)]),
    "svk_validate_patches": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "svk_device_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "svk_launch_count": (C.c_int64, [C.c_void_p]),
    "svk_set_profiling": (C.c_int, [C.c_void_p, C.c_int32]),
    "svk_sweep_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]),
    "svk_partition": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "svk_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "svk_allgather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "svk_status_string": (C.c_char_p, [C.c_int]),
    "svk_last_error": (C.c_char_p, [C.c_void_p]),
}


def load_library(path: str = LIB_PATH):
    """Load libsvk.so (no compute).  Raises ImportError if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libsvk.so not built (%s); run `python -m paper_2401_06277_b200.build`" % path)
    lib = C.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def partition(n_elem: int, n_coarse: int, nranks: int, rank: int, agglom_rows: int, N: int):
    """Node-row slab (r0, r1, distributed) of `rank` on the level with N elements (svk_partition)."""
    lib = load_library()
    r0, r1, d = C.c_int32(), C.c_int32(), C.c_int32()
    st = lib.svk_partition(n_elem, n_coarse, nranks, rank, agglom_rows, N, C.byref(r0), C.byref(r1), C.byref(d))
    if st != SVK_OK:
        raise SvkError("svk_partition: %s" % lib.svk_status_string(st).decode())
    return r0.value, r1.value, bool(d.value)


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes); call on rank 0 only."""
    lib = load_library()
    buf = (C.c_uint8 * 128)()
    st = lib.svk_nccl_unique_id(buf)
    if st != SVK_OK:
        raise SvkError("svk_nccl_unique_id: %s" % lib.svk_status_string(st).decode())
    return bytes(buf)


def nccl_id_broadcast(group=None, make_id=None) -> bytes:
    """Rank 0 creates the NCCL id and torch.distributed broadcasts it to every rank
    (any backend; the bootstrap is host-side plumbing, the solver's traffic is NCCL)."""
    import torch.distributed as dist
    make_id = nccl_unique_id if make_id is None else make_id
    obj = [make_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not isinstance(obj[0], (bytes, bytearray)) or len(obj[0]) != 128:
        raise SvkError("bad NCCL id broadcast")
    return bytes(obj[0])


class Solver:
    """One libsvk context: hierarchy N, N/2, ..., n_coarse on one CUDA device."""

    def __init__(self, n_elem: int, n_coarse: int = 4, nu: float = 1.0, omega: float = 0.8,
                 weighting: str = "mult", nu_pre: int = 1, nu_post: int = 1, coarse: str = "exact",
                 sweep: str = "fused", device: int = 0, rank: int = 0, nranks: int = 1,
                 transport: str = "none", agglom_rows: int = 64, emul_group: int = 0, nccl_id: bytes | None = None,
                 orth: str = "adaptive", relax: str = "vanka", relax_t: float | None = None,
                 relax_omega: float | None = None, jacobi_omega: float | None = None,
                 jacobi_sweeps: int | None = None, precond: str = "mg", bt_cycles: int = 3, bt_nu: int = 3,
                 bt_omega_u: float = 1.0, bt_omega_p: float = 0.6, validate: bool = False,
                 low_memory: bool = False, allocator: str = "cuda"):
        """nranks > 1: row-slab multi-GPU mode (include/svk.h, MULTI-GPU).  transport "nccl" needs
        `nccl_id` (128 bytes from `nccl_unique_id()` on rank 0, see `nccl_id_broadcast`);
        "emulated" runs nranks logical ranks of one process on one device (one thread each).
        relax: "vanka" (the hot path), "bs" (Braess-Sarazin) or "su" (Schur-Uzawa) comparators;
        unset comparator parameters take RELAX_DEFAULTS[relax].
        allocator: "cuda" (cudaMalloc), "torch" (vector workspaces from torch's
        caching allocator, svk_config.alloc_fn) or an (ALLOC_FN, FREE_FN) pair of
        the caller's ctypes callbacks."""
        import torch
        if not torch.cuda.is_available():
            raise SvkError("libsvk needs a CUDA device (B200, sm_100a); none is visible")
        self.torch = torch
        self.lib = load_library()
        cfg = Config()
        self.lib.svk_config_default(C.byref(cfg), n_elem)
        cfg.n_coarse, cfg.nu, cfg.omega_v = n_coarse, nu, omega
        cfg.weighting, cfg.nu_pre, cfg.nu_post = WEIGHTING[weighting], nu_pre, nu_post
        cfg.coarse, cfg.sweep_impl, cfg.device = COARSE[coarse], SWEEP[sweep], device
        cfg.rank, cfg.nranks, cfg.transport = rank, nranks, TRANSPORT[transport]
        cfg.agglom_rows, cfg.emul_group, cfg.orth = agglom_rows, emul_group, ORTH[orth]
        cfg.relax = RELAX[relax]
        cfg.precond, cfg.bt_cycles, cfg.bt_nu = PRECOND[precond], bt_cycles, bt_nu
        cfg.bt_omega_u, cfg.bt_omega_p = bt_omega_u, bt_omega_p
        cfg.validate = 1 if validate else 0
        cfg.krylov_store_z = 0 if low_memory else 1
        if relax != "vanka":
            d = RELAX_DEFAULTS[relax]
            cfg.relax_t = d[0] if relax_t is None else relax_t
            cfg.relax_omega = d[1] if relax_omega is None else relax_omega
            cfg.jacobi_omega = d[2] if jacobi_omega is None else jacobi_omega
            cfg.jacobi_sweeps = d[3] if jacobi_sweeps is None else jacobi_sweeps
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise SvkError("nccl_id must be 128 bytes")
            C.memmove(cfg.nccl_id, bytes(nccl_id), 128)
        self._alloc_cbs = None
        if allocator == "torch":
            self._alloc_cbs = torch_allocator_callbacks()
            cfg.alloc_fn = C.cast(self._alloc_cbs[0], C.c_void_p)
            cfg.free_fn = C.cast(self._alloc_cbs[1], C.c_void_p)
        elif isinstance(allocator, tuple) and len(allocator) == 2:  # (ALLOC_FN, FREE_FN) of the caller
            self._alloc_cbs = allocator
            cfg.alloc_fn = C.cast(self._alloc_cbs[0], C.c_void_p)
            cfg.free_fn = C.cast(self._alloc_cbs[1], C.c_void_p)
        elif allocator != "cuda":
            raise SvkError("allocator must be 'cuda', 'torch' or an (ALLOC_FN, FREE_FN) pair")
        self.rank, self.nranks = rank, nranks
        self.cfg = cfg
        self.device = torch.device("cuda", device)
        torch.cuda.set_device(self.device)
        h = C.c_void_p()
        st = self.lib.svk_create(C.byref(cfg), C.byref(h))
        if st != SVK_OK:
            raise SvkError("svk_create failed: %s (%d)" % (self.lib.svk_status_string(st).decode(), st))
        self._h = h
        nl = C.c_int32()
        self.lib.svk_num_levels(self._h, C.byref(nl))
        self.levels = nl.value
        self.info = []
        for l in range(self.levels):
            li = LevelInfo()
            self._chk(self.lib.svk_level_info(self._h, l, C.byref(li)))
            self.info.append(li)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.svk_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ helpers
    def _chk(self, st):
        if st < 0:
            msg = self.lib.svk_last_error(self._h)
            raise SvkError("%s: %s" % (self.lib.svk_status_string(st).decode(), msg.decode() if msg else ""))
        return st

    def _stream(self):
        """This context's device's current torch stream (the library itself runs
        every call on cfg.device and restores the caller's device)."""
        return C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)

    @property
    def fine(self) -> int:
        return self.levels - 1

    def _vec(self, t, level, name):
        li = self.info[level]
        if (t.dtype != self.torch.float64 or not t.is_cuda or t.device != self.device or not t.is_contiguous()
                or t.numel() != li.vec_len):
            raise SvkError("%s: expected a contiguous float64 tensor of %d elements on %s"
                           % (name, li.vec_len, self.device))
        return C.c_void_p(t.data_ptr())

    def new_vector(self, level: int | None = None):
        level = self.fine if level is None else level
        return self.torch.zeros(self.info[level].vec_len, dtype=self.torch.float64, device=self.device)

    def planes(self, v, level: int | None = None):
        """(ux, uy, p) views of a pitched vector, shapes (2N+1, 2N+1), (2N+1, 2N+1), (N+1, N+1)."""
        level = self.fine if level is None else level
        li = self.info[level]
        n = li.lat
        ux = v[li.off_ux:li.off_ux + n * li.pitch_u].view(n, li.pitch_u)[:, :n]
        uy = v[li.off_uy:li.off_uy + n * li.pitch_u].view(n, li.pitch_u)[:, :n]
        p = v[li.off_p:li.off_p + (li.N + 1) * li.pitch_p].view(li.N + 1, li.pitch_p)[:, :li.N + 1]
        return ux, uy, p

    def to_compact(self, v, level: int | None = None):
        ux, uy, p = self.planes(v, level)
        return self.torch.cat([ux.reshape(-1), uy.reshape(-1), p.reshape(-1)])

    def from_compact(self, c, level: int | None = None):
        level = self.fine if level is None else level
        t = self.torch
        c = t.as_tensor(np.asarray(c) if not isinstance(c, t.Tensor) else c, dtype=t.float64).to(self.device)
        li = self.info[level]
        nv = li.lat * li.lat
        v = self.new_vector(level)
        ux, uy, p = self.planes(v, level)
        ux.copy_(c[:nv].view(li.lat, li.lat))
        uy.copy_(c[nv:2 * nv].view(li.lat, li.lat))
        p.copy_(c[2 * nv:].view(li.N + 1, li.N + 1))
        return v

    # ------------------------------------------------------------------ API
    def set_problem(self, kind: str = "mms_paper", level: int | None = None):
        level = self.fine if level is None else level
        b, x0 = self.new_vector(level), self.new_vector(level)
        self._chk(self.lib.svk_set_problem(self._h, level, PROBLEMS[kind], C.c_void_p(b.data_ptr()),
                                           C.c_void_p(x0.data_ptr()), self._stream()))
        return b, x0

    def residual(self, level, x, b, out=None):
        out = self.new_vector(level) if out is None else out
        self._chk(self.lib.svk_residual(self._h, level, self._vec(x, level, "x"), self._vec(b, level, "b"),
                                        self._vec(out, level, "r"), self._stream()))
        return out

    def matvec(self, level, x, out=None):
        out = self.new_vector(level) if out is None else out
        self._chk(self.lib.svk_matvec(self._h, level, self._vec(x, level, "x"), self._vec(out, level, "y"),
                                      self._stream()))
        return out

    def sweep(self, level, x, b, nsweeps: int = 1, out=None):
        out = self.new_vector(level) if out is None else out
        self._chk(self.lib.svk_vanka_sweep(self._h, level, self._vec(x, level, "x_in"), self._vec(b, level, "b"),
                                           self._vec(out, level, "x_out"), nsweeps, self._stream()))
        return out

    def relax_sweep(self, level, x, b, out=None):
        """One sweep of the configured relaxation (svk_relax_sweep)."""
        out = self.new_vector(level) if out is None else out
        self._chk(self.lib.svk_relax_sweep(self._h, level, self._vec(x, level, "x_in"), self._vec(b, level, "b"),
                                           self._vec(out, level, "x_out"), self._stream()))
        return out

    def precond_apply(self, b, out=None):
        """z = M b with the configured FGMRES preconditioner (svk_precond_apply)."""
        out = self.new_vector() if out is None else out
        self._chk(self.lib.svk_precond_apply(self._h, self._vec(b, self.fine, "b"), self._vec(out, self.fine, "z"),
                                             self._stream()))
        return out

    def restrict(self, level, rf, out=None):
        out = self.new_vector(level - 1) if out is None else out
        self._chk(self.lib.svk_restrict(self._h, level, self._vec(rf, level, "r_fine"),
                                        self._vec(out, level - 1, "r_coarse"), self._stream()))
        return out

    def residual_restrict(self, level, x, b, out=None):
        """r_c = P^T (b - A x) on level-1 in one pass (svk_residual_restrict)."""
        out = self.new_vector(level - 1) if out is None else out
        self._chk(self.lib.svk_residual_restrict(self._h, level, self._vec(x, level, "x"), self._vec(b, level, "b"),
                                                 self._vec(out, level - 1, "r_coarse"), self._stream()))
        return out

    def prolong_add(self, level, ec, xf):
        self._chk(self.lib.svk_prolong_add(self._h, level, self._vec(ec, level - 1, "e_coarse"),
                                           self._vec(xf, level, "x_fine"), self._stream()))
        return xf

    def coarse_solve(self, b, out=None):
        out = self.new_vector(0) if out is None else out
        self._chk(self.lib.svk_coarse_solve(self._h, self._vec(b, 0, "b"), self._vec(out, 0, "x"),
                                            self._stream()))
        return out

    def vcycle(self, b, x=None):
        x = self.new_vector() if x is None else x
        self._chk(self.lib.svk_vcycle(self._h, self._vec(b, self.fine, "b"), self._vec(x, self.fine, "x"),
                                      self._stream()))
        return x

    def fgmres(self, b, x, rtol: float = 1e-10, maxit: int = 200):
        """In-place on x.  Returns (report dict, history np.ndarray)."""
        hist = np.zeros(maxit + 1)
        rep = Report()
        st = self._chk(self.lib.svk_fgmres(self._h, self._vec(b, self.fine, "b"), self._vec(x, self.fine, "x"),
                                           rtol, maxit, hist.ctypes.data_as(C.c_void_p), C.byref(rep),
                                           self._stream()))
        d = rep.as_dict()
        d["status"] = st
        return d, hist[: rep.iterations + 1].copy()

    def _host(self, a, name, writable=False):
        li = self.info[self.fine]
        n = 2 * li.lat * li.lat + (li.N + 1) ** 2
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
                and a.ndim == 1 and a.size == n and (a.flags["WRITEABLE"] or not writable)):
            raise SvkError("%s: expected a C-contiguous%s float64 host array of %d elements"
                           % (name, " writable" if writable else "", n))
        return a

    def solve_host_batch(self, b_hosts, x0_hosts, rtol: float = 1e-10, maxit: int = 200, x_hosts=None):
        """Pipelined end-to-end solves of several problems from host arrays
        (svk_solve_host_batch): the copies of problems k+1 / k-1 overlap the solve of
        problem k.  Returns (list of x arrays, list of report dicts, status)."""
        k = len(b_hosts)
        if k < 1 or len(x0_hosts) != k or (x_hosts is not None and len(x_hosts) != k):
            raise SvkError("b_hosts / x0_hosts / x_hosts: equal non-zero lengths expected")
        bs = [self._host(a, "b_hosts[%d]" % i) for i, a in enumerate(b_hosts)]
        x0s = [self._host(a, "x0_hosts[%d]" % i) for i, a in enumerate(x0_hosts)]
        xs = ([np.empty_like(bs[0]) for _ in range(k)] if x_hosts is None
              else [self._host(a, "x_hosts[%d]" % i, writable=True) for i, a in enumerate(x_hosts)])
        for i, x in enumerate(xs):
            if np.shares_memory(x, bs[i]) or np.shares_memory(x, x0s[i]):
                raise SvkError("x_hosts[%d] aliases an input" % i)
        ptrs = lambda arrs: (C.c_void_p * k)(*[a.ctypes.data for a in arrs])
        reps = (Report * k)()
        st = self._chk(self.lib.svk_solve_host_batch(self._h, k, ptrs(bs), ptrs(x0s), ptrs(xs), rtol, maxit,
                                                     reps, self._stream()))
        out = []
        for r in reps:
            d = r.as_dict()
            out.append(d)
        return xs, out, st

    def solve_host(self, b_host: np.ndarray, x0_host: np.ndarray, rtol: float = 1e-10, maxit: int = 200,
                   x_host: np.ndarray | None = None):
        """End-to-end solve from host arrays in the compact layout (svk_solve_host)."""
        host = self._host
        b_host, x0_host = host(b_host, "b_host"), host(x0_host, "x0_host")
        x_host = np.empty_like(b_host) if x_host is None else host(x_host, "x_host", writable=True)
        if np.shares_memory(x_host, b_host) or np.shares_memory(x_host, x0_host):
            raise SvkError("x_host aliases an input")
        rep = Report()
        st = self._chk(self.lib.svk_solve_host(self._h, b_host.ctypes.data_as(C.c_void_p),
                                               x0_host.ctypes.data_as(C.c_void_p), x_host.ctypes.data_as(C.c_void_p),
                                               rtol, maxit, C.byref(rep), self._stream()))
        d = rep.as_dict()
        d["status"] = st
        return x_host, d

    def allgather(self, v):
        """Distributed mode: complete every rank's copy of a finest-level vector (in place)."""
        self._chk(self.lib.svk_allgather(self._h, self._vec(v, self.fine, "v"), self._stream()))
        return v

    def owned_rows(self, level: int | None = None):
        """(row0, row1, distributed) node-row slab of this rank on a level."""
        li = self.info[self.fine if level is None else level]
        return li.row0, li.row1, bool(li.distributed)

    def patch_inverse(self, level: int, cat_x: int, cat_y: int) -> np.ndarray:
        out = np.zeros(51 * 51)
        n = C.c_int32()
        self._chk(self.lib.svk_patch_inverse(self._h, level, cat_x, cat_y, out.ctypes.data_as(C.c_void_p),
                                             C.byref(n)))
        return out[: n.value * n.value].reshape(n.value, n.value).copy()

    def validate_patches(self, level: int | None = None):
        """Validation mode on one level (svk_validate_patches): (max relative deviation,
        patch count); raises SvkError if a patch differs from its group by more than 1e-12."""
        level = self.fine if level is None else level
        dev, n = C.c_double(), C.c_int64()
        st = self.lib.svk_validate_patches(self._h, level, C.byref(dev), C.byref(n))
        if st < 0:
            msg = self.lib.svk_last_error(self._h)
            raise SvkError("%s: %s" % (self.lib.svk_status_string(st).decode(), msg.decode() if msg else ""))
        return dev.value, n.value

    def set_profiling(self, on: bool = True):
        self._chk(self.lib.svk_set_profiling(self._h, 1 if on else 0))

    def sweep_stats(self):
        """(number of finest-level sweeps, summed device ms) since the last call."""
        n, t = C.c_int64(), C.c_double()
        self._chk(self.lib.svk_sweep_stats(self._h, C.byref(n), C.byref(t)))
        return int(n.value), float(t.value)

    @property
    def device_bytes(self) -> int:
        """Device memory held by the context (svk_device_bytes)."""
        n = C.c_int64()
        self._chk(self.lib.svk_device_bytes(self._h, C.byref(n)))
        return int(n.value)

    @property
    def launch_count(self) -> int:
        return int(self.lib.svk_launch_count(self._h))
