"""latbench-b200: the BSMBench Wilson-Dirac / CG hot path on B200 (sm_100a).

Python mirror of the reference operator API (latbench, C++20:
``proj/include/latbench/{fields,kernels,solver}.hpp``) over the C-ABI in
``include/lbcu.h`` (``liblbcu.so``, built in-tree by ``_build.py``). Names,
argument meaning and error behaviour follow the reference:

==========================  =====================================================
reference (latbench::)      here
==========================  =====================================================
GaugeField / make_gauge     ``GaugeField(ctx, group_rank, rep, bc_time)``
SpinorField / make_spinor   ``SpinorField(ctx, dr, subset=FULL)``
init_spinor_random          ``init_spinor_random`` (host, bit-identical)
randomize_gauge_interior    ``init_gauge_random`` (host, bit-identical)
apply_dirac                 ``apply_dirac(out, gauge, in_, mass)``
apply_h                     ``apply_h(out, gauge, in_, mass)``
sqnorm / mul_add / dot ...  same names
cg_solve(LinearOp)          ``cg_solve(op, rhs, settings)`` (op: Python callable)
consistency_check           ``consistency_check(gauge, rhs, mass, settings)``
(none) Dphi_eo / Mhat / eo  ``dphi_eo``, ``dphi_oe``, ``mhat``, ``cg_solve_eo``
==========================  =====================================================

There is no CPU fallback: importing this package without the built library,
or calling a device operator without a CUDA device, raises.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LBCU_LIBRARY") or os.path.join(_PKG, "liblbcu.so")

FUNDAMENTAL, ADJOINT, SYMMETRIC, ANTISYMMETRIC = 0, 1, 2, 3
SQNORM, MULADD, DIRAC = 0, 1, 2
FULL, EVEN, ODD = 0, 1, 2
PERIODIC, ANTIPERIODIC_T = 0, 1
LINKS_UNIT, LINKS_HAAR, LINKS_NEAR_UNIT = 0, 1, 2

_REP_NAMES = {"fundamental": FUNDAMENTAL, "adjoint": ADJOINT, "symmetric": SYMMETRIC,
              "antisymmetric": ANTISYMMETRIC}


# ---------------------------------------------------------------- errors
# proj/include/latbench/errors.hpp:9-63
class Error(RuntimeError):
    code = -1


class ContractViolation(Error):
    code = 1


class ConfigError(Error):
    code = 2


class DecompositionError(ConfigError):
    pass


class TransportError(Error):
    code = 3


class NonConvergence(Error):
    code = 4

    def __init__(self, msg, iterations=0, best_residual=float("nan")):
        super().__init__(msg)
        self.iterations = iterations
        self.best_residual = best_residual


class CudaError(Error):
    code = 5


_ERRS = {1: ContractViolation, 2: ConfigError, 3: TransportError, 4: NonConvergence, 5: CudaError}

# ---------------------------------------------------------------- library
_lib = None

_ip = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)
_vp = C.c_void_p


class CgSettings(C.Structure):
    """latbench::CgSettings (solver.hpp:13-16)."""
    _fields_ = [("tolerance", C.c_double), ("max_iterations", C.c_int)]

    def __init__(self, tolerance=1e-7, max_iterations=10000):
        super().__init__(float(tolerance), int(max_iterations))


class _Outcome(C.Structure):
    _fields_ = [("iterations", C.c_long), ("rel_residual", C.c_double),
                ("true_rel_residual", C.c_double), ("best_residual", C.c_double),
                ("seconds", C.c_double)]


LINOP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


def lib():
    """The loaded C-ABI library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        sig = {
            "lbcu_last_error": (C.c_char_p, []),
            "lbcu_abi_version": (C.c_int, []),
            "lbcu_device_count": (C.c_int, []),
            "lbcu_flops_per_site": (C.c_longlong, [C.c_int, C.c_int, C.c_int]),
            "lbcu_rep_dim": (C.c_int, [C.c_int, C.c_int, _ip, _ip]),
            "lbcu_check_geometry": (C.c_int, [_ip, _ip, C.c_int, C.c_int, _ip]),
            "lbcu_host_spinor_random": (C.c_int, [_ip, _ip, C.c_int, C.c_int, C.c_uint64, C.c_uint64, _dp]),
            "lbcu_host_gauge_random": (C.c_int, [_ip, _ip, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                                 C.c_double, C.c_int, _dp]),
            "lbcu_plan_faces": (C.c_int, [_ip, _ip, C.c_int, C.c_int, _ip, _ip, C.POINTER(C.c_int32)]),
            "lbcu_world_single": (C.c_int, [C.POINTER(_vp)]),
            "lbcu_world_threads": (C.c_int, [C.c_int, C.POINTER(_vp)]),
            "lbcu_world_threads_direct": (C.c_int, [C.c_int, C.POINTER(_vp)]),
            "lbcu_world_set_direct": (C.c_int, [_vp, C.c_int]),
            "lbcu_world_ipc": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.POINTER(_vp)]),
            "lbcu_nccl_unique_id": (C.c_int, [C.c_char_p]),
            "lbcu_world_nccl": (C.c_int, [C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]),
            "lbcu_world_destroy": (C.c_int, [_vp]),
            "lbcu_ctx_create": (C.c_int, [_vp, C.c_int, C.c_int, _ip, _ip, C.c_int, C.POINTER(_vp)]),
            "lbcu_ctx_destroy": (C.c_int, [_vp]),
            "lbcu_ctx_synchronize": (C.c_int, [_vp]),
            "lbcu_ctx_stream": (_vp, [_vp]),
            "lbcu_ctx_local": (C.c_int, [_vp, _ip]),
            "lbcu_barrier": (C.c_int, [_vp]),
            "lbcu_ctx_kernel_launches": (C.c_longlong, [_vp]),
            "lbcu_ctx_cached_solves": (C.c_longlong, [_vp]),
            "lbcu_event_record": (C.c_int, [_vp, C.c_int]),
            "lbcu_event_elapsed_ms": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(C.c_float)]),
            "lbcu_gauge_create": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]),
            "lbcu_gauge_upload": (C.c_int, [_vp, _dp]),
            "lbcu_gauge_download": (C.c_int, [_vp, _dp]),
            "lbcu_gauge_destroy": (C.c_int, [_vp]),
            "lbcu_gauge_set_compact": (C.c_int, [_vp, C.c_int]),
            "lbcu_gauge_upload_fundamental": (C.c_int, [_vp, _dp]),
            "lbcu_gauge_generate": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_double]),
            "lbcu_spinor_random": (C.c_int, [_vp, C.c_uint64, C.c_uint64]),
            "lbcu_gauge_storage": (C.c_int, [_vp, _ip, _dp]),
            "lbcu_spinor_create": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp)]),
            "lbcu_spinor_upload": (C.c_int, [_vp, _dp]),
            "lbcu_spinor_download": (C.c_int, [_vp, _dp]),
            "lbcu_spinor_subset": (C.c_int, [_vp]),
            "lbcu_spinor_destroy": (C.c_int, [_vp]),
            "lbcu_dphi": (C.c_int, [_vp, _vp, _vp, C.c_double]),
            "lbcu_dphi_host": (C.c_int, [_vp, C.c_double, C.c_int, C.POINTER(_dp), C.POINTER(_dp)]),
            "lbcu_allreduce_sum": (C.c_int, [_vp, _dp, C.c_int]),
            "lbcu_g5dphi": (C.c_int, [_vp, _vp, _vp, C.c_double]),
            "lbcu_dphi_eo": (C.c_int, [_vp, _vp, _vp]),
            "lbcu_dphi_oe": (C.c_int, [_vp, _vp, _vp]),
            "lbcu_mhat": (C.c_int, [_vp, _vp, _vp, C.c_double]),
            "lbcu_mhat_dag_mhat": (C.c_int, [_vp, _vp, _vp, C.c_double]),
            "lbcu_h": (C.c_int, [_vp, _vp, _vp, C.c_double]),
            "lbcu_sqnorm": (C.c_int, [_vp, _dp]),
            "lbcu_mul_add": (C.c_int, [_vp, C.c_double, C.c_double, _vp]),
            "lbcu_dot": (C.c_int, [_vp, _vp, _dp, _dp]),
            "lbcu_axpy": (C.c_int, [_vp, C.c_double, C.c_double, _vp]),
            "lbcu_xpay": (C.c_int, [_vp, C.c_double, C.c_double, _vp]),
            "lbcu_copy": (C.c_int, [_vp, _vp]),
            "lbcu_zero": (C.c_int, [_vp]),
            "lbcu_gamma5": (C.c_int, [_vp]),
            "lbcu_cg_solve": (C.c_int, [_vp, LINOP, _vp, _vp, _vp, C.POINTER(CgSettings),
                                        C.POINTER(_Outcome), _dp]),
            "lbcu_cg_solve_h": (C.c_int, [_vp, C.c_double, _vp, _vp, C.POINTER(CgSettings),
                                          C.POINTER(_Outcome), _dp]),
            "lbcu_cg_solve_eo": (C.c_int, [_vp, C.c_double, _vp, _vp, C.POINTER(CgSettings),
                                           C.POINTER(_Outcome), _dp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, extra=None):
    if rc == 0:
        return
    msg = lib().lbcu_last_error().decode(errors="replace")
    cls = _ERRS.get(rc, Error)
    if cls is ConfigError and ("divisible" in msg or "odd" in msg or "floor" in msg or "even local" in msg):
        cls = DecompositionError
    if cls is NonConvergence and extra is not None:
        raise NonConvergence(msg, extra.iterations, extra.best_residual)
    raise cls(msg)


def _i4(v):
    return (C.c_int * 4)(*[int(x) for x in v])


def _dptr(a: np.ndarray):
    if not a.flags["C_CONTIGUOUS"]:
        raise ContractViolation("array must be C-contiguous")
    return a.ctypes.data_as(_dp)


def device_count() -> int:
    return int(lib().lbcu_device_count())


def rep_dim(rep, n: int) -> int:
    rep = _REP_NAMES.get(rep, rep) if isinstance(rep, str) else rep
    dr, real = C.c_int(), C.c_int()
    _check(lib().lbcu_rep_dim(int(rep), int(n), C.byref(dr), C.byref(real)))
    return dr.value


def rep_is_real(rep) -> bool:
    rep = _REP_NAMES.get(rep, rep) if isinstance(rep, str) else rep
    return int(rep) == ADJOINT


def flops_per_site(kernel: int, dr: int, real_rep: bool) -> int:
    """latbench::flops_per_site (flops.cpp:14-25)."""
    return int(lib().lbcu_flops_per_site(int(kernel), int(dr), int(bool(real_rep))))


def local_extents(global_, grid, rank=0, enforce_floor=False):
    out = (C.c_int * 4)()
    _check(lib().lbcu_check_geometry(_i4(global_), _i4(grid), int(rank), int(enforce_floor), out))
    return tuple(out)


# ------------------------------------------------------- host field generation
def init_spinor_random(global_, dr, seed, field_index, grid=(1, 1, 1, 1), rank=0):
    """init_spinor_random (fields.cpp:22-40): this rank's interior, ref layout."""
    loc = local_extents(global_, grid, rank)
    out = np.empty((int(np.prod(loc)), 4, dr), np.complex128)
    _check(lib().lbcu_host_spinor_random(_i4(global_), _i4(grid), int(rank), int(dr), int(seed),
                                         int(field_index), out.ctypes.data_as(_dp)))
    return out


def init_gauge_random(global_, group_rank, rep, seed, grid=(1, 1, 1, 1), rank=0, links=LINKS_HAAR,
                      eps=0.3, nthreads=0):
    """randomize_gauge_interior (fields.cpp:86-107) / unit / near-unit links."""
    rep = _REP_NAMES.get(rep, rep) if isinstance(rep, str) else rep
    loc = local_extents(global_, grid, rank)
    dr = rep_dim(rep, group_rank)
    dt = np.float64 if rep_is_real(rep) else np.complex128
    out = np.empty((int(np.prod(loc)), 4, dr, dr), dt)
    _check(lib().lbcu_host_gauge_random(_i4(global_), _i4(grid), int(rank), int(group_rank), int(rep),
                                        int(links), int(seed), float(eps), int(nthreads),
                                        out.ctypes.data_as(_dp)))
    return out


def plan_faces(global_, grid, rank, input_parity):
    """Face schedule of the even-odd halo exchange (host logic of the N>1 path)."""
    partner, count = (C.c_int * 8)(), (C.c_int * 8)()
    _check(lib().lbcu_plan_faces(_i4(global_), _i4(grid), int(rank), int(input_parity), partner, count, None))
    sites = np.empty(int(sum(count)), np.int32)
    _check(lib().lbcu_plan_faces(_i4(global_), _i4(grid), int(rank), int(input_parity), partner, count,
                                 sites.ctypes.data_as(C.POINTER(C.c_int32))))
    return list(partner), list(count), sites


# ---------------------------------------------------------------- ownership
def _release(destroy: str, handle):
    """Free one library handle (never raises)."""
    try:
        if _lib is not None and handle:
            getattr(_lib, destroy)(handle)
    except Exception:  # pragma: no cover - interpreter shutdown
        pass


def _release_tree(rec):
    """rec = [destroy, handle, children]: children first (fields before their
    context, contexts before their world), then the handle itself."""
    children = rec[2]
    while children:
        _, child = children.popitem()
        _release_tree(child)
    _release(rec[0], rec[1])


def _finalize(registry, key, rec):
    # a parent that was released first already freed this handle
    if registry is not None and registry.pop(key, None) is None:
        return
    _release_tree(rec)


class _Owned:
    """A library handle freed exactly once: by close(), or by a finalizer when
    the Python object is collected. Every handle is recorded in its parent's
    record (field -> context -> world), and releasing a parent releases its
    remaining children first, so no handle is ever freed through an already
    destroyed context or world — whatever order the garbage collector
    finalises a cycle in."""

    _destroy = ""

    def _own(self, handle, parent=None):
        self._h = handle
        self._rec = [self._destroy, handle, {}]
        self._live = weakref.WeakSet()  # child objects, to clear their _h on close()
        registry = parent._rec[2] if parent is not None else None
        key = id(self._rec)
        if parent is not None:
            registry[key] = self._rec
            parent._live.add(self)
        self._fin = weakref.finalize(self, _finalize, registry, key, self._rec)

    def close(self):
        for ch in list(getattr(self, "_live", ())):
            ch.close()
        fin = getattr(self, "_fin", None)
        if fin is not None:
            fin()
        self._h = None


# ---------------------------------------------------------------- worlds
class World(_Owned):
    """Transport shared by the ranks of one decomposition (WorkerGroup)."""

    _destroy = "lbcu_world_destroy"

    def __init__(self, handle):
        self._own(handle)

    @classmethod
    def single(cls):
        h = _vp()
        _check(lib().lbcu_world_single(C.byref(h)))
        return cls(h)

    @classmethod
    def threads(cls, nranks: int, direct: bool = False):
        """In-process world: one host thread per rank (reference run_workers).
        direct: halos stored by the pack kernel into the peer's arena (the IPC
        world's protocol) instead of copied between barriers."""
        h = _vp()
        fn = lib().lbcu_world_threads_direct if direct else lib().lbcu_world_threads
        _check(fn(int(nranks), C.byref(h)))
        return cls(h)

    @classmethod
    def ipc(cls, nranks: int, rank: int, name: str, uid: Optional[bytes] = None):
        """One process per GPU on one node, direct peer-memory halos (CUDA IPC);
        `name`: a POSIX shared-memory name ("/...") unique to the job; `uid`:
        an NCCL unique id for the CG sums (None: sums through the segment)."""
        h = _vp()
        _check(lib().lbcu_world_ipc(int(nranks), int(rank), name.encode(),
                                    None if uid is None else C.c_char_p(uid), C.byref(h)))
        return cls(h)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().lbcu_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, nranks: int, rank: int, uid: bytes):
        h = _vp()
        _check(lib().lbcu_world_nccl(int(nranks), int(rank), C.c_char_p(uid), C.byref(h)))
        return cls(h)

    def set_direct(self, on: bool):
        """Collective: direct peer-memory halos (True) or message exchange."""
        _check(lib().lbcu_world_set_direct(self._h, 1 if on else 0))


class Context(_Owned):
    """One rank: Geometry + ExchangePlan + Worker + a CUDA stream."""

    _destroy = "lbcu_ctx_destroy"

    def __init__(self, global_, grid=(1, 1, 1, 1), rank=0, device=0, world: Optional[World] = None,
                 enforce_floor=False):
        self.global_ = tuple(int(x) for x in global_)
        self.grid = tuple(int(x) for x in grid)
        self.rank = int(rank)
        self.world = world
        h = _vp()
        _check(lib().lbcu_ctx_create(world._h if world else None, self.rank, int(device),
                                     _i4(self.global_), _i4(self.grid), int(enforce_floor), C.byref(h)))
        self._own(h, world)
        loc = (C.c_int * 4)()
        _check(lib().lbcu_ctx_local(h, loc))
        self.local = tuple(loc)
        self.volume = int(np.prod(self.local))

    def synchronize(self):
        _check(lib().lbcu_ctx_synchronize(self._h))

    def barrier(self):
        _check(lib().lbcu_barrier(self._h))

    @property
    def stream(self) -> int:
        return int(lib().lbcu_ctx_stream(self._h) or 0)

    def kernel_launches(self) -> int:
        return int(lib().lbcu_ctx_kernel_launches(self._h))

    def cached_solves(self) -> int:
        """Instantiated CG solve graphs held by the context."""
        return int(lib().lbcu_ctx_cached_solves(self._h))

    def event_record(self, slot: int):
        _check(lib().lbcu_event_record(self._h, int(slot)))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        _check(lib().lbcu_event_elapsed_ms(self._h, int(a), int(b), C.byref(ms)))
        return float(ms.value)



class GaugeField(_Owned):
    """latbench::GaugeField on the device (fields.hpp:37-57)."""

    _destroy = "lbcu_gauge_destroy"

    def __init__(self, ctx: Context, group_rank: int, rep=FUNDAMENTAL, bc_time=ANTIPERIODIC_T):
        rep = _REP_NAMES.get(rep, rep) if isinstance(rep, str) else rep
        self.ctx, self.group_rank, self.rep, self.bc_time = ctx, int(group_rank), int(rep), int(bc_time)
        self.dr = rep_dim(rep, group_rank)
        self.real_links = rep_is_real(rep)
        h = _vp()
        _check(lib().lbcu_gauge_create(ctx._h, self.group_rank, self.rep, self.bc_time, C.byref(h)))
        self._own(h, ctx)

    @property
    def host_shape(self):
        return (self.ctx.volume, 4, self.dr, self.dr)

    def upload(self, links: np.ndarray):
        dt = np.float64 if self.real_links else np.complex128
        a = np.ascontiguousarray(links, dtype=dt)
        if a.size != int(np.prod(self.host_shape)):
            raise ContractViolation(f"gauge upload expects {self.host_shape}, got {a.shape}")
        _check(lib().lbcu_gauge_upload(self._h, a.ctypes.data_as(_dp)))
        return self

    def upload_fundamental(self, links: np.ndarray):
        """Upload the fundamental SU(N) links ([V, 4, N, N] complex); the
        representation is formed in the kernels (SU(4) antisymmetric)."""
        a = np.ascontiguousarray(links, dtype=np.complex128)
        if a.size != self.ctx.volume * 4 * self.group_rank ** 2:
            raise ContractViolation("fundamental upload expects [V, 4, N, N] complex")
        _check(lib().lbcu_gauge_upload_fundamental(self._h, a.ctypes.data_as(_dp)))
        return self

    def generate(self, seed: int, links=LINKS_HAAR, eps: float = 0.3):
        """init_gauge_random on the device (keyed per global site, any decomposition)."""
        _check(lib().lbcu_gauge_generate(self._h, int(links), int(seed), float(eps)))
        return self

    def set_compact(self, enable: bool):
        """Allow (default) or forbid compact link storage for later uploads."""
        _check(lib().lbcu_gauge_set_compact(self._h, int(bool(enable))))
        return self

    def storage(self):
        """(format name, max reconstruction error at the last upload)."""
        f, e = C.c_int(), C.c_double()
        _check(lib().lbcu_gauge_storage(self._h, C.byref(f), C.byref(e)))
        return {0: "full", 1: "su2", 2: "r12", 3: "as4", 4: "as4r", 5: "r10"}[f.value], e.value

    def download(self) -> np.ndarray:
        dt = np.float64 if self.real_links else np.complex128
        out = np.empty(self.host_shape, dt)
        _check(lib().lbcu_gauge_download(self._h, out.ctypes.data_as(_dp)))
        return out


class SpinorField(_Owned):
    """latbench::SpinorField on the device (fields.hpp:15-24); subset FULL/EVEN/ODD."""

    _destroy = "lbcu_spinor_destroy"

    def __init__(self, ctx: Context, dr: int, subset=FULL):
        self.ctx, self.dr, self.subset = ctx, int(dr), int(subset)
        h = _vp()
        _check(lib().lbcu_spinor_create(ctx._h, self.dr, self.subset, C.byref(h)))
        self._own(h, ctx)

    @property
    def host_shape(self):
        return (self.ctx.volume, 4, self.dr)

    def upload(self, data: np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.complex128)
        if a.size != int(np.prod(self.host_shape)):
            raise ContractViolation(f"spinor upload expects {self.host_shape}, got {a.shape}")
        _check(lib().lbcu_spinor_upload(self._h, a.ctypes.data_as(_dp)))
        return self

    def randomize(self, seed: int, field_index: int):
        """init_spinor_random on the device (fields.cpp:22-40)."""
        _check(lib().lbcu_spinor_random(self._h, int(seed), int(field_index)))
        return self

    def upload_ptr(self, ptr: int):
        """Upload from a host address (pinned buffers in the e2e benchmark)."""
        _check(lib().lbcu_spinor_upload(self._h, C.cast(C.c_void_p(ptr), _dp)))

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.host_shape, np.complex128)
        _check(lib().lbcu_spinor_download(self._h, out.ctypes.data_as(_dp)))
        return out

    def download_ptr(self, ptr: int):
        _check(lib().lbcu_spinor_download(self._h, C.cast(C.c_void_p(ptr), _dp)))


# ---------------------------------------------------------------- operators
def apply_dirac(out: SpinorField, gauge: GaugeField, in_: SpinorField, mass: float):
    """kernels.hpp:19-20 — out = (4+m) in - 1/2 sum_mu hops."""
    _check(lib().lbcu_dphi(out._h, gauge._h, in_._h, float(mass)))


def dphi_host(gauge: GaugeField, mass: float, ins: Sequence[int], outs: Sequence[int]):
    """apply_dirac on host fields (addresses of reference-layout buffers):
    outs[k] = D ins[k], transfers overlapped with the kernels."""
    n = len(ins)
    if len(outs) != n:
        raise ContractViolation("dphi_host: ins and outs differ in length")
    ia = (_dp * n)(*[C.cast(C.c_void_p(int(p)), _dp) for p in ins])
    oa = (_dp * n)(*[C.cast(C.c_void_p(int(p)), _dp) for p in outs])
    _check(lib().lbcu_dphi_host(gauge._h, float(mass), n, ia, oa))


def apply_g5dirac(out, gauge, in_, mass):
    _check(lib().lbcu_g5dphi(out._h, gauge._h, in_._h, float(mass)))


def dphi_eo(out_even, gauge, in_odd):
    _check(lib().lbcu_dphi_eo(out_even._h, gauge._h, in_odd._h))


def dphi_oe(out_odd, gauge, in_even):
    _check(lib().lbcu_dphi_oe(out_odd._h, gauge._h, in_even._h))


def mhat(out_even, gauge, in_even, mass):
    _check(lib().lbcu_mhat(out_even._h, gauge._h, in_even._h, float(mass)))


def mhat_dag_mhat(out_even, gauge, in_even, mass):
    _check(lib().lbcu_mhat_dag_mhat(out_even._h, gauge._h, in_even._h, float(mass)))


def apply_h(out, gauge, in_, mass):
    """solver.hpp:32-33 — out = g5 D g5 D in."""
    _check(lib().lbcu_h(out._h, gauge._h, in_._h, float(mass)))


def sqnorm(f: SpinorField) -> float:
    v = C.c_double()
    _check(lib().lbcu_sqnorm(f._h, C.byref(v)))
    return v.value


def mul_add(psi2, c, psi1):
    c = complex(c)
    _check(lib().lbcu_mul_add(psi2._h, c.real, c.imag, psi1._h))


def dot(a, b) -> complex:
    re, im = C.c_double(), C.c_double()
    _check(lib().lbcu_dot(a._h, b._h, C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


def axpy(y, a, x):
    a = complex(a)
    _check(lib().lbcu_axpy(y._h, a.real, a.imag, x._h))


def xpay(y, a, x):
    a = complex(a)
    _check(lib().lbcu_xpay(y._h, a.real, a.imag, x._h))


def copy_interior(dst, src):
    _check(lib().lbcu_copy(dst._h, src._h))


def zero_interior(f):
    _check(lib().lbcu_zero(f._h))


def apply_gamma5(f):
    _check(lib().lbcu_gamma5(f._h))


# ---------------------------------------------------------------- solver
@dataclass
class CgOutcome:
    """latbench::CgOutcome (solver.hpp:18-25)."""
    solution: SpinorField
    iterations: int = 0
    rel_residual: float = 0.0
    true_rel_residual: float = 0.0
    seconds: float = 0.0
    best_residual: float = 0.0
    residual_history: list = field(default_factory=list)


def _run_cg(fn, args, rhs: SpinorField, settings: CgSettings, x: Optional[SpinorField]):
    x = x or SpinorField(rhs.ctx, rhs.dr, rhs.subset)
    oc = _Outcome()
    hist = np.zeros(max(1, settings.max_iterations), np.float64)
    rc = fn(*args, rhs._h, x._h, C.byref(settings), C.byref(oc), hist.ctypes.data_as(_dp))
    _check(rc, oc)
    return CgOutcome(x, int(oc.iterations), oc.rel_residual, oc.true_rel_residual, oc.seconds,
                     oc.best_residual, hist[: oc.iterations].tolist())


def cg_solve(op: Callable[[SpinorField, SpinorField], None], rhs: SpinorField,
             settings: CgSettings = None, x: Optional[SpinorField] = None) -> CgOutcome:
    """cg_solve(LinearOp, rhs, settings) — solver.cpp:24-82; op(out, in)."""
    settings = settings or CgSettings()
    by_handle = {}

    def trampoline(_user, out_h, in_h):
        try:
            op(by_handle[out_h], by_handle[in_h])
            return 0
        except Error as e:
            return e.code if e.code > 0 else 1
        except Exception:
            return 1

    ctx, dr, sub = rhs.ctx, rhs.dr, rhs.subset
    x = x or SpinorField(ctx, dr, sub)

    # the library hands out its own scratch handles; wrap them on first sight
    class _View(SpinorField):
        def __init__(self, h):
            self.ctx, self.dr, self.subset, self._h = ctx, dr, sub, C.c_void_p(h)

        def close(self):
            pass

    class _Map(dict):
        def __missing__(self, h):
            v = _View(h)
            self[h] = v
            return v

    by_handle = _Map()
    cb = LINOP(trampoline)
    return _run_cg(lib().lbcu_cg_solve, (ctx._h, cb, None), rhs, settings, x)


def cg_solve_h(gauge: GaugeField, mass: float, rhs: SpinorField, settings: CgSettings = None,
               x: Optional[SpinorField] = None) -> CgOutcome:
    """cg_solve(make_h_operator(...)) with fused device kernels (FULL fields)."""
    return _run_cg(lib().lbcu_cg_solve_h, (gauge._h, float(mass)), rhs, settings or CgSettings(), x)


def cg_solve_eo(gauge: GaugeField, mass: float, rhs_even: SpinorField, settings: CgSettings = None,
                x: Optional[SpinorField] = None) -> CgOutcome:
    """Even-odd preconditioned CG on Mhat^dag Mhat (EVEN fields)."""
    return _run_cg(lib().lbcu_cg_solve_eo, (gauge._h, float(mass)), rhs_even, settings or CgSettings(), x)


@dataclass
class ConsistencyResult:
    """latbench::ConsistencyResult (solver.hpp:46-51)."""
    status: str
    iterations: int
    residual: float
    seconds: float


def consistency_check(gauge: GaugeField, rhs: SpinorField, mass: float, settings: CgSettings = None,
                      eo: bool = False) -> ConsistencyResult:
    """solver.cpp:93-108: pass iff the recomputed residual < 2 tol."""
    settings = settings or CgSettings()
    if eo:
        even = SpinorField(rhs.ctx, rhs.dr, EVEN)
        even.upload(rhs.download())
        o = cg_solve_eo(gauge, mass, even, settings)
    else:
        o = cg_solve_h(gauge, mass, rhs, settings)
    status = "passed" if o.true_rel_residual < 2.0 * settings.tolerance else "failed"
    return ConsistencyResult(status, o.iterations, o.true_rel_residual, o.seconds)
