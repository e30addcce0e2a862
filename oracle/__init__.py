"""TEST INFRASTRUCTURE ONLY — the CPU checker for the hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline, never as the thing measured or shipped.

Two libraries, both built by ``oracle/Makefile`` into ``oracle/_ref/``:

* ``liblatbench_ref.so`` — the UNMODIFIED reference (``/root/reference/proj``,
  compiled from its own sources) plus ``ref_shim.cpp``. Functions prefixed
  ``ref_``. ``liblatbench_ref_v4.so`` is the same build for x86-64-v4
  (AVX-512), loaded instead on hosts that support it (``LBCU_REF_ISA=v3``
  forces the AVX2 build).
* ``liboracle.so`` — ``oracle.c``, the plain-C restatement, pinned against the
  reference by ``tests/test_oracle.py``. Functions prefixed ``port_``.

Array convention (both): global lexicographic (t,x,y,z) order, z fastest;
spinors ``complex128[V, 4, dr]``; gauge ``complex128[V, 4, dr, dr]`` or
``float64[V, 4, dr, dr]`` for the adjoint representation.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
REF_SO = os.path.join(REF_DIR, "liblatbench_ref.so")
REF_EXACT_SO = os.path.join(REF_DIR, "liblatbench_ref_exact.so")
REF_V4_SO = os.path.join(REF_DIR, "liblatbench_ref_v4.so")
PORT_SO = os.path.join(REF_DIR, "liboracle.so")

FUNDAMENTAL, ADJOINT, SYMMETRIC, ANTISYMMETRIC = 0, 1, 2, 3
SQNORM, MULADD, DIRAC = 0, 1, 2


def rep_dim(rep: int, n: int) -> int:
    return {FUNDAMENTAL: n, ADJOINT: n * n - 1, ANTISYMMETRIC: n * (n - 1) // 2,
            SYMMETRIC: n * (n + 1) // 2}[rep]


def rep_is_real(rep: int) -> bool:
    return rep == ADJOINT


def build(quiet: bool = True) -> None:
    """Compile the checkers (reference only when /root/reference is present)."""
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1401_3733_b200", "liblbcu.so")):
            targets.append("dropin")
    subprocess.run(["make", "-C", HERE, *targets], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_refs = {}
_port = None
_exact = False

_i4 = C.POINTER(C.c_int)
_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_long)


def _arr4(v):
    return (C.c_int * 4)(*[int(x) for x in v])


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def host_cpu():
    """lscpu-style facts of this host: model name, logical CPUs usable by this
    process, physical cores (unique (package, core) pairs), ISA level of the
    reference build that ref_lib() loads."""
    model, cores, pkg = None, set(), None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                k, _, v = line.partition(":")
                k, v = k.strip(), v.strip()
                if k == "model name" and model is None:
                    model = v
                elif k == "physical id":
                    pkg = v
                elif k == "core id":
                    cores.add((pkg, v))
    except OSError:
        pass
    try:
        logical = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        logical = os.cpu_count() or 1
    return {"model": model, "logical_cpus": logical, "physical_cores": len(cores) or None,
            "reference_isa": ref_isa()}


def ref_isa() -> str:
    v4 = {"avx512f", "avx512bw", "avx512dq", "avx512vl"}
    if os.environ.get("LBCU_REF_ISA") != "v3" and os.path.exists(REF_V4_SO) and v4 <= cpu_flags():
        return "x86-64-v4"
    return "x86-64-v3"


def ref_lib():
    """The compiled reference (the highest ISA build the host supports); the
    FMA-free build inside ``exact_reference()``."""
    path = REF_EXACT_SO if _exact else (REF_V4_SO if ref_isa() == "x86-64-v4" else REF_SO)
    lib = _refs.get(path)
    if lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_flops_per_site.restype = C.c_longlong
        lib.ref_key_hash.restype = C.c_uint64
        _refs[path] = lib
    return lib


class exact_reference:
    """Context manager: route ref_* calls to the -ffp-contract=off build."""

    def __enter__(self):
        global _exact
        self._prev, _exact = _exact, True
        return self

    def __exit__(self, *exc):
        global _exact
        _exact = self._prev
        return False


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            raise RuntimeError(f"{PORT_SO} missing: run `make -C oracle oracle`")
        _port = C.CDLL(PORT_SO)
        _port.oracle_flops_per_site.restype = C.c_longlong
        _port.oracle_sqnorm.restype = C.c_double
        _port.oracle_mix64.restype = C.c_uint64
        _port.oracle_key_hash.restype = C.c_uint64
    return _port


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _chk(rc: int):
    if rc != 0:
        raise OracleError(rc, ref_lib().ref_last_error().decode())


def volume(L) -> int:
    return int(np.prod(L))


def _gauge_dtype(rep):
    return np.float64 if rep_is_real(rep) else np.complex128


# ----------------------------------------------------------------- reference

def ref_spinor_random(L, dr, seed, field_index):
    out = np.empty((volume(L), 4, dr), np.complex128)
    _chk(ref_lib().ref_spinor_random(_arr4(L), dr, C.c_uint64(seed), C.c_uint64(field_index), _ptr(out)))
    return out


def ref_spinor_random_local(L, grid, rank, dr, seed, field_index):
    loc = [L[d] // grid[d] for d in range(4)]
    out = np.empty((volume(loc), 4, dr), np.complex128)
    _chk(ref_lib().ref_spinor_random_local(_arr4(L), _arr4(grid), rank, dr, C.c_uint64(seed),
                                           C.c_uint64(field_index), _ptr(out)))
    return out


def ref_gauge_random(L, n, rep, seed, nthreads=None):
    dr = rep_dim(rep, n)
    out = np.empty((volume(L), 4, dr, dr), _gauge_dtype(rep))
    nthreads = nthreads or os.cpu_count() or 1
    _chk(ref_lib().ref_gauge_random(_arr4(L), n, rep, C.c_uint64(seed), nthreads, _ptr(out)))
    return out


def ref_gauge_unit(L, n, rep):
    dr = rep_dim(rep, n)
    out = np.empty((volume(L), 4, dr, dr), _gauge_dtype(rep))
    _chk(ref_lib().ref_gauge_unit(_arr4(L), n, rep, _ptr(out)))
    return out


def ref_gauge_near_unit(L, n, eps, seed):
    out = np.empty((volume(L), 4, n, n), np.complex128)
    _chk(ref_lib().ref_gauge_near_unit(_arr4(L), n, C.c_double(eps), C.c_uint64(seed), _ptr(out)))
    return out


def _dr_of(gauge):
    return gauge.shape[-1]


def ref_apply_dirac(L, grid, n, rep, bc_time, mass, gauge, inp):
    out = np.empty_like(inp)
    _chk(ref_lib().ref_apply_dirac(_arr4(L), _arr4(grid), n, rep, int(bc_time), C.c_double(mass),
                                   _ptr(gauge), _ptr(np.ascontiguousarray(inp)), _ptr(out)))
    return out


def ref_apply_h(L, grid, n, rep, bc_time, mass, gauge, inp):
    out = np.empty_like(inp)
    _chk(ref_lib().ref_apply_h(_arr4(L), _arr4(grid), n, rep, int(bc_time), C.c_double(mass),
                               _ptr(gauge), _ptr(np.ascontiguousarray(inp)), _ptr(out)))
    return out


def ref_mhat(L, grid, n, rep, bc_time, mass, gauge, inp):
    out = np.empty_like(inp)
    _chk(ref_lib().ref_mhat(_arr4(L), _arr4(grid), n, rep, int(bc_time), C.c_double(mass),
                            _ptr(gauge), _ptr(np.ascontiguousarray(inp)), _ptr(out)))
    return out


def ref_sqnorm(L, grid, field):
    res = C.c_double()
    _chk(ref_lib().ref_sqnorm(_arr4(L), _arr4(grid), field.shape[-1], _ptr(field), C.byref(res)))
    return res.value


def ref_mul_add(L, grid, c, psi2, psi1):
    out = psi2.copy()
    _chk(ref_lib().ref_mul_add(_arr4(L), _arr4(grid), psi2.shape[-1], C.c_double(c.real),
                               C.c_double(c.imag), _ptr(out), _ptr(psi1)))
    return out


def ref_dot(L, grid, a, b):
    re, im = C.c_double(), C.c_double()
    _chk(ref_lib().ref_dot(_arr4(L), _arr4(grid), a.shape[-1], _ptr(a), _ptr(b), C.byref(re), C.byref(im)))
    return complex(re.value, im.value)


def _ref_cg(fn, L, grid, n, rep, bc_time, mass, gauge, rhs, tol, maxit):
    x = np.empty_like(rhs)
    it, rel, trel, secs = C.c_long(), C.c_double(), C.c_double(), C.c_double()
    hist = np.zeros(maxit, np.float64)
    _chk(fn(_arr4(L), _arr4(grid), n, rep, int(bc_time), C.c_double(mass), _ptr(gauge),
            _ptr(np.ascontiguousarray(rhs)), C.c_double(tol), int(maxit), _ptr(x), C.byref(it),
            C.byref(rel), C.byref(trel), C.byref(secs), _ptr(hist)))
    return dict(x=x, iterations=it.value, rel_residual=rel.value, true_rel_residual=trel.value,
                seconds=secs.value, history=hist[: it.value].copy())


def ref_cg_h(L, grid, n, rep, bc_time, mass, gauge, rhs, tol, maxit=10000):
    return _ref_cg(ref_lib().ref_cg_h, L, grid, n, rep, bc_time, mass, gauge, rhs, tol, maxit)


def ref_cg_eo(L, grid, n, rep, bc_time, mass, gauge, rhs, tol, maxit=10000):
    return _ref_cg(ref_lib().ref_cg_eo, L, grid, n, rep, bc_time, mass, gauge, rhs, tol, maxit)


def ref_flops_per_site(kernel, dr, real):
    return int(ref_lib().ref_flops_per_site(kernel, dr, int(real)))


def ref_counted_dirac(L, n, rep):
    v = C.c_longlong()
    _chk(ref_lib().ref_counted_dirac(_arr4(L), n, rep, C.byref(v)))
    return v.value


LINKS_HAAR, LINKS_NEAR_UNIT = 0, 1


def ref_bench_dirac(L, grid, n, rep, mass, seed, napps, links=LINKS_HAAR, bc_time=1, eps=0.3, nwarm=1,
                    nsamples=1):
    """Seconds for `napps` reference apply_dirac on the BASELINE workload
    (inputs generated per worker: Haar or near-unit links, antiperiodic t),
    after `nwarm` untimed applications; a list when nsamples > 1."""
    secs = (C.c_double * max(1, nsamples))()
    _chk(ref_lib().ref_bench_dirac(_arr4(L), _arr4(grid), n, rep, int(links), C.c_double(eps), int(bc_time),
                                   C.c_double(mass), C.c_uint64(seed), int(nwarm), int(napps), int(nsamples),
                                   secs))
    return list(secs) if nsamples > 1 else secs[0]


def ref_cg_probe(L, grid, n, rep, mass, seed, eo, max_iterations, tol=0.0, links=LINKS_HAAR, bc_time=1,
                 eps=0.3):
    """The reference cg_solve on the BASELINE workload (plain on H, or the
    composed eo operator), inputs generated per worker. tol > 0: a solve;
    tol = 0: a bounded sample of exactly max_iterations iterations (plus a
    1-iteration calibration call). Returns dict(seconds, iterations,
    true_rel_residual, seconds_per_iteration), wall times."""
    secs, its, trel, per = C.c_double(), C.c_long(), C.c_double(), C.c_double()
    _chk(ref_lib().ref_cg_probe(_arr4(L), _arr4(grid), n, rep, int(links), C.c_double(eps), int(bc_time),
                                C.c_double(mass), C.c_uint64(seed), int(bool(eo)), C.c_double(tol),
                                int(max_iterations), C.byref(secs), C.byref(its), C.byref(trel), C.byref(per)))
    return dict(seconds=secs.value, iterations=its.value, true_rel_residual=trel.value,
                seconds_per_iteration=per.value)


def ref_report_reformat(text: str, fmt: str = "json") -> str:
    """Parse a format-1 JSON report with the reference's report_from_json and
    re-emit it with its format_report (report.cpp:152-217)."""
    lib = ref_lib()
    if not hasattr(lib, "ref_report_reformat"):
        raise RuntimeError("reference built without report.cpp (nlohmann json.hpp not found)")
    code = {"text": 0, "json": 1, "csv": 2}[fmt]
    n = C.c_size_t()
    data = text.encode()
    _chk(lib.ref_report_reformat(data, code, None, C.c_size_t(0), C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _chk(lib.ref_report_reformat(data, code, buf, C.c_size_t(n.value + 1), C.byref(n)))
    return buf.value.decode()


def ref_hop_tables():
    out = (C.c_int * 32)()
    ref_lib().ref_hop_tables(out)
    return np.array(out[:], np.int32).reshape(4, 4, 2)


def ref_gamma_matrices():
    out = np.empty((5, 4, 4), np.complex128)
    ref_lib().ref_gamma_matrices(_ptr(out))
    return out


def ref_generators(n):
    out = np.empty((n * n - 1, n, n), np.complex128)
    _chk(ref_lib().ref_generators(n, _ptr(out)))
    return out


def ref_random_group_element(n, key):
    out = np.empty((n, n), np.complex128)
    _chk(ref_lib().ref_random_group_element(n, C.c_uint64(key), _ptr(out)))
    return out


def ref_represent(u, rep):
    n = u.shape[0]
    d = rep_dim(rep, n)
    out = np.empty((d, d), np.complex128)
    _chk(ref_lib().ref_represent(n, rep, _ptr(np.ascontiguousarray(u, np.complex128)), _ptr(out)))
    return out


def ref_key_hash(words):
    arr = (C.c_uint64 * len(words))(*words)
    return int(ref_lib().ref_key_hash(arr, len(words)))


def grid_for_threads_balanced(L, nthreads):
    """The worker grid (prod == nthreads, even local extents) with the fewest
    face sites per worker, then the largest smallest local extent: the
    reference's fastest layout for its halo exchange (profiles/r03_ref_grid*.log:
    2x2x2x2 runs config 2 at 54-58 GFLOP/s on 16 cores against 38-47 for the
    T-only 16x1x1x1). Falls back to grid_for_threads."""
    best, best_cost = None, None

    def rec(d, left, g):
        nonlocal best, best_cost
        if d == 4:
            if left != 1:
                return
            loc = [L[k] // g[k] for k in range(4)]
            vol = loc[0] * loc[1] * loc[2] * loc[3]
            cost = (sum(2 * vol // loc[k] for k in range(4) if g[k] > 1), -min(loc))
            if best_cost is None or cost < best_cost:
                best, best_cost = list(g), cost
            return
        for k in range(1, left + 1):
            if left % k == 0 and L[d] % k == 0 and (L[d] // k) % 2 == 0:
                rec(d + 1, left // k, g + [k])

    rec(0, nthreads, [])
    return best if best is not None else grid_for_threads(L, nthreads)


def grid_for_threads(L, nthreads):
    """A worker grid with prod == nthreads splitting T first (as SURVEY §8e)."""
    grid = [1, 1, 1, 1]
    left = nthreads
    for d in (0, 3, 2, 1):
        for k in range(left, 0, -1):
            if left % k == 0 and L[d] % k == 0 and (L[d] // k) % 2 == 0:
                grid[d] = k
                left //= k
                break
    return grid


# ----------------------------------------------------------------- restatement

def port_spinor_random(L, dr, seed, field_index):
    out = np.empty((volume(L), 4, dr), np.complex128)
    port_lib().oracle_spinor_random(_arr4(L), dr, C.c_uint64(seed), C.c_uint64(field_index), _ptr(out))
    return out


def port_dirac(L, bc_time, mass, gauge, inp, real=None):
    real = gauge.dtype == np.float64 if real is None else real
    out = np.empty_like(inp)
    port_lib().oracle_dirac(_arr4(L), _dr_of(gauge), int(real), int(bc_time), C.c_double(mass),
                            _ptr(gauge), _ptr(np.ascontiguousarray(inp)), _ptr(out))
    return out


def port_hop_parity(L, bc_time, par, coef, gauge, inp):
    out = np.empty_like(inp)
    port_lib().oracle_hop_parity(_arr4(L), _dr_of(gauge), int(gauge.dtype == np.float64), int(bc_time),
                                 int(par), C.c_double(coef), _ptr(gauge),
                                 _ptr(np.ascontiguousarray(inp)), _ptr(out))
    return out


def port_mhat(L, bc_time, mass, gauge, inp):
    out = np.empty_like(inp)
    port_lib().oracle_mhat(_arr4(L), _dr_of(gauge), int(gauge.dtype == np.float64), int(bc_time),
                           C.c_double(mass), _ptr(gauge), _ptr(np.ascontiguousarray(inp)), _ptr(out))
    return out


def port_cg(L, bc_time, eo, mass, gauge, rhs, tol, maxit=10000):
    x = np.empty_like(rhs)
    stats = np.zeros(4, np.float64)
    hist = np.zeros(maxit, np.float64)
    rc = port_lib().oracle_cg(_arr4(L), _dr_of(gauge), int(gauge.dtype == np.float64), int(bc_time),
                              int(eo), C.c_double(mass), _ptr(gauge), _ptr(np.ascontiguousarray(rhs)),
                              C.c_double(tol), int(maxit), _ptr(x), _ptr(stats), _ptr(hist))
    it = int(stats[0])
    return dict(rc=rc, x=x, iterations=it, rel_residual=stats[1], true_rel_residual=stats[2],
                best_residual=stats[3], history=hist[:it].copy())


def port_sqnorm(field):
    return float(port_lib().oracle_sqnorm(C.c_int64(field.size), _ptr(np.ascontiguousarray(field))))


def port_mul_add(c, psi2, psi1):
    out = np.ascontiguousarray(psi2).copy()
    port_lib().oracle_mul_add(C.c_int64(out.size), C.c_double(c.real), C.c_double(c.imag), _ptr(out),
                              _ptr(np.ascontiguousarray(psi1)))
    return out


def port_flops_per_site(kernel, dr, real):
    return int(port_lib().oracle_flops_per_site(kernel, dr, int(real)))


def port_hop_tables():
    out = (C.c_int * 32)()
    port_lib().oracle_hop_tables(out)
    return np.array(out[:], np.int32).reshape(4, 4, 2)


def parity_mask(L):
    """bool[V]: True on even global sites."""
    t, x, y, z = np.meshgrid(*[np.arange(n) for n in L], indexing="ij")
    return (((t + x + y + z) & 1) == 0).reshape(-1)
