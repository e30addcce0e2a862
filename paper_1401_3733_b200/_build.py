"""In-tree build of the CUDA library (sm_100a) — no JIT cache, no pip install.

Produces ``paper_1401_3733_b200/liblbcu.so`` from ``csrc/*.cu`` and
``csrc/*.cpp`` with nvcc (``-gencode arch=compute_100a,code=sm_100a
-lineinfo``), so the built library travels with the repo snapshot to the GPU
box. Object files go to ``build/`` (git-ignored).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "lbcu")
LIB = os.path.join(PKG, "liblbcu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    return hs + [os.path.join(ROOT, "include", "lbcu.h")]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not _newer(obj, [src, *_headers(), __file__]):
        return obj
    # .cpp sources see the device headers (objects.hpp -> device.cuh): compile as CUDA
    cmd = [NVCC, *ARCH, *COMMON, "-x", "cu", "-c", src, "-o", obj]
    if os.path.basename(src) == "generate.cu":
        cmd += ["--fmad=false"]  # keep the host generators' rounding order
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    if verbose and r.stderr:
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
    return obj


DRIVER_SRC = os.path.join(ROOT, "tools", "latbench_b200.cpp")
DRIVER = os.path.join(ROOT, "tools", "latbench_b200")


def build_driver() -> str:
    """The C++ benchmark driver (run_suite on the device path) over liblbcu.so."""
    deps = [DRIVER_SRC, LIB, os.path.join(ROOT, "include", "latbench_b200.hpp"),
            os.path.join(ROOT, "include", "lbcu.h")]
    if not _newer(DRIVER, deps):
        return DRIVER
    cmd = [os.environ.get("CXX_DRIVER", "g++"), "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
           DRIVER_SRC, "-o", DRIVER, "-L", PKG, "-llbcu", "-Wl,-rpath,$ORIGIN/../paper_1401_3733_b200",
           "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"driver build failed:\n{r.stderr}")
    return DRIVER


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    if not force and not _newer(LIB, [*srcs, *_headers(), __file__]):
        build_driver()
        return LIB  # up to date (the GPU box receives the library without build/)
    if force:
        for s in srcs:
            o = os.path.join(BUILD, os.path.basename(s) + ".o")
            if os.path.exists(o):
                os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if _newer(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static", "-ldl", "-lpthread", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    build_driver()
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
