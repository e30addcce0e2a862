"""The header-only C++ API (include/latbench_b200.hpp) compiles against the
C-ABI and behaves like the reference API on the device."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_1401_3733_b200 as lb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "api_demo.cpp")
BIN = os.path.join(ROOT, "build", "api_demo")


def build_demo():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    pkg = os.path.join(ROOT, "paper_1401_3733_b200")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC, "-o", BIN,
           "-L", pkg, "-llbcu", f"-Wl,-rpath,{pkg}", "-lpthread"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return BIN


def test_cpp_header_compiles_and_links():
    assert os.path.exists(build_demo())


@pytest.mark.gpu
def test_cpp_api_on_device():
    out = subprocess.run([build_demo()], check=True, capture_output=True, text=True, timeout=300).stdout
    r = json.loads(out.strip().splitlines()[-1])
    L = [8, 4, 4, 4]
    g = lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1)
    s = lb.init_spinor_random(L, 3, 1, 0)
    d = O.port_dirac(L, 1, 0.1, g, s)
    nd = float(np.vdot(d, d).real)
    assert abs(r["sqnorm_Db"] - nd) < 1e-12 * nd
    assert abs(r["bHb_re"] - nd) < 1e-10 * nd and abs(r["bHb_im"]) < 1e-10 * nd
    ref = O.ref_cg_h(L, [1, 1, 1, 1], 3, 0, 1, 0.1, g, s, 1e-10)
    assert abs(r["cg_iters"] - ref["iterations"]) <= 1 and abs(r["cg_h_iters"] - ref["iterations"]) <= 1
    assert r["cg_true"] < 2e-10 and r["cg_eo_true"] < 2e-10
    assert r["history"] == r["cg_iters"]
    assert r["consistency"] == 1 and r["nonconvergence"] == 1 and r["contract"] == 1
