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
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin_demo")
REF_INCLUDE = "/root/reference/proj/include"
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


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference headers absent (GPU box)")
def test_dropin_header_compiles_against_reference_types():
    """include/latbench_b200_dropin.hpp: a caller written on the reference's own
    headers and types (latbench::SpinorField/GaugeField/Worker/ExchangePlan/
    Clock) compiles and links with the device versions of apply_dirac,
    apply_h, make_h_operator, cg_solve and consistency_check beside the
    reference's CPU ones (oracle/Makefile `dropin`)."""
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "dropin"], check=True, capture_output=True, text=True)
    assert os.path.exists(DROPIN)
    # every device entry point the header names is exported by the library
    syms = subprocess.run(["nm", "-D", "--defined-only", os.path.join(ROOT, "paper_1401_3733_b200", "liblbcu.so")],
                          check=True, capture_output=True, text=True).stdout
    for name in ("lbcu_dphi", "lbcu_h", "lbcu_cg_solve", "lbcu_cg_solve_h", "lbcu_world_threads"):
        assert f" {name}\n" in syms


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["8", "4", "4", "4", "1", "1", "1", "1", "3", "0", "0.1"],   # SU(3)F, one worker
    ["8", "4", "4", "8", "2", "1", "1", "2", "2", "0", "0.05"],  # SU(2)F, 4 workers (T and Z split)
    ["8", "4", "4", "4", "2", "1", "1", "1", "2", "1", "0.05"],  # SU(2) adjoint (real links), 2 workers
], ids=["su3f_1", "su2f_2x1x1x2", "su2a_2x1x1x1"])
def test_dropin_matches_reference_on_its_own_types(args):
    """The reference's caller, unchanged but for the namespace of its hot
    calls, gets the reference's results from the device: Dphi and H within
    1e-12, CG iterations within +-1 (fused device CG and host-callback CG),
    the reference exception types, re-upload after invalidate()."""
    if not os.path.exists(DROPIN):
        pytest.skip("dropin_demo not built (needs the reference headers at build time)")
    out = subprocess.run([DROPIN, *args], check=True, capture_output=True, text=True, timeout=600).stdout
    r = json.loads(out.strip().splitlines()[-1])
    assert r["dirac_rel"] < 1e-12 and r["h_rel"] < 1e-12 and r["invalidate_rel"] < 1e-12
    assert abs(r["cg_dev_iters"] - r["cg_ref_iters"]) <= 1 and abs(r["cg_cb_iters"] - r["cg_ref_iters"]) <= 1
    assert r["cg_dev_true"] < 2e-10 and r["cg_cb_true"] < 2e-10
    assert r["x_rel"] < 1e-8 and r["x_cb_rel"] < 1e-8
    assert r["history"] == r["cg_dev_iters"]
    assert r["consistency"] == 1 and r["nonconvergence"] == 1 and r["config_error"] == 1
