"""Parity at BASELINE.json's full sizes.

* Dphi against the unmodified reference (oracle/_ref, one worker thread per
  host core) on the full lattice of every config, 1e-12 relative L2;
* size-independent properties on the device: gamma5-hermiticity
  <phi, g5 D g5 psi> = conj <psi, D phi>, linearity, and the Schur relation
  D (x_e - D_oe x_e / A) = (Mhat x_e, 0);
* eo and plain CG iteration counts within +-1 of the unmodified reference's
  at full size (tests/golden/cg_cfg*.npz), the true residual below 2 tol.
"""
import os

import numpy as np
import pytest

import bench
import oracle as O
import paper_1401_3733_b200 as lb
from helpers import rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

LINKS = {"haar": lb.LINKS_HAAR, "near_unit": lb.LINKS_NEAR_UNIT}


def setup_cfg(c, host_gauge=None):
    cfg = bench.CONFIGS[c]
    L, n, rep = cfg["L"], cfg["n"], cfg["rep"]
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T)
    if host_gauge is None:
        gauge.generate(1, links=LINKS[cfg["links"]], eps=0.3)
    else:
        gauge.upload(host_gauge)
    return cfg, ctx, gauge, lb.rep_dim(rep, n)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_dphi_full_size_matches_reference(c):
    cfg = bench.CONFIGS[c]
    L, n, rep, m = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
    g = lb.init_gauge_random(L, n, rep, 1, links=LINKS[cfg["links"]], eps=0.3)
    cfg, ctx, gauge, dr = setup_cfg(c, g)
    s = lb.init_spinor_random(L, dr, 1, 0)
    a, b = lb.SpinorField(ctx, dr).upload(s), lb.SpinorField(ctx, dr)
    lb.apply_dirac(b, gauge, a, m)
    got = b.download()
    grid = O.grid_for_threads(L, os.cpu_count() or 1)
    want = O.ref_apply_dirac(L, grid, n, rep, 1, m, g, s)
    assert rel_l2(got, want) < 1e-12


@pytest.mark.parametrize("c", [2, 3, 4, 5])
def test_full_size_identities(c):
    cfg, ctx, gauge, dr = setup_cfg(c)
    m = cfg["mass"]
    psi = lb.SpinorField(ctx, dr).randomize(1, 0)
    phi = lb.SpinorField(ctx, dr).randomize(1, 1)
    t1, t2 = lb.SpinorField(ctx, dr), lb.SpinorField(ctx, dr)
    # gamma5-hermiticity: <phi, g5 D g5 psi> = conj <psi, D phi>
    lb.copy_interior(t1, psi)
    lb.apply_gamma5(t1)
    lb.apply_dirac(t2, gauge, t1, m)
    lb.apply_gamma5(t2)
    lhs = lb.dot(phi, t2)
    lb.apply_dirac(t1, gauge, phi, m)
    rhs = np.conj(lb.dot(psi, t1))
    assert abs(lhs - rhs) < 1e-12 * abs(rhs)
    # linearity: D(a psi + phi) = a D psi + D phi
    a = 0.7 - 0.2j
    lb.copy_interior(t1, phi)
    lb.axpy(t1, a, psi)
    lb.apply_dirac(t2, gauge, t1, m)
    dpsi, dphi = lb.SpinorField(ctx, dr), lb.SpinorField(ctx, dr)
    lb.apply_dirac(dpsi, gauge, psi, m)
    lb.apply_dirac(dphi, gauge, phi, m)
    lb.axpy(dphi, a, dpsi)
    lb.axpy(t2, -1.0, dphi)
    assert np.sqrt(lb.sqnorm(t2) / lb.sqnorm(dphi)) < 1e-13
    # Schur: x = (x_e, -D_oe x_e / A)  =>  D x = (Mhat x_e, 0)
    A = 4.0 + m
    xe = lb.SpinorField(ctx, dr, lb.EVEN).randomize(1, 2)
    xo = lb.SpinorField(ctx, dr, lb.ODD)
    lb.dphi_oe(xo, gauge, xe)
    host = xe.download() - xo.download() / A  # even and odd parts are disjoint
    x = lb.SpinorField(ctx, dr).upload(host)
    lb.apply_dirac(t1, gauge, x, m)
    me = lb.SpinorField(ctx, dr, lb.EVEN)
    lb.mhat(me, gauge, xe, m)
    full = t1.download()
    even = O.parity_mask(cfg["L"])
    assert rel_l2(full[even], me.download()[even]) < 1e-12
    assert np.abs(full[~even]).max() < 1e-12 * np.abs(full[even]).max()


def golden_cg(c):
    """The unmodified reference's CG at this config's full size
    (tests/golden/make_fullsize_cg.py): plain cg_solve(make_h_operator) and
    the cg_solve driven by the composed eo operator."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"cg_cfg{c}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return np.load(path)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_full_size_eo_cg(c):
    """eo CG iterations within +-1 of the reference-composed eo CG at full size."""
    cfg, ctx, gauge, dr = setup_cfg(c)
    rhs = lb.SpinorField(ctx, dr, lb.EVEN).randomize(1, 0)
    o = lb.cg_solve_eo(gauge, cfg["mass"], rhs, lb.CgSettings(cfg["tol"], 5000))
    z = golden_cg(c)
    assert o.true_rel_residual < 2 * cfg["tol"]
    assert abs(o.iterations - int(z["eo_iterations"])) <= 1, (o.iterations, int(z["eo_iterations"]))
    # the residual history follows the reference's until rounding separates them
    k = min(10, o.iterations, len(z["eo_history"]))
    assert np.allclose(o.residual_history[:k], z["eo_history"][:k], rtol=1e-6)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_full_size_plain_cg(c):
    """Plain CG on D^dag D (the reference's own consistency solve, solver.cpp:24-82)
    within +-1 of the reference's iteration count at full size."""
    cfg, ctx, gauge, dr = setup_cfg(c)
    rhs = lb.SpinorField(ctx, dr).randomize(1, 0)
    o = lb.cg_solve_h(gauge, cfg["mass"], rhs, lb.CgSettings(cfg["tol"], 5000))
    z = golden_cg(c)
    assert o.true_rel_residual < 2 * cfg["tol"]
    assert abs(o.iterations - int(z["h_iterations"])) <= 1, (o.iterations, int(z["h_iterations"]))
    k = min(10, o.iterations, len(z["h_history"]))
    assert np.allclose(o.residual_history[:k], z["h_history"][:k], rtol=1e-6)
