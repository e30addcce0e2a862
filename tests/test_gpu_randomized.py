"""Randomised parity (hypothesis): lattice shapes, representations, storage
formats, masses, boundary conditions, seeds and operator variants drawn at
random, every draw checked against the plain-C oracle (oracle/oracle.c,
pinned to the reference by tests/test_oracle.py). Shapes cover the ragged
cases the tiled layout has to handle: extents of 2, odd numbers of 32-site
tiles, z-rows that do not divide a warp."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle as O
import paper_1401_3733_b200 as lb
from helpers import rel_l2

pytestmark = pytest.mark.gpu

# (group rank, representation, link generator) pairs the device specialises
REPS = [(3, lb.FUNDAMENTAL, lb.LINKS_HAAR), (3, lb.FUNDAMENTAL, lb.LINKS_NEAR_UNIT), (2, lb.FUNDAMENTAL, lb.LINKS_HAAR),
        (2, lb.ADJOINT, lb.LINKS_HAAR), (4, lb.ANTISYMMETRIC, lb.LINKS_HAAR), (4, lb.FUNDAMENTAL, lb.LINKS_HAAR),
        (3, lb.SYMMETRIC, lb.LINKS_HAAR)]

extent = st.sampled_from([2, 4, 6, 8, 10])
case = st.fixed_dictionaries({
    "L": st.tuples(extent, extent, extent, extent),
    "rep": st.sampled_from(range(len(REPS))),
    "mass": st.floats(min_value=-0.5, max_value=1.0, allow_nan=False),
    "bc": st.sampled_from([lb.PERIODIC, lb.ANTIPERIODIC_T]),
    "seed": st.integers(min_value=1, max_value=2 ** 40),
    "compact": st.booleans(),
})


def _setup(c):
    n, rep, links = REPS[c["rep"]]
    L = list(c["L"])
    dr = lb.rep_dim(rep, n)
    g = lb.init_gauge_random(L, n, rep, c["seed"], links=links)
    s = lb.init_spinor_random(L, dr, c["seed"], 3)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, c["bc"]).set_compact(c["compact"]).upload(g)
    return L, dr, g, s, ctx, gauge


@settings(max_examples=40, deadline=None, suppress_health_check=list(HealthCheck))
@given(case)
def test_random_dphi_and_eo_blocks(c):
    L, dr, g, s, ctx, gauge = _setup(c)
    m = c["mass"]
    a, b = lb.SpinorField(ctx, dr).upload(s), lb.SpinorField(ctx, dr)
    lb.apply_dirac(b, gauge, a, m)
    assert rel_l2(b.download(), O.port_dirac(L, c["bc"], m, g, s)) < 1e-12
    e_in, e_out = lb.SpinorField(ctx, dr, lb.EVEN).upload(s), lb.SpinorField(ctx, dr, lb.EVEN)
    lb.mhat(e_out, gauge, e_in, m)
    assert rel_l2(e_out.download(), O.port_mhat(L, c["bc"], m, g, s)) < 1e-12
    # gamma5-hermiticity of D on the device: <phi, g5 D g5 psi> = conj <psi, D phi>
    phi = lb.SpinorField(ctx, dr).upload(lb.init_spinor_random(L, dr, c["seed"], 4))
    t1, t2 = lb.SpinorField(ctx, dr), lb.SpinorField(ctx, dr)
    lb.copy_interior(t1, a)
    lb.apply_gamma5(t1)
    lb.apply_dirac(t2, gauge, t1, m)
    lb.apply_gamma5(t2)
    lhs = lb.dot(phi, t2)
    lb.apply_dirac(t1, gauge, phi, m)
    rhs = np.conj(lb.dot(a, t1))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(rhs), 1.0)
    ctx.close()


@settings(max_examples=12, deadline=None, suppress_health_check=list(HealthCheck))
@given(case, st.booleans())
def test_random_cg_matches_oracle(c, eo):
    c = dict(c, mass=abs(c["mass"]) + 0.05)  # keep D^dag D well conditioned
    L, dr, g, s, ctx, gauge = _setup(c)
    sub = lb.EVEN if eo else lb.FULL
    rhs = lb.SpinorField(ctx, dr, sub).upload(s)
    run = lb.cg_solve_eo if eo else lb.cg_solve_h
    o = run(gauge, c["mass"], rhs, lb.CgSettings(1e-10, 2000))
    ref = O.port_cg(L, c["bc"], int(eo), c["mass"], g, s, 1e-10, 2000)
    assert abs(o.iterations - ref["iterations"]) <= 1
    assert o.true_rel_residual < 2e-10
    assert rel_l2(o.solution.download(), ref["x"]) < 1e-8
    ctx.close()
