"""GPU parity: the CUDA path through the C-ABI against the CPU oracle.

Bar (BASELINE.json north_star): Dphi within 1e-12 relative L2 per field in
fp64; CG iterations within +-1 of the reference with the true residual below
the tolerance. Inputs are the reference's own seeded generators (seed 1).
"""
import numpy as np
import pytest

import oracle as O
import paper_1401_3733_b200 as lb
from helpers import REP_IDS, REPS, global_index, rel_l2, run_ranks

pytestmark = pytest.mark.gpu

TOL_DPHI = 1e-12  # relative L2, north_star


def fields(L, n, rep, seed=1, field=0, links=lb.LINKS_HAAR):
    dr = lb.rep_dim(rep, n)
    g = lb.init_gauge_random(L, n, rep, seed, links=links)
    s = lb.init_spinor_random(L, dr, seed, field)
    return dr, g, s


def setup(L, n, rep, bc=lb.ANTIPERIODIC_T, grid=(1, 1, 1, 1)):
    ctx = lb.Context(L, grid)
    dr, g, s = fields(L, n, rep)
    gauge = lb.GaugeField(ctx, n, rep, bc).upload(g)
    return ctx, dr, g, s, gauge


@pytest.mark.parametrize("n,rep", REPS, ids=REP_IDS)
@pytest.mark.parametrize("bc", [lb.PERIODIC, lb.ANTIPERIODIC_T], ids=["periodic", "antiperiodic"])
def test_dphi_matches_oracle(n, rep, bc):
    L = [8, 4, 4, 6]
    ctx, dr, g, s, gauge = setup(L, n, rep, bc)
    inp = lb.SpinorField(ctx, dr).upload(s)
    out = lb.SpinorField(ctx, dr)
    lb.apply_dirac(out, gauge, inp, 0.1)
    got = out.download()
    want = O.port_dirac(L, bc, 0.1, g, s)
    assert rel_l2(got, want) < TOL_DPHI
    # and the unmodified reference itself
    ref = O.ref_apply_dirac(L, [1, 1, 1, 1], n, rep, bc, 0.1, g, s)
    assert rel_l2(got, ref) < TOL_DPHI


@pytest.mark.parametrize("n,rep", REPS, ids=REP_IDS)
def test_g5dphi_and_h(n, rep):
    L = [4, 4, 6, 4]
    ctx, dr, g, s, gauge = setup(L, n, rep)
    inp = lb.SpinorField(ctx, dr).upload(s)
    out = lb.SpinorField(ctx, dr)
    lb.apply_g5dirac(out, gauge, inp, 0.05)
    want = O.port_dirac(L, 1, 0.05, g, s)
    want[:, 2:, :] *= -1
    assert rel_l2(out.download(), want) < TOL_DPHI
    lb.apply_h(out, gauge, inp, 0.05)
    ref = O.ref_apply_h(L, [1, 1, 1, 1], n, rep, 1, 0.05, g, s)
    assert rel_l2(out.download(), ref) < TOL_DPHI


@pytest.mark.parametrize("n,rep", REPS, ids=REP_IDS)
def test_eo_blocks_and_mhat(n, rep):
    L = [4, 6, 4, 4]
    ctx, dr, g, s, gauge = setup(L, n, rep)
    even = O.parity_mask(L)
    e_in = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    o_in = lb.SpinorField(ctx, dr, lb.ODD).upload(s)
    e_out = lb.SpinorField(ctx, dr, lb.EVEN)
    o_out = lb.SpinorField(ctx, dr, lb.ODD)
    lb.dphi_eo(e_out, gauge, o_in)
    s_odd = s.copy()
    s_odd[even] = 0
    want = O.port_hop_parity(L, 1, 0, -0.5, g, s_odd)
    assert rel_l2(e_out.download(), want) < TOL_DPHI
    lb.dphi_oe(o_out, gauge, e_in)
    s_even = s.copy()
    s_even[~even] = 0
    want = O.port_hop_parity(L, 1, 1, -0.5, g, s_even)
    assert rel_l2(o_out.download(), want) < TOL_DPHI
    lb.mhat(e_out, gauge, e_in, 0.1)
    got = e_out.download()
    assert rel_l2(got, O.port_mhat(L, 1, 0.1, g, s)) < TOL_DPHI
    assert rel_l2(got, O.ref_mhat(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s)) < TOL_DPHI


def test_unit_gauge_constant_spinor_mass_identity():
    """unit links, constant spinor, periodic BC -> D psi = m psi."""
    L = [4, 4, 4, 4]
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, 3, lb.FUNDAMENTAL, lb.PERIODIC)
    gauge.upload(lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1, links=lb.LINKS_UNIT))
    rng = np.random.default_rng(0)
    site = rng.normal(size=(4, 3)) + 1j * rng.normal(size=(4, 3))
    s = np.broadcast_to(site, (256, 4, 3)).copy()
    inp = lb.SpinorField(ctx, 3).upload(s)
    out = lb.SpinorField(ctx, 3)
    lb.apply_dirac(out, gauge, inp, 0.37)
    assert np.abs(out.download() - 0.37 * s).max() < 1e-13


@pytest.mark.parametrize("n,rep", REPS[:2], ids=REP_IDS[:2])
def test_blas_matches_reference(n, rep):
    L = [4, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, n, rep)
    s1 = lb.init_spinor_random(L, dr, 1, 1)
    a = lb.SpinorField(ctx, dr).upload(s)
    b = lb.SpinorField(ctx, dr).upload(s1)
    assert abs(lb.sqnorm(a) - O.ref_sqnorm(L, [1, 1, 1, 1], s)) < 1e-10 * O.ref_sqnorm(L, [1, 1, 1, 1], s)
    d = lb.dot(a, b)
    dr_ = O.ref_dot(L, [1, 1, 1, 1], s, s1)
    assert abs(d - dr_) < 1e-10 * abs(dr_) + 1e-9
    lb.mul_add(a, 0.3 + 0.7j, b)
    assert rel_l2(a.download(), O.ref_mul_add(L, [1, 1, 1, 1], 0.3 + 0.7j, s, s1)) < 1e-15
    lb.apply_gamma5(b)
    w = s1.copy()
    w[:, 2:] *= -1
    assert np.array_equal(b.download(), w)


@pytest.mark.parametrize("n,rep", REPS[:2], ids=REP_IDS[:2])
def test_xpay_axpy_copy_zero_match_reference(n, rep):
    """kernels.cpp:45-49,75-104: xpay y = x + a y, axpy y += a x, copy, zero —
    against the reference's formulas on the same fields (bit-exact: one
    complex multiply-add per component, no reduction)."""
    L = [4, 4, 6, 4]
    dr = lb.rep_dim(rep, n)
    ctx = lb.Context(L)
    s0 = lb.init_spinor_random(L, dr, 1, 0)
    s1 = lb.init_spinor_random(L, dr, 1, 1)
    a = 0.3 - 1.7j
    x, y = lb.SpinorField(ctx, dr).upload(s0), lb.SpinorField(ctx, dr).upload(s1)
    lb.xpay(y, a, x)
    assert rel_l2(y.download(), s0 + a * s1) < 1e-15
    y.upload(s1)
    lb.axpy(y, a, x)
    assert rel_l2(y.download(), s1 + a * s0) < 1e-15
    lb.copy_interior(y, x)
    assert np.array_equal(y.download(), s0)
    lb.zero_interior(y)
    assert not y.download().any()
    # parity subsets: xpay on EVEN fields touches even sites only
    even = O.parity_mask(L)
    xe, ye = lb.SpinorField(ctx, dr, lb.EVEN).upload(s0), lb.SpinorField(ctx, dr, lb.EVEN).upload(s1)
    lb.xpay(ye, a, xe)
    got = ye.download()
    assert rel_l2(got[even], (s0 + a * s1)[even]) < 1e-15 and not got[~even].any()


def test_cg_graph_cache_follows_field_lifetimes():
    """The cached CG graph (one per context + field set) is dropped when a
    field it names is destroyed or the links are re-uploaded: a re-upload
    that changes the link storage format, and fields re-created at a recycled
    address, still solve correctly."""
    L = [8, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, 3, lb.FUNDAMENTAL)
    rhs = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    x = lb.SpinorField(ctx, dr, lb.EVEN)
    st = lb.CgSettings(1e-10, 500)
    ref = O.port_cg(L, 1, 1, 0.1, g, s, 1e-10)
    o1 = lb.cg_solve_eo(gauge, 0.1, rhs, st, x)
    assert ctx.cached_solves() == 1
    lb.cg_solve_eo(gauge, 0.1, rhs, st, x)
    assert ctx.cached_solves() == 1  # replayed, not re-captured
    assert gauge.storage()[0] == "r10"
    gauge.set_compact(False).upload(g)  # new link buffer, dense format
    assert ctx.cached_solves() == 0 and gauge.storage()[0] == "full"
    o2 = lb.cg_solve_eo(gauge, 0.1, rhs, st, x)
    assert abs(o2.iterations - ref["iterations"]) <= 1 and o2.true_rel_residual < 2e-10
    x2 = o2.solution.download()
    assert rel_l2(x2, O.port_cg(L, 1, 1, 0.1, g, s, 1e-10)["x"]) < 1e-8
    x.close()
    assert ctx.cached_solves() == 0
    for _ in range(3):  # handles recycled at the same addresses
        x = lb.SpinorField(ctx, dr, lb.EVEN)
        o3 = lb.cg_solve_eo(gauge, 0.1, rhs, st, x)
        assert o3.iterations == o2.iterations and rel_l2(x.download(), x2) < 1e-12
        x.close()
    gauge.close()
    assert ctx.cached_solves() == 0


def test_fields_are_freed_with_their_context():
    """Python fields free their device memory when collected, a context
    closes its live fields before itself, and a garbage cycle holding a
    context and its fields is finalised fields-first (no handle is ever freed
    through a destroyed context)."""
    import gc
    L = [8, 8, 8, 8]
    ctx = lb.Context(L)
    fs = [lb.SpinorField(ctx, 3) for _ in range(4)]
    g = lb.GaugeField(ctx, 3)
    del fs
    gc.collect()
    assert len(ctx._rec[2]) == 1  # only the gauge field is still registered
    ctx.close()
    assert g._h is None and not ctx._rec[2]
    g.close()  # idempotent
    for _ in range(3):  # cycles: context <-> fields collected together
        c2 = lb.Context(L)
        f2 = [lb.SpinorField(c2, 3), lb.GaugeField(c2, 3)]
        c2.cycle = f2
        for f in f2:
            f.cycle = c2
        del c2, f2, f
        gc.collect()
    w = lb.World.threads(1)
    c3 = lb.Context(L, (1, 1, 1, 1), 0, 0, w)
    lb.SpinorField(c3, 3)
    w.close()  # the world closes its context, which closes its field
    assert c3._h is None


@pytest.mark.parametrize("n,rep", REPS, ids=REP_IDS)
def test_cg_h_matches_reference(n, rep):
    L = [8, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, n, rep)
    rhs = lb.SpinorField(ctx, dr).upload(s)
    st = lb.CgSettings(1e-10, 1000)
    o = lb.cg_solve_h(gauge, 0.1, rhs, st)
    ref = O.ref_cg_h(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s, 1e-10)
    assert abs(o.iterations - ref["iterations"]) <= 1
    assert o.true_rel_residual < 2e-10
    assert rel_l2(o.solution.download(), ref["x"]) < 1e-8
    assert len(o.residual_history) == o.iterations


@pytest.mark.parametrize("n,rep", REPS, ids=REP_IDS)
def test_cg_eo_matches_oracle(n, rep):
    L = [8, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, n, rep)
    rhs = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    o = lb.cg_solve_eo(gauge, 0.1, rhs, lb.CgSettings(1e-10, 1000))
    ref = O.ref_cg_eo(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s, 1e-10)
    assert abs(o.iterations - ref["iterations"]) <= 1
    assert o.true_rel_residual < 2e-10
    x = o.solution.download()
    assert rel_l2(x, ref["x"]) < 1e-8


def test_cg_callback_operator_matches_fused():
    L = [8, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, 3, lb.FUNDAMENTAL)
    rhs = lb.SpinorField(ctx, dr).upload(s)
    tmp = lb.SpinorField(ctx, dr)
    calls = []

    def op(out, inp):  # make_h_operator composed from the public kernels (solver.cpp:9-15)
        calls.append(1)
        lb.apply_dirac(tmp, gauge, inp, 0.1)
        lb.apply_gamma5(tmp)
        lb.apply_dirac(out, gauge, tmp, 0.1)
        lb.apply_gamma5(out)

    o = lb.cg_solve(op, rhs, lb.CgSettings(1e-10, 500))
    f = lb.cg_solve_h(gauge, 0.1, rhs, lb.CgSettings(1e-10, 500))
    assert abs(o.iterations - f.iterations) <= 1
    assert len(calls) == o.iterations + 1  # + the true-residual application
    assert rel_l2(o.solution.download(), f.solution.download()) < 1e-8


def test_cg_zero_rhs_and_nonconvergence():
    L = [4, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, 3, lb.FUNDAMENTAL)
    z = lb.SpinorField(ctx, dr)
    o = lb.cg_solve_h(gauge, 0.1, z)
    assert o.iterations == 0 and not np.any(o.solution.download())
    rhs = lb.SpinorField(ctx, dr).upload(s)
    with pytest.raises(lb.NonConvergence) as ei:
        lb.cg_solve_h(gauge, 0.1, rhs, lb.CgSettings(1e-12, 3))
    assert ei.value.iterations == 3 and 0 < ei.value.best_residual < 1


def test_planted_solution_recovered():
    """rhs = H x0 -> x0 recovered to 1e-5 at tol 1e-7."""
    L = [4, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, 2, lb.FUNDAMENTAL)
    x0 = lb.SpinorField(ctx, dr).upload(s)
    rhs = lb.SpinorField(ctx, dr)
    lb.apply_h(rhs, gauge, x0, 0.1)
    o = lb.cg_solve_h(gauge, 0.1, rhs, lb.CgSettings(1e-7))
    assert rel_l2(o.solution.download(), s) < 1e-5


def test_tampered_operator_fails_consistency():
    """a sign-flipped Dirac operator must fail the true-residual check."""
    L = [4, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, 3, lb.FUNDAMENTAL)
    rhs = lb.SpinorField(ctx, dr).upload(s)
    tmp = lb.SpinorField(ctx, dr)
    state = {"n": 0}

    def op(out, inp):
        state["n"] += 1
        lb.apply_h(out, gauge, inp, 0.1)
        if state["n"] % 2 == 0:  # corrupt every second application
            lb.axpy(out, -1e-3, inp)

    try:
        o = lb.cg_solve(op, rhs, lb.CgSettings(1e-10, 300))
        assert o.true_rel_residual >= 2e-10
    except lb.NonConvergence:
        pass


@pytest.mark.parametrize("direct", [False, True], ids=["copy", "direct"])
@pytest.mark.parametrize("grid", [(2, 1, 1, 1), (2, 1, 1, 2), (1, 2, 2, 1)], ids=["t2", "t2z2", "x2y2"])
@pytest.mark.parametrize("n,rep", [REPS[0], REPS[1], REPS[3]], ids=[REP_IDS[0], REP_IDS[1], REP_IDS[3]])
def test_decomposed_dphi_matches_single(grid, n, rep, direct):
    """Serial oracle vs decomposition: ranks as host threads on one GPU,
    half-spinor halos packed by kernels and exchanged by the thread transport
    (copy: buffers copied between barriers; direct: the pack kernel stores
    into the receiving rank's arena, event + host barrier per exchange)."""
    L = [8, 4, 4, 8]
    dr, g, s = fields(L, n, rep)
    want = O.port_dirac(L, 1, 0.1, g, s)
    nranks = int(np.prod(grid))
    world = lb.World.threads(nranks, direct=direct)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        idx = global_index(L, grid, r)
        gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g[idx])
        inp = lb.SpinorField(ctx, dr).upload(s[idx])
        out = lb.SpinorField(ctx, dr)
        lb.apply_dirac(out, gauge, inp, 0.1)
        return idx, out.download()

    got = np.empty_like(want)
    for idx, part in run_ranks(nranks, body):
        got[idx] = part
    assert rel_l2(got, want) < 1e-14


@pytest.mark.parametrize("single", ["0", "1"], ids=["two-reductions", "single-reduction"])
@pytest.mark.parametrize("solver", ["eo", "h"])
@pytest.mark.parametrize("direct", [False, True], ids=["copy", "direct"])
def test_decomposed_cg_matches_single(direct, solver, single, monkeypatch):
    """Decomposed eo and plain CG against the reference CG on the whole
    lattice: the reference recurrence (pAp and rr summed across ranks one
    after the other) and the single-reduction Chronopoulos-Gear form (both
    in one allreduce, LBCU_CG_SINGLE_REDUCE) give the reference's iteration
    count +-1, its solution and the same residual history to rounding."""
    monkeypatch.setenv("LBCU_CG_SINGLE_REDUCE", single)
    L = [8, 4, 4, 8]
    n, rep = 3, lb.FUNDAMENTAL
    dr, g, s = fields(L, n, rep)
    refn = O.ref_cg_eo if solver == "eo" else O.ref_cg_h
    ref = refn(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s, 1e-10)
    grid = (2, 1, 1, 2)
    world = lb.World.threads(4, direct=direct)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        idx = global_index(L, grid, r)
        gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g[idx])
        rhs = lb.SpinorField(ctx, dr, lb.EVEN if solver == "eo" else lb.FULL).upload(s[idx])
        run = lb.cg_solve_eo if solver == "eo" else lb.cg_solve_h
        o = run(gauge, 0.1, rhs, lb.CgSettings(1e-10, 500))
        return idx, o.iterations, o.true_rel_residual, o.solution.download(), o.residual_history

    x = np.empty_like(s)
    for idx, it, tr, part, hist in run_ranks(4, body):
        assert abs(it - ref["iterations"]) <= 1
        assert tr < 2e-10
        k = min(it, ref["iterations"]) - 2
        assert np.allclose(hist[:k], ref["history"][:k], rtol=1e-6)
        x[idx] = part
    assert rel_l2(x, ref["x"]) < 1e-8


@pytest.mark.parametrize("solver", ["eo", "h"])
def test_single_reduction_cg_on_one_rank(solver, monkeypatch):
    """The single-reduction recurrence forced on one rank (host loop) agrees
    with the reference CG: iterations +-1, solution, true residual."""
    monkeypatch.setenv("LBCU_CG_SINGLE_REDUCE", "1")
    L = [8, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, 2, lb.ADJOINT)
    rhs = lb.SpinorField(ctx, dr, lb.EVEN if solver == "eo" else lb.FULL).upload(s)
    run = lb.cg_solve_eo if solver == "eo" else lb.cg_solve_h
    o = run(gauge, 0.1, rhs, lb.CgSettings(1e-10, 500))
    refn = O.ref_cg_eo if solver == "eo" else O.ref_cg_h
    ref = refn(L, [1, 1, 1, 1], 2, lb.ADJOINT, 1, 0.1, g, s, 1e-10)
    assert abs(o.iterations - ref["iterations"]) <= 1 and o.true_rel_residual < 2e-10
    assert rel_l2(o.solution.download(), ref["x"]) < 1e-8
    with pytest.raises(lb.NonConvergence):
        run(gauge, 0.1, rhs, lb.CgSettings(1e-10, ref["iterations"] - 3))


def test_near_unit_links_cg_eo():
    """BASELINE config 3 structure (near-unit links, small mass) at a reduced volume."""
    L = [8, 4, 4, 4]
    n, rep = 3, lb.FUNDAMENTAL
    dr, g, s = fields(L, n, rep, links=lb.LINKS_NEAR_UNIT)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g)
    rhs = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    o = lb.cg_solve_eo(gauge, 0.02, rhs, lb.CgSettings(1e-12, 2000))
    ref = O.ref_cg_eo(L, [1, 1, 1, 1], n, rep, 1, 0.02, g, s, 1e-12)
    assert abs(o.iterations - ref["iterations"]) <= 1
    assert o.true_rel_residual < 2e-12


@pytest.mark.parametrize("n,rep,links,fmt", [
    (2, lb.FUNDAMENTAL, lb.LINKS_HAAR, "su2"),
    (2, lb.ADJOINT, lb.LINKS_HAAR, "su2"),
    (3, lb.FUNDAMENTAL, lb.LINKS_HAAR, "r10"),
    (3, lb.FUNDAMENTAL, lb.LINKS_NEAR_UNIT, "r10"),
    (3, lb.FUNDAMENTAL, lb.LINKS_HAAR, "r12"),
    (3, lb.FUNDAMENTAL, lb.LINKS_NEAR_UNIT, "r12"),
    (4, lb.ANTISYMMETRIC, lb.LINKS_HAAR, "as4r"),
], ids=["su2f", "su2a", "su3f-r10", "su3f-near-unit-r10", "su3f-r12", "su3f-near-unit-r12", "su4as"])
@pytest.mark.parametrize("bc", [lb.PERIODIC, lb.ANTIPERIODIC_T], ids=["periodic", "antiperiodic"])
def test_compact_link_storage_is_exact(n, rep, links, fmt, bc, monkeypatch):
    """Compact link formats (links.cuh) give the same Dphi as dense storage and
    the oracle, and download the uploaded links (SU(3): R10 by default, R12
    with LBCU_SU3_STORAGE=r12)."""
    if fmt == "r12":
        monkeypatch.setenv("LBCU_SU3_STORAGE", "r12")
    L = [4, 4, 6, 4]
    dr, g, s = fields(L, n, rep, links=links)
    ctx = lb.Context(L)
    gc = lb.GaugeField(ctx, n, rep, bc).upload(g)
    gf = lb.GaugeField(ctx, n, rep, bc).set_compact(False).upload(g)
    assert gc.storage()[0] == fmt and gf.storage()[0] == "full"
    if fmt != "full":
        assert gc.storage()[1] < 1e-13
    inp = lb.SpinorField(ctx, dr).upload(s)
    oc, of = lb.SpinorField(ctx, dr), lb.SpinorField(ctx, dr)
    lb.apply_dirac(oc, gc, inp, 0.1)
    lb.apply_dirac(of, gf, inp, 0.1)
    want = O.port_dirac(L, bc, 0.1, g, s)
    assert rel_l2(oc.download(), want) < TOL_DPHI
    assert rel_l2(of.download(), want) < TOL_DPHI
    assert np.abs(gc.download() - g).max() < 1e-12
    assert np.array_equal(gf.download(), g)


def test_r10_falls_back_to_r12_when_the_pivot_is_tiny():
    """R10 divides by U_00: a link with U_00 ~ 1e-14 cannot be rebuilt to
    1e-12 from 5 entries, so the upload keeps R12 for that field (exact)."""
    L = [4, 4, 4, 4]
    g = lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1)
    # an SU(3) link with |U_00| = 1e-13: row 0 fixed, row 1 a random unit
    # vector orthogonal to it, row 2 = conj(row0 x row1)
    rng = np.random.default_rng(5)
    r0 = np.array([1e-13, 0.6 + 0.2j, 0.0])
    r0[2] = np.sqrt(1 - np.vdot(r0, r0).real)
    v = rng.normal(size=3) + 1j * rng.normal(size=3)
    r1 = v - np.vdot(r0, v) * r0
    r1 /= np.linalg.norm(r1)
    q = np.array([r0, r1, np.conj(np.cross(r0, r1))])
    assert np.abs(q @ q.conj().T - np.eye(3)).max() < 1e-14 and abs(np.linalg.det(q) - 1) < 1e-14
    g[5, 1] = q
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, 3, lb.FUNDAMENTAL, lb.ANTIPERIODIC_T).upload(g)
    assert gauge.storage()[0] == "r12"
    s = lb.init_spinor_random(L, 3, 1, 0)
    inp, out = lb.SpinorField(ctx, 3).upload(s), lb.SpinorField(ctx, 3)
    lb.apply_dirac(out, gauge, inp, 0.1)
    assert rel_l2(out.download(), O.port_dirac(L, 1, 0.1, g, s)) < TOL_DPHI


def test_non_group_links_stay_dense():
    """Arbitrary (non-unitary) links must not be compressed."""
    L = [4, 4, 4, 4]
    rng = np.random.default_rng(3)
    g = rng.normal(size=(256, 4, 3, 3)) + 1j * rng.normal(size=(256, 4, 3, 3))
    s = lb.init_spinor_random(L, 3, 1, 0)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, 3, lb.FUNDAMENTAL, lb.ANTIPERIODIC_T).upload(g)
    assert gauge.storage()[0] == "full"
    inp, out = lb.SpinorField(ctx, 3).upload(s), lb.SpinorField(ctx, 3)
    lb.apply_dirac(out, gauge, inp, 0.1)
    assert rel_l2(out.download(), O.port_dirac(L, 1, 0.1, g, s)) < TOL_DPHI


@pytest.mark.parametrize("solver", ["eo", "h"])
def test_cg_host_loop_matches_graph(solver, monkeypatch):
    """The host-driven loop (multi-rank path, one iteration enqueued ahead of
    the state read-back) gives the same iterations, history and solution as
    the single-rank CUDA-graph loop: the speculative iteration after
    convergence must leave x, p and the CG state untouched."""
    L = [8, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, 2, lb.FUNDAMENTAL)
    sub = lb.EVEN if solver == "eo" else lb.FULL
    rhs = lb.SpinorField(ctx, dr, sub).upload(s)
    st = lb.CgSettings(1e-10, 1000)
    run = lb.cg_solve_eo if solver == "eo" else lb.cg_solve_h
    a = run(gauge, 0.1, rhs, st)
    monkeypatch.setenv("LBCU_CG_GRAPH", "0")
    b = run(gauge, 0.1, rhs, st)
    assert a.iterations == b.iterations
    assert np.array_equal(np.asarray(a.residual_history), np.asarray(b.residual_history))
    assert np.array_equal(a.solution.download(), b.solution.download())
    assert a.true_rel_residual == b.true_rel_residual
    # a tolerance reached at the iteration cap: the loop stops at max_iterations
    with pytest.raises(lb.NonConvergence):
        run(gauge, 0.1, rhs, lb.CgSettings(1e-10, a.iterations - 2))


def test_direct_halo_toggle_matches():
    """A direct thread world switched to message exchange and back
    (lbcu_world_set_direct, as bench.py's IPC/NCCL cross-check does) gives
    the same decomposed Dphi bit for bit in every mode."""
    L, grid = [8, 4, 4, 8], (2, 1, 1, 2)
    n, rep = 2, lb.FUNDAMENTAL
    dr, g, s = fields(L, n, rep)
    world = lb.World.threads(4, direct=True)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        idx = global_index(L, grid, r)
        gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g[idx])
        inp = lb.SpinorField(ctx, dr).upload(s[idx])
        out = lb.SpinorField(ctx, dr)
        res = []
        for mode in (True, False, True):
            ctx.barrier()
            if r == 0:
                world.set_direct(mode)
            ctx.barrier()
            lb.apply_dirac(out, gauge, inp, 0.1)
            res.append(out.download())
        return res

    for res in run_ranks(4, body):
        assert np.array_equal(res[0], res[1]) and np.array_equal(res[0], res[2])


def test_tma_rowblock_dphi_matches_oracle(monkeypatch):
    """The TMA-staged row-block full Dphi (experiment, LBCU_HOP_RB=1; DESIGN
    §4: correct but 8 % slower than the default kernel): persistent blocks,
    cp.async.bulk tiles completed on an mbarrier, double-buffered."""
    monkeypatch.setenv("LBCU_HOP_RB", "1")
    L = [4, 6, 16, 32]
    dr, g, s = fields(L, 2, lb.FUNDAMENTAL)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, 2, lb.FUNDAMENTAL, lb.ANTIPERIODIC_T).upload(g)
    a, b = lb.SpinorField(ctx, dr).upload(s), lb.SpinorField(ctx, dr)
    lb.apply_dirac(b, gauge, a, 0.1)
    assert gauge.storage()[0] == "su2"
    assert rel_l2(b.download(), O.port_dirac(L, 1, 0.1, g, s)) < 1e-13


@pytest.mark.parametrize("n,rep,L", [(3, lb.FUNDAMENTAL, [4, 4, 8, 8]), (2, lb.FUNDAMENTAL, [4, 4, 8, 8]),
                                      (2, lb.ADJOINT, [4, 6, 16, 4])], ids=["su3f", "su2f", "su2a"])
def test_block_shape_and_link_staging_knobs_are_bit_identical(monkeypatch, n, rep, L):
    """The default full Dphi runs mixed-parity blocks (LBCU_HOP_MIX) and, for
    SU(3) links, stages the forward link tiles of each warp in shared memory
    with bulk async copies (LBCU_HOP_LS; lattices whose x-planes hold whole
    32-site tiles). Both only change where operands come from: the output is
    bit-identical with either switched off, and matches the oracle."""
    dr, g, s = fields(L, n, rep)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g)
    a = lb.SpinorField(ctx, dr).upload(s)
    ae = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    outs = []
    for mix, ls in (("1", "1"), ("0", "1"), ("1", "0"), ("0", "0")):
        monkeypatch.setenv("LBCU_HOP_MIX", mix)
        monkeypatch.setenv("LBCU_HOP_LS", ls)
        b, bo = lb.SpinorField(ctx, dr), lb.SpinorField(ctx, dr, lb.ODD)
        lb.apply_dirac(b, gauge, a, 0.1)
        lb.dphi_oe(bo, gauge, ae)
        outs.append((b.download(), bo.download()))
    for full, hop in outs[1:]:
        assert np.array_equal(full, outs[0][0]) and np.array_equal(hop, outs[0][1])
    assert rel_l2(outs[0][0], O.port_dirac(L, 1, 0.1, g, s)) < TOL_DPHI


EXTRA_REPS = [(3, lb.SYMMETRIC), (4, lb.FUNDAMENTAL), (3, lb.ADJOINT), (4, lb.SYMMETRIC), (6, lb.FUNDAMENTAL)]


@pytest.mark.parametrize("n,rep", EXTRA_REPS, ids=["su3s", "su4f", "su3a", "su4s", "su6f"])
def test_other_representations_match_oracle(n, rep):
    """Every other device specialisation (dense links: dr 4, 6, 8 real, 10):
    Dphi and Mhat against the oracle, eo CG against the reference-composed
    solver."""
    L = [4, 4, 4, 4]
    ctx, dr, g, s, gauge = setup(L, n, rep)
    out = lb.SpinorField(ctx, dr)
    lb.apply_dirac(out, gauge, lb.SpinorField(ctx, dr).upload(s), 0.1)
    assert rel_l2(out.download(), O.port_dirac(L, 1, 0.1, g, s)) < TOL_DPHI
    me = lb.SpinorField(ctx, dr, lb.EVEN)
    lb.mhat(me, gauge, lb.SpinorField(ctx, dr, lb.EVEN).upload(s), 0.1)
    assert rel_l2(me.download(), O.port_mhat(L, 1, 0.1, g, s)) < TOL_DPHI
    o = lb.cg_solve_eo(gauge, 0.1, lb.SpinorField(ctx, dr, lb.EVEN).upload(s), lb.CgSettings(1e-10, 1000))
    ref = O.ref_cg_eo(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s, 1e-10)
    assert abs(o.iterations - ref["iterations"]) <= 1 and o.true_rel_residual < 2e-10


@pytest.mark.parametrize("n,rep", EXTRA_REPS, ids=["su3s", "su4f", "su3a", "su4s", "su6f"])
def test_other_representations_decomposed(n, rep):
    """Halo pack (dense links of every size, real and complex) and boundary
    kernels for the remaining specialisations: 2x1x1x2 thread ranks with
    direct halos against the serial oracle."""
    L, grid = [8, 4, 4, 8], (2, 1, 1, 2)
    dr, g, s = fields(L, n, rep)
    want = O.port_dirac(L, 1, 0.1, g, s)
    world = lb.World.threads(4, direct=True)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        idx = global_index(L, grid, r)
        gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g[idx])
        out = lb.SpinorField(ctx, dr)
        lb.apply_dirac(out, gauge, lb.SpinorField(ctx, dr).upload(s[idx]), 0.1)
        return idx, out.download()

    got = np.empty_like(want)
    for idx, part in run_ranks(4, body):
        got[idx] = part
    assert rel_l2(got, want) < 1e-14


def test_dphi_host_pipeline_distinct_fields():
    """lbcu_dphi_host over 5 distinct host fields (two device slots reused
    through the copy/compute pipeline): every output is the Dphi of its own
    input (reference layout both ways)."""
    L, n, rep, m = [4, 4, 4, 8], 2, lb.FUNDAMENTAL, 0.1
    ctx, dr, g, s, gauge = setup(L, n, rep)
    ins = [np.ascontiguousarray(lb.init_spinor_random(L, dr, 1, k)) for k in range(5)]
    outs = [np.zeros_like(x) for x in ins]
    lb.dphi_host(gauge, m, [x.ctypes.data for x in ins], [y.ctypes.data for y in outs])
    for x, y in zip(ins, outs):
        assert rel_l2(y, O.port_dirac(L, 1, m, g, x)) < TOL_DPHI
