"""Ragged geometries on the GPU: checkerboard volumes that are not a multiple
of the 32-site tile (padded last tile), z-rows of odd cb length that straddle
tiles, extent-2 directions (both neighbours are the same site), and a
decomposition whose local blocks are ragged too. Every representation,
against the oracle / the unmodified reference."""
import numpy as np
import pytest

import oracle as O
import paper_1401_3733_b200 as lb
from helpers import REP_IDS, REPS, global_index, rel_l2, run_ranks

pytestmark = pytest.mark.gpu

SHAPES = [[6, 2, 10, 6], [2, 6, 2, 14], [10, 2, 2, 2]]  # vh = 360, 168, 40


@pytest.mark.parametrize("L", SHAPES, ids=["x".join(map(str, s)) for s in SHAPES])
@pytest.mark.parametrize("n,rep", REPS, ids=REP_IDS)
def test_ragged_operators(L, n, rep):
    dr = lb.rep_dim(rep, n)
    g = lb.init_gauge_random(L, n, rep, 1)
    s = lb.init_spinor_random(L, dr, 1, 0)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g)
    a, b = lb.SpinorField(ctx, dr).upload(s), lb.SpinorField(ctx, dr)
    lb.apply_dirac(b, gauge, a, 0.1)
    assert rel_l2(b.download(), O.ref_apply_dirac(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s)) < 1e-12
    # round trips through the tiled layout leave the padding untouched
    assert np.array_equal(a.download(), s)
    assert np.array_equal(gauge.download(), g) or gauge.storage()[0] != "full"
    ae = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    me = lb.SpinorField(ctx, dr, lb.EVEN)
    lb.mhat(me, gauge, ae, 0.1)
    assert rel_l2(me.download(), O.ref_mhat(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s)) < 1e-12
    # norms see no padding
    assert abs(lb.sqnorm(a) - O.ref_sqnorm(L, [1, 1, 1, 1], s)) < 1e-12 * O.ref_sqnorm(L, [1, 1, 1, 1], s)
    o = lb.cg_solve_eo(gauge, 0.1, ae, lb.CgSettings(1e-10, 1000))
    ref = O.ref_cg_eo(L, [1, 1, 1, 1], n, rep, 1, 0.1, g, s, 1e-10)
    assert abs(o.iterations - ref["iterations"]) <= 1 and o.true_rel_residual < 2e-10


@pytest.mark.parametrize("n,rep", [REPS[0], REPS[2]], ids=[REP_IDS[0], REP_IDS[2]])
def test_ragged_decomposed(n, rep):
    L, grid = [12, 2, 6, 10], (2, 1, 1, 1)  # local 6x2x6x10: vh = 360
    dr = lb.rep_dim(rep, n)
    g = lb.init_gauge_random(L, n, rep, 1)
    s = lb.init_spinor_random(L, dr, 1, 0)
    want = O.port_dirac(L, 1, 0.1, g, s)
    world = lb.World.threads(2)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        idx = global_index(L, grid, r)
        gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g[idx])
        out = lb.SpinorField(ctx, dr)
        lb.apply_dirac(out, gauge, lb.SpinorField(ctx, dr).upload(s[idx]), 0.1)
        return idx, out.download()

    got = np.empty_like(want)
    for idx, part in run_ranks(2, body):
        got[idx] = part
    assert rel_l2(got, want) < 1e-14
