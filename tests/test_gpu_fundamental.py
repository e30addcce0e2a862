"""SU(4) antisymmetric links uploaded as fundamental elements, stored either
as real SO(6) matrices in the real basis (LBCU_GAUGE_AS4R, default) or as the
fundamental elements with the minors formed in-kernel (LBCU_GAUGE_AS4,
LBCU_AS4_STORAGE=fund), against the oracle on the reference's represented
links."""
import numpy as np
import pytest

import oracle as O
import paper_1401_3733_b200 as lb
from helpers import global_index, rel_l2, run_ranks

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["as4r", "as4"])
def storage(request, monkeypatch):
    if request.param == "as4":
        monkeypatch.setenv("LBCU_AS4_STORAGE", "fund")
    else:
        monkeypatch.delenv("LBCU_AS4_STORAGE", raising=False)
    return request.param


@pytest.mark.parametrize("bc", [lb.PERIODIC, lb.ANTIPERIODIC_T], ids=["periodic", "antiperiodic"])
def test_as4_dphi_eo_and_download(bc, storage):
    L = [4, 4, 6, 4]
    fund = lb.init_gauge_random(L, 4, lb.FUNDAMENTAL, 1)
    rep = lb.init_gauge_random(L, 4, lb.ANTISYMMETRIC, 1)  # represent() of the same elements
    s = lb.init_spinor_random(L, 6, 1, 0)
    ctx = lb.Context(L)
    g = lb.GaugeField(ctx, 4, lb.ANTISYMMETRIC, bc).upload_fundamental(fund)
    assert g.storage()[0] == storage
    assert np.abs(g.download() - rep).max() < 1e-14
    inp, out = lb.SpinorField(ctx, 6).upload(s), lb.SpinorField(ctx, 6)
    lb.apply_dirac(out, g, inp, 0.1)
    assert rel_l2(out.download(), O.port_dirac(L, bc, 0.1, rep, s)) < 1e-12
    e_in, e_out = lb.SpinorField(ctx, 6, lb.EVEN).upload(s), lb.SpinorField(ctx, 6, lb.EVEN)
    lb.mhat(e_out, g, e_in, 0.1)
    assert rel_l2(e_out.download(), O.port_mhat(L, bc, 0.1, rep, s)) < 1e-12


def test_as4_cg_eo_matches_reference(storage):
    L = [8, 4, 4, 4]
    fund = lb.init_gauge_random(L, 4, lb.FUNDAMENTAL, 1)
    rep = lb.init_gauge_random(L, 4, lb.ANTISYMMETRIC, 1)
    s = lb.init_spinor_random(L, 6, 1, 0)
    ctx = lb.Context(L)
    g = lb.GaugeField(ctx, 4, lb.ANTISYMMETRIC, lb.ANTIPERIODIC_T).upload_fundamental(fund)
    o = lb.cg_solve_eo(g, 0.1, lb.SpinorField(ctx, 6, lb.EVEN).upload(s), lb.CgSettings(1e-10, 500))
    ref = O.ref_cg_eo(L, [1, 1, 1, 1], 4, O.ANTISYMMETRIC, 1, 0.1, rep, s, 1e-10)
    assert abs(o.iterations - ref["iterations"]) <= 1 and o.true_rel_residual < 2e-10


def test_as4_decomposed_matches_serial(storage):
    L = [8, 4, 4, 4]
    fund = lb.init_gauge_random(L, 4, lb.FUNDAMENTAL, 1)
    rep = lb.init_gauge_random(L, 4, lb.ANTISYMMETRIC, 1)
    s = lb.init_spinor_random(L, 6, 1, 0)
    want = O.port_dirac(L, 1, 0.1, rep, s)
    grid = (2, 1, 1, 1)
    world = lb.World.threads(2)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        idx = global_index(L, grid, r)
        g = lb.GaugeField(ctx, 4, lb.ANTISYMMETRIC, lb.ANTIPERIODIC_T).upload_fundamental(fund[idx])
        inp, out = lb.SpinorField(ctx, 6).upload(s[idx]), lb.SpinorField(ctx, 6)
        lb.apply_dirac(out, g, inp, 0.1)
        return idx, out.download()

    got = np.empty_like(want)
    for idx, part in run_ranks(2, body):
        got[idx] = part
    assert rel_l2(got, want) < 1e-13


def test_fundamental_upload_rejects_other_reps():
    ctx = lb.Context([4, 4, 4, 4])
    g = lb.GaugeField(ctx, 3, lb.FUNDAMENTAL, lb.PERIODIC)
    with pytest.raises(lb.ConfigError):
        g.upload_fundamental(np.zeros((256, 4, 3, 3), np.complex128))


def test_dense_as_upload_compacts_to_real_basis():
    """Dense represented AS links (reference layout) compress to AS4R; links
    that are not SU(4) images stay exact: dense, or AS4 for fundamentals."""
    L = [4, 4, 4, 4]
    rep = lb.init_gauge_random(L, 4, lb.ANTISYMMETRIC, 1)
    s = lb.init_spinor_random(L, 6, 1, 0)
    ctx = lb.Context(L)
    g = lb.GaugeField(ctx, 4, lb.ANTISYMMETRIC, lb.ANTIPERIODIC_T).upload(rep)
    assert g.storage()[0] == "as4r" and g.storage()[1] < 1e-13
    a, b = lb.SpinorField(ctx, 6).upload(s), lb.SpinorField(ctx, 6)
    lb.apply_dirac(b, g, a, 0.1)
    assert rel_l2(b.download(), O.port_dirac(L, 1, 0.1, rep, s)) < 1e-12
    bad = rep.copy()
    bad[0, 0, 0, 0] += 0.25j
    g.upload(bad)
    assert g.storage()[0] == "full"
    assert np.array_equal(g.download(), bad)
    fund = lb.init_gauge_random(L, 4, lb.FUNDAMENTAL, 1)
    fund[3, 1] *= 1 + 0.5j  # not an SU(4) element: R picks up a complex factor
    g.upload_fundamental(fund)
    assert g.storage()[0] == "as4"
