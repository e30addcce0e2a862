"""On-device keyed field generation against the host
generators (bit-identical to the reference, tests/test_host.py)."""
import numpy as np
import pytest

import oracle as O
import paper_1401_3733_b200 as lb
from helpers import global_index, rel_l2, run_ranks

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dr", [2, 3, 6])
def test_spinor_generate_matches_host(dr):
    L = [4, 4, 6, 8]
    ctx = lb.Context(L)
    s = lb.SpinorField(ctx, dr).randomize(7, 3)
    host = lb.init_spinor_random(L, dr, 7, 3)
    assert np.abs(s.download() - host).max() < 1e-13
    e = lb.SpinorField(ctx, dr, lb.EVEN).randomize(7, 3)
    even = O.parity_mask(L)
    got = e.download()
    assert np.abs(got[even] - host[even]).max() < 1e-13 and not np.any(got[~even])


@pytest.mark.parametrize("n,rep,links,fmt", [
    (2, lb.FUNDAMENTAL, lb.LINKS_HAAR, "su2"),
    (3, lb.FUNDAMENTAL, lb.LINKS_HAAR, "r10"),
    (3, lb.FUNDAMENTAL, lb.LINKS_NEAR_UNIT, "r10"),
    (2, lb.ADJOINT, lb.LINKS_HAAR, "su2"),
    (4, lb.ANTISYMMETRIC, lb.LINKS_HAAR, "as4r"),
    (4, lb.FUNDAMENTAL, lb.LINKS_HAAR, "full"),
    (3, lb.FUNDAMENTAL, lb.LINKS_UNIT, "r10"),
], ids=["su2f", "su3f", "su3f-near-unit", "su2a", "su4as", "su4f", "unit"])
def test_gauge_generate_matches_host(n, rep, links, fmt):
    L = [4, 4, 4, 6]
    ctx = lb.Context(L)
    g = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).generate(1, links=links, eps=0.3)
    assert g.storage()[0] == fmt
    host = lb.init_gauge_random(L, n, rep, 1, links=links, eps=0.3)
    assert np.abs(g.download() - host).max() < 1e-12
    # and the operator built on it matches the oracle on the host links
    dr = lb.rep_dim(rep, n)
    s = lb.init_spinor_random(L, dr, 1, 0)
    a, b = lb.SpinorField(ctx, dr).randomize(1, 0), lb.SpinorField(ctx, dr)
    lb.apply_dirac(b, g, a, 0.1)
    assert rel_l2(b.download(), O.port_dirac(L, 1, 0.1, host, s)) < 1e-12


def test_generation_is_decomposition_invariant():
    L = [8, 4, 4, 8]
    grid = (2, 1, 1, 2)
    host = lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1)
    world = lb.World.threads(4)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        g = lb.GaugeField(ctx, 3, lb.FUNDAMENTAL, lb.PERIODIC).generate(1)
        return global_index(L, grid, r), g.download()

    for idx, part in run_ranks(4, body):
        assert np.abs(part - host[idx]).max() < 1e-12
