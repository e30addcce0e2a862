"""The multi-rank flow of bench.py, with ranks as host threads on one GPU
(thread transport; NCCL needs one GPU per rank): device-generated links,
host-buffer Dphi (lbcu_dphi_host), eo hop and eo CG, each against the serial
result."""
import numpy as np
import pytest

import bench
import oracle as O
import paper_1401_3733_b200 as lb
from helpers import global_index, rel_l2, run_ranks

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks", [2, 4])
def test_bench_flow_decomposed(nranks):
    L = [16, 4, 4, 8]
    n, rep, mass = 2, lb.FUNDAMENTAL, 0.05
    grid = bench.decompose(L, nranks)
    assert int(np.prod(grid)) == nranks
    g = lb.init_gauge_random(L, n, rep, 1)
    s = lb.init_spinor_random(L, 2, 1, 0)
    want = O.port_dirac(L, 1, mass, g, s)
    even = O.parity_mask(L)
    s_even = s.copy()
    s_even[~even] = 0
    want_hop = O.port_hop_parity(L, 1, 1, -0.5, g, s_even)
    ref_cg = O.port_cg(L, 1, 1, mass, g, s, 1e-10)
    world = lb.World.threads(nranks)

    def body(r):
        ctx = lb.Context(L, grid, r, 0, world)
        idx = global_index(L, grid, r)
        gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).generate(1)
        local = lb.init_spinor_random(L, 2, 1, 0, grid=grid, rank=r)
        out = np.empty_like(local)
        lb.dphi_host(gauge, mass, [local.ctypes.data] * 2, [out.ctypes.data] * 2)
        ae = lb.SpinorField(ctx, 2, lb.EVEN).upload(local)
        bo = lb.SpinorField(ctx, 2, lb.ODD)
        lb.dphi_oe(bo, gauge, ae)
        o = lb.cg_solve_eo(gauge, mass, ae, lb.CgSettings(1e-10, 500))
        return idx, out, bo.download(), o.iterations, o.true_rel_residual

    got, hop = np.empty_like(want), np.empty_like(want)
    for idx, out, h, it, tr in run_ranks(nranks, body):
        got[idx] = out
        hop[idx] = h
        assert abs(it - ref_cg["iterations"]) <= 1 and tr < 2e-10
    assert rel_l2(got, want) < 1e-12
    assert rel_l2(hop, want_hop) < 1e-12

