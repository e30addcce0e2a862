"""The NCCL transport on one GPU: dlopen of libnccl, communicator creation from
a unique id, and the operator/solver paths running through it. (Multi-rank
NCCL needs several GPUs; the decomposed kernels are covered by the thread
transport in test_gpu_parity.py and the exchange schedule in test_host.py.)"""
import pytest

import oracle as O
import paper_1401_3733_b200 as lb
from helpers import rel_l2

pytestmark = pytest.mark.gpu


def test_single_rank_nccl_world_runs_dphi_and_cg():
    uid = lb.World.nccl_unique_id()
    assert len(uid) == 128
    world = lb.World.nccl(1, 0, uid)
    L = [8, 4, 4, 4]
    ctx = lb.Context(L, (1, 1, 1, 1), 0, 0, world)
    g = lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1)
    s = lb.init_spinor_random(L, 3, 1, 0)
    gauge = lb.GaugeField(ctx, 3, lb.FUNDAMENTAL, lb.ANTIPERIODIC_T).upload(g)
    a, b = lb.SpinorField(ctx, 3).upload(s), lb.SpinorField(ctx, 3)
    lb.apply_dirac(b, gauge, a, 0.1)
    assert rel_l2(b.download(), O.port_dirac(L, 1, 0.1, g, s)) < 1e-12
    o = lb.cg_solve_eo(gauge, 0.1, lb.SpinorField(ctx, 3, lb.EVEN).upload(s), lb.CgSettings(1e-10, 500))
    ref = O.port_cg(L, 1, 1, 0.1, g, s, 1e-10)
    assert abs(o.iterations - ref["iterations"]) <= 1 and o.true_rel_residual < 2e-10
    ctx.barrier()


def test_world_size_must_match_grid():
    world = lb.World.threads(2)
    with pytest.raises(lb.ContractViolation):
        lb.Context([8, 4, 4, 4], (1, 1, 1, 1), 0, 0, world)
