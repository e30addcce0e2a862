"""One rank of the two-process IPC-world test (tests/test_gpu_ipc.py); test
infrastructure. usage: python tests/ipc_worker.py RANK NRANKS SHM_NAME OUT.npz"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_3733_b200 as lb  # noqa: E402


def main():
    rank, nranks, name, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    L, grid, n, rep, m = [8, 4, 4, 8], [nranks, 1, 1, 1], 2, lb.FUNDAMENTAL, 0.1
    dr = lb.rep_dim(rep, n)
    world = lb.World.ipc(nranks, rank, name)
    ctx = lb.Context(L, grid, rank, 0, world)
    g = lb.init_gauge_random(L, n, rep, 1, grid=grid, rank=rank)
    s = lb.init_spinor_random(L, dr, 1, 0, grid=grid, rank=rank)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g)
    a = lb.SpinorField(ctx, dr).upload(s)
    b = lb.SpinorField(ctx, dr)
    lb.apply_dirac(b, gauge, a, m)
    d1 = b.download()
    for _ in range(5):  # several exchanges: both arena / event slots reused
        lb.apply_dirac(b, gauge, a, m)
    rhs = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    o = lb.cg_solve_eo(gauge, m, rhs, lb.CgSettings(1e-10, 500))
    np.savez(out, dphi=d1, dphi6=b.download(), its=o.iterations, tr=o.true_rel_residual,
             x=o.solution.download())
    ctx.barrier()  # no rank unmaps an arena while a peer still stores into it
    ctx.close()
    world.close()


if __name__ == "__main__":
    main()
