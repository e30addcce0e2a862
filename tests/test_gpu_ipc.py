"""The IPC world (lbcu_world_ipc): one process per rank, halo records stored
by the pack kernel straight into the peer's arena through CUDA IPC mappings,
an interprocess event per exchange and a host barrier in POSIX shared memory.
Two processes on the one GPU of the test box (no kernel waits on another
rank, so sharing a GPU is safe); compared with the serial oracle."""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

import oracle as O
import paper_1401_3733_b200 as lb
from helpers import global_index, rel_l2

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_ipc_world_two_processes(tmp_path):
    L, grid, n, rep, m = [8, 4, 4, 8], [2, 1, 1, 1], 2, lb.FUNDAMENTAL, 0.1
    name = f"/lbcu_test_{uuid.uuid4().hex[:12]}"
    outs = [str(tmp_path / f"r{r}.npz") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "ipc_worker.py"), str(r), "2", name, outs[r]],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(2)]
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log
    dr = lb.rep_dim(rep, n)
    g = lb.init_gauge_random(L, n, rep, 1)
    s = lb.init_spinor_random(L, dr, 1, 0)
    want = O.port_dirac(L, 1, m, g, s)
    ref = O.ref_cg_eo(L, [1, 1, 1, 1], n, rep, 1, m, g, s, 1e-10)
    got, got6, x = np.empty_like(want), np.empty_like(want), np.empty_like(s)
    for r in range(2):
        d = np.load(outs[r])
        idx = global_index(L, grid, r)
        got[idx] = d["dphi"]
        got6[idx] = d["dphi6"]
        x[idx] = d["x"]
        assert abs(int(d["its"]) - ref["iterations"]) <= 1
        assert float(d["tr"]) < 2e-10
    assert rel_l2(got, want) < 1e-14
    assert np.array_equal(got, got6)
    assert rel_l2(x, ref["x"]) < 1e-8


def test_ipc_world_single_rank_rules():
    """A one-rank IPC world runs undecomposed; without NCCL its halos cannot
    be switched to message exchange."""
    name = f"/lbcu_test_{uuid.uuid4().hex[:12]}"
    w = lb.World.ipc(1, 0, name)
    with pytest.raises(lb.TransportError):
        w.set_direct(False)
    ctx = lb.Context([4, 4, 4, 4], (1, 1, 1, 1), 0, 0, w)
    g = lb.init_gauge_random([4, 4, 4, 4], 2, lb.FUNDAMENTAL, 1)
    s = lb.init_spinor_random([4, 4, 4, 4], 2, 1, 0)
    gauge = lb.GaugeField(ctx, 2, lb.FUNDAMENTAL, lb.ANTIPERIODIC_T).upload(g)
    a, b = lb.SpinorField(ctx, 2).upload(s), lb.SpinorField(ctx, 2)
    lb.apply_dirac(b, gauge, a, 0.1)
    assert rel_l2(b.download(), O.port_dirac([4, 4, 4, 4], 1, 0.1, g, s)) < 1e-13
    ctx.close()
    w.close()
