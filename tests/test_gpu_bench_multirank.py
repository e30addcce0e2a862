"""bench.py's N > 1 flow (torchrun, decomposition, IPC world with direct
halos, decomposed CG, end-to-end host path) run with every rank on the one
GPU of the test box (--emulate: gloo for the Python-side collectives, host CG
sums; nothing waits on another rank inside a kernel). Correctness only."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench_tol(c):
    import bench
    return bench.CONFIGS[c]["tol"]


@pytest.mark.parametrize("nranks,config,table", [(2, 1, True), (4, 2, False)])
def test_bench_multirank_emulated(nranks, config, table):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nranks), os.path.join(ROOT, "bench.py"),
           "--gpus", str(nranks), "--steps", "3", "--warmup", "3", "--config", str(config), "--emulate", "--no-cpu"]
    if not table:
        cmd.append("--no-all-configs")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == nranks
    assert line["halo_transport"].startswith("ipc")
    assert line["cg"]["eo"]["iterations"] == 23 and line["cg"]["eo"]["true_rel_residual"] < 2e-10
    assert abs(line["cg"]["plain"]["iterations"] - (47 if config == 1 else 48)) <= 1
    assert line["roofline"]["traffic"] is None  # single-GPU ncu bytes are not a rank's
    if table:
        assert sorted(line["configs"]) == ["1", "2", "3", "4", "5"]
        for c, row in line["configs"].items():
            assert row["eo_cg"]["true_rel_residual"] < 2 * bench_tol(int(c))
    assert line["e2e"]["check_rel_err"] == 0.0
    assert line["value"] > 0
