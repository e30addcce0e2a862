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


@pytest.mark.parametrize("nranks,config", [(2, 1), (4, 2)])
def test_bench_multirank_emulated(nranks, config):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nranks), os.path.join(ROOT, "bench.py"),
           "--gpus", str(nranks), "--steps", "3", "--warmup", "3", "--config", str(config), "--emulate", "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == nranks
    assert line["config"]["halo_transport"].startswith("ipc")
    assert line["cg"]["iterations"] == 23 and line["cg"]["true_rel_residual"] < 2e-10
    assert line["e2e"]["check_rel_err"] == 0.0
    assert line["value"] > 0
