"""bench.py: the N > 1 flow (torchrun, decomposition, IPC world with direct
halos, decomposed CG, end-to-end host path) run with every rank on the one
GPU of the test box (--emulate: gloo for the Python-side collectives, host CG
sums; nothing waits on another rank inside a kernel; correctness only), the
one-GPU bench line and a stock-regime line."""
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
    assert line["cg"]["eo"]["e2e"]["iterations"] == 23 and line["cg"]["eo"]["e2e"]["seconds"] > 0
    assert line["roofline"]["traffic"] is None  # single-GPU ncu bytes are not a rank's
    if table:
        assert sorted(line["configs"]) == ["1", "2", "3", "4", "5"]
        for c, row in line["configs"].items():
            assert row["eo_cg"]["true_rel_residual"] < 2 * bench_tol(int(c))
    assert line["e2e"]["check_rel_err"] == 0.0
    assert line["value"] > 0


def test_bench_single_gpu_line():
    """The one-GPU bench line carries every key the driver reads (value,
    roofline with the kernel's launch count, e2e with the copied bytes and the
    PCIe bound, CPU baseline with the reference CG, clocks, per-config table)."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "2", "--steps", "5", "--warmup", "3",
           "--cpu-seconds", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] == 5
    assert line["config"]["workload"].startswith("cfg2") and line["dtype"] == "f64"
    rf = line["roofline"]
    assert rf["bound"] == "hbm" and 0 < rf["frac"] < 1.2 and rf["kernels_per_step"] == 1.0
    assert line["e2e"]["h2d_bytes_per_step"] == 32 ** 4 * 4 * 2 * 16 and line["e2e"]["check_rel_err"] < 1e-15
    assert line["cg"]["eo"]["iterations"] == 23 and line["cg"]["plain"]["iterations"] == 48
    assert line["cg"]["eo"]["e2e"]["seconds"] >= line["cg"]["eo"]["seconds"]
    cpu = line["cpu_baseline"]
    assert cpu["kind"] == "reference" and cpu["value"] > 0 and cpu["cores"] >= 1
    assert cpu["cg"]["eo"]["iterations"] == 23 and cpu["cg"]["plain"]["iterations"] == 48
    assert sorted(line["configs"]) == ["1", "2", "3", "4", "5"]
    assert all(row["cpu_reference_gflops"] > 0 for row in line["configs"].values())
    assert "sm_mhz" in line["clocks"]


def test_bench_regime_line():
    """bench.py --regime: a stock regime at 64x32^3 with the GPU Dphi checked
    against the unmodified reference apply_dirac on the same host inputs."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--regime", "comms", "--steps", "5", "--warmup", "3",
           "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["regime"] == "comms" and line["config"]["lattice_TXYZ"] == [64, 32, 32, 32]
    assert line["parity_vs_reference_rel_l2"] < 1e-12
    assert line["cg"]["eo"]["iterations"] > 0 and line["cg"]["eo"]["true_rel_residual"] < 2e-10
    assert line["value"] > 0 and line["roofline"]["frac"] > 0
