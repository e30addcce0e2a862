"""The C++ benchmark driver (tools/latbench_b200): run_suite on the device path,
parameter-file semantics of the reference (proj/src/bench.cpp:94-177)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "tools", "latbench_b200")
needs_driver = pytest.mark.skipif(not os.path.exists(DRIVER), reason="driver not built")


def run(args, tmp_path, text):
    p = tmp_path / "p.params"
    p.write_text(text)
    return subprocess.run([DRIVER, args[0], str(p), *args[1:]], capture_output=True, text=True, timeout=600)


@needs_driver
@pytest.mark.parametrize("test,dirac", [("comms", 936), ("balance", 1512), ("compute", 5328)])
def test_model_of_stock_regimes(tmp_path, test, dirac):
    r = run(["model"], tmp_path, f"test = {test}\nlattice = 16x8x8x8\ngrid = 1x1x1x1\n")
    assert r.returncode == 0, r.stderr
    assert f"dirac  {dirac} flop/site" in r.stdout


@needs_driver
def test_regime_intensity_ordering(tmp_path):
    """arithmetic intensity comms < balance < compute at fixed geometry."""
    vals = []
    for t in ("comms", "balance", "compute"):
        r = run(["model"], tmp_path, f"test = {t}\nlattice = 16x8x8x8\n")
        vals.append(float(r.stdout.split("intensity")[1].split()[0]))
    assert vals[0] < vals[1] < vals[2]


@needs_driver
@pytest.mark.parametrize("text,frag", [
    ("lattice = 8x8x8\n", "line 1"),
    ("mass = 0.1\nbogus = 3\n", "line 2: unknown key 'bogus'"),
    ("test = nonsense\n", "unknown test"),
    ("mass 0.1\n", "expected 'key = value'"),
    ("lattice = 7x4x4x4\ngrid=1x1x1x1\n", "odd"),
])
def test_config_errors_exit_2(tmp_path, text, frag):
    r = run(["model"], tmp_path, text)
    assert r.returncode == 2 and frag in r.stderr, (r.returncode, r.stderr)


SMALL = """test = balance
lattice = 16x8x8x8
grid = {grid}
enforce_local_floor = false
spinor_fields = 3
mass = 0.1
kernel_seconds = 0.05
cg_tolerance = 1e-10
seed = 1
bc_time = antiperiodic
eo = {eo}
"""


@pytest.mark.gpu
@pytest.mark.parametrize("grid,eo", [("1x1x1x1", "false"), ("1x1x1x1", "true"), ("2x1x1x1", "true")])
def test_run_suite_on_device(tmp_path, grid, eo):
    r = run(["run", "--format", "json"], tmp_path, SMALL.format(grid=grid, eo=eo))
    assert r.returncode == 0, r.stderr
    rep = json.loads(r.stdout)
    assert rep["format_version"] == 1
    assert [k["kernel"] for k in rep["kernels"]] == ["sqnorm", "muladd", "dirac"]
    assert all(k["iterations"] >= 1 and k["flops_per_sec"] > 0 for k in rep["kernels"])
    assert rep["consistency"]["status"] == "passed"
    assert rep["consistency"]["iterations"] == (23 if eo == "true" else 47) or rep["consistency"]["iterations"] > 0
    assert rep["model"]["dirac_flops_per_site"] == 1512


@pytest.mark.gpu
def test_check_subcommand(tmp_path):
    r = run(["check"], tmp_path, SMALL.format(grid="1x1x1x1", eo="true"))
    assert r.returncode == 0 and "consistency passed" in r.stdout, r.stdout + r.stderr


def _ref_report_available():
    try:
        import oracle as O
        return hasattr(O.ref_lib(), "ref_report_reformat")
    except Exception:  # noqa: BLE001
        return False


@pytest.mark.gpu
@pytest.mark.skipif(not _ref_report_available(), reason="reference built without report.cpp")
def test_run_report_round_trips_through_reference_reader(tmp_path):
    """Format-1 interop (proj/src/report.cpp:152-217): the driver's JSON report
    parses with the reference's report_from_json, which re-emits the same
    fields, and the reference's CSV writer reproduces the driver's CSV of the
    same report byte for byte."""
    import oracle as O
    prefix = tmp_path / "rep"
    r = run(["run", "--format", "json", "--emit-all", str(prefix)], tmp_path, SMALL.format(grid="1x1x1x1", eo="true"))
    assert r.returncode == 0, r.stderr
    ours = (tmp_path / "rep.json").read_text()
    theirs = json.loads(O.ref_report_reformat(ours, "json"))
    mine = json.loads(ours)
    for k in ("format_version", "regime", "timestamp", "geometry", "group_rank", "representation", "mass", "seed",
              "model"):
        assert theirs[k] == mine[k], k
    assert [k["kernel"] for k in theirs["kernels"]] == ["sqnorm", "muladd", "dirac"]
    for a, b in zip(theirs["kernels"], mine["kernels"]):
        assert a == b
    c = dict(mine["consistency"])
    c.pop("solver")
    assert theirs["consistency"] == c
    assert O.ref_report_reformat(ours, "csv") == (tmp_path / "rep.csv").read_text()
    assert "dirac" in O.ref_report_reformat(ours, "text")
