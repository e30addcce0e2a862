"""Pin the CPU oracle (oracle/oracle.c) against the reference and the golden
fixtures (tests/golden/, generated from the unmodified reference by
make_golden.py). CPU only."""
import hashlib
import os

import numpy as np
import pytest

import oracle as O
from helpers import rel_l2

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = ["su3f", "su2f", "su2a", "su4as", "su3s"]
HAVE_REF = os.path.exists(O.REF_SO) and os.path.exists(O.REF_EXACT_SO)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (needs /root/reference)")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def golden(name):
    return np.load(os.path.join(GOLD, f"{name}.npz"))


def port_inputs(d):
    L, n, rep = list(d["lattice"]), int(d["n"]), int(d["rep"])
    dr = O.rep_dim(rep, n)
    return L, n, rep, dr


@pytest.mark.parametrize("name", CASES)
def test_port_reproduces_golden_bitwise(name):
    """The C restatement reproduces the FMA-free reference outputs bit for bit."""
    d = golden(name)
    L, n, rep, dr = port_inputs(d)
    s = O.port_spinor_random(L, dr, 1, 0)
    assert sha(s) == str(d["spinor_sha"])
    # gauge fixtures are pinned through the product generator in test_host.py;
    # here they come from the reference when available, else from the product
    if HAVE_REF:
        with O.exact_reference():
            g = O.ref_gauge_random(L, n, rep, 1)
    else:
        import paper_1401_3733_b200 as lb
        g = lb.init_gauge_random(L, n, rep, 1)
    assert sha(g) == str(d["gauge_sha"])
    m = float(d["mass"])
    assert np.array_equal(O.port_dirac(L, 0, m, g, s), d["dphi_periodic"])
    assert np.array_equal(O.port_dirac(L, 1, m, g, s), d["dphi_antiperiodic"])
    # Mhat: the reference composition hop = (4+m)psi - D psi rounds differently
    assert rel_l2(O.port_mhat(L, 1, m, g, s), d["mhat_antiperiodic"]) < 1e-14


def test_cfg1_golden_cg_counts():
    """BASELINE config 1: reference plain CG 47 iterations, eo oracle 23."""
    d = golden("cfg1")
    L = list(d["lattice"])
    s = O.port_spinor_random(L, 3, 1, 0)
    assert sha(s) == str(d["spinor_sha"])
    import paper_1401_3733_b200 as lb
    g = lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1)
    assert sha(g) == str(d["gauge_sha"])
    assert sha(O.port_dirac(L, 1, 0.1, g, s)) == str(d["dphi_sha"])
    r = O.port_cg(L, 1, 0, 0.1, g, s, 1e-10)
    assert r["rc"] == 0 and r["iterations"] == int(d["cg_h_iterations"]) == 47
    np.testing.assert_allclose(r["history"], d["cg_h_history"], rtol=1e-8)
    e = O.port_cg(L, 1, 1, 0.1, g, s, 1e-10)
    assert e["rc"] == 0 and e["iterations"] == int(d["cg_eo_iterations"]) == 23
    assert e["true_rel_residual"] < 2e-10


@needs_ref
@pytest.mark.parametrize("n,rep", [(3, 0), (2, 0), (2, 1), (4, 3)], ids=["su3f", "su2f", "su2a", "su4as"])
def test_port_vs_reference_live(n, rep):
    L = [4, 4, 2, 6]
    dr = O.rep_dim(rep, n)
    g = O.ref_gauge_random(L, n, rep, 7)
    s = O.ref_spinor_random(L, dr, 7, 3)
    assert np.array_equal(s, O.port_spinor_random(L, dr, 7, 3))
    for bc in (0, 1):
        p = O.port_dirac(L, bc, 0.2, g, s)
        with O.exact_reference():
            assert np.array_equal(p, O.ref_apply_dirac(L, [1, 1, 1, 1], n, rep, bc, 0.2, g, s))
        # the default (FMA-contracting) reference build agrees to rounding
        assert rel_l2(p, O.ref_apply_dirac(L, [1, 1, 1, 1], n, rep, bc, 0.2, g, s)) < 1e-14
        # the reference's serial/parallel equivalence holds for the shim
        assert rel_l2(p, O.ref_apply_dirac(L, [2, 1, 1, 2], n, rep, bc, 0.2, g, s)) < 1e-14


@needs_ref
def test_hop_tables_and_flops_match_reference():
    assert np.array_equal(O.port_hop_tables(), O.ref_hop_tables())
    for dr in (1, 2, 3, 6, 10):
        for real in (0, 1):
            for k in (O.SQNORM, O.MULADD, O.DIRAC):
                assert O.port_flops_per_site(k, dr, real) == O.ref_flops_per_site(k, dr, real)
    # the integer FLOP model equals the instrumented twin
    for n, rep, want in [(2, 0, 752), (3, 0, 1512), (2, 1, 936), (4, 3, 5328)]:
        assert O.ref_counted_dirac([2, 2, 2, 2], n, rep) == want
        dr = O.rep_dim(rep, n)
        assert O.port_flops_per_site(O.DIRAC, dr, O.rep_is_real(rep)) == want


def test_gamma_algebra_golden():
    d = golden("group")
    gam = d["gammas"]
    eye = np.eye(4)
    for a in range(4):
        for b in range(4):
            anti = gam[a] @ gam[b] + gam[b] @ gam[a]
            assert np.abs(anti - 2 * (a == b) * eye).max() == 0
    assert np.abs(gam[0] @ gam[1] @ gam[2] @ gam[3] - gam[4]).max() == 0
    assert np.array_equal(O.port_hop_tables(), d["hop_tables"])


def _inner(a, b):
    return np.vdot(a.reshape(-1), b.reshape(-1))


def test_gamma5_hermiticity_and_linearity():
    """<phi, g5 D g5 psi> = conj <psi, D phi> at 8x4^3; linearity."""
    import paper_1401_3733_b200 as lb
    L = [8, 4, 4, 4]
    g = lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1)
    psi = O.port_spinor_random(L, 3, 1, 0)
    phi = O.port_spinor_random(L, 3, 1, 1)

    def g5(x):
        y = x.copy()
        y[:, 2:] *= -1
        return y

    lhs = _inner(phi, g5(O.port_dirac(L, 1, 0.1, g, g5(psi))))
    rhs = np.conj(_inner(psi, O.port_dirac(L, 1, 0.1, g, phi)))
    assert abs(lhs - rhs) < 1e-12 * abs(rhs)
    mh = lambda x: O.port_mhat(L, 1, 0.1, g, x)  # noqa: E731
    even = O.parity_mask(L)
    pe, fe = psi.copy(), phi.copy()
    pe[~even] = 0
    fe[~even] = 0
    assert abs(_inner(fe, g5(mh(g5(pe)))) - np.conj(_inner(pe, mh(fe)))) < 1e-12 * abs(_inner(pe, mh(fe)))
    a = 0.3 - 1.7j
    lin = O.port_dirac(L, 1, 0.1, g, a * psi + phi)
    assert rel_l2(lin, a * O.port_dirac(L, 1, 0.1, g, psi) + O.port_dirac(L, 1, 0.1, g, phi)) < 1e-12


def test_schur_relation_ties_eo_to_full_dirac():
    """x_o = -D_oe x_e / A  =>  D (x_e + x_o) = (Mhat x_e, 0)."""
    import paper_1401_3733_b200 as lb
    L = [4, 4, 4, 6]
    m = 0.1
    g = lb.init_gauge_random(L, 2, lb.FUNDAMENTAL, 3)
    s = O.port_spinor_random(L, 2, 3, 0)
    even = O.parity_mask(L)
    xe = s.copy()
    xe[~even] = 0
    xo = -O.port_hop_parity(L, 1, 1, -0.5, g, xe) / (4 + m)
    full = O.port_dirac(L, 1, m, g, xe + xo)
    mh = O.port_mhat(L, 1, m, g, xe)
    assert rel_l2(full[even], mh[even]) < 1e-13
    assert np.abs(full[~even]).max() < 1e-13 * np.abs(full).max()


def test_unit_gauge_mass_identity_port():
    """unit gauge, constant spinor, periodic -> D psi = m psi."""
    L = [4, 4, 4, 4]
    g = np.zeros((256, 4, 3, 3), np.complex128)
    g[:, :, range(3), range(3)] = 1
    s = np.broadcast_to(np.arange(12).reshape(4, 3) * (1 + 0.5j), (256, 4, 3)).copy()
    assert np.abs(O.port_dirac(L, 0, 0.25, g, s) - 0.25 * s).max() < 1e-13


def test_cg_edge_cases_port():
    import paper_1401_3733_b200 as lb
    L = [4, 4, 4, 4]
    g = lb.init_gauge_random(L, 2, lb.FUNDAMENTAL, 1)
    z = np.zeros((256, 4, 2), np.complex128)
    r = O.port_cg(L, 1, 0, 0.1, g, z, 1e-10)
    assert r["rc"] == 0 and r["iterations"] == 0 and not np.any(r["x"])
    s = O.port_spinor_random(L, 2, 1, 0)
    r = O.port_cg(L, 1, 0, 0.1, g, s, 1e-12, maxit=2)
    assert r["rc"] == 4 and 0 < r["best_residual"] < 1
    assert O.port_cg(L, 1, 0, 0.1, g, s, 1.5)["rc"] == 2


@needs_ref
def test_port_cg_matches_reference_iterations():
    import paper_1401_3733_b200 as lb
    L = [8, 4, 4, 4]
    for n, rep in [(2, 1), (4, 3)]:
        dr = O.rep_dim(rep, n)
        g = lb.init_gauge_random(L, n, rep, 1)
        s = O.port_spinor_random(L, dr, 1, 0)
        ref = O.ref_cg_h(L, [2, 1, 1, 1], n, rep, 1, 0.05, g, s, 1e-10)
        p = O.port_cg(L, 1, 0, 0.05, g, s, 1e-10)
        assert abs(p["iterations"] - ref["iterations"]) <= 1
        refe = O.ref_cg_eo(L, [1, 1, 1, 1], n, rep, 1, 0.05, g, s, 1e-10)
        pe = O.port_cg(L, 1, 1, 0.05, g, s, 1e-10)
        assert abs(pe["iterations"] - refe["iterations"]) <= 1
        assert rel_l2(pe["x"], refe["x"]) < 1e-8


@needs_ref
def test_cpu_baseline_entry_points_run_the_baseline_workload():
    """bench.py's CPU legs: ref_cg_probe solves to the same iteration counts as
    the global-array reference CG on the same inputs (keyed per worker:
    decomposition-invariant), and its bounded-sample mode runs exactly the
    requested iterations; ref_bench_dirac returns one time per sample."""
    L, n, rep, m = [8, 8, 8, 8], 3, O.FUNDAMENTAL, 0.1
    z = np.load(os.path.join(GOLD, "cfg1.npz"))
    for grid in ([1, 1, 1, 1], [2, 1, 1, 2]):
        h = O.ref_cg_probe(L, grid, n, rep, m, 1, False, 1000, tol=1e-10)
        e = O.ref_cg_probe(L, grid, n, rep, m, 1, True, 1000, tol=1e-10)
        assert h["iterations"] == int(z["cg_h_iterations"]) and h["true_rel_residual"] < 2e-10
        assert e["iterations"] == int(z["cg_eo_iterations"]) and e["true_rel_residual"] < 2e-10
    p = O.ref_cg_probe(L, [2, 1, 1, 1], n, rep, m, 1, True, 4, tol=0.0)
    assert p["iterations"] == 4 and p["true_rel_residual"] == -1.0 and p["seconds"] > 0
    t = O.ref_bench_dirac(L, [2, 1, 1, 1], n, rep, m, 1, 3, nsamples=3)
    assert len(t) == 3 and min(t) > 0
    # near-unit links (config 3's generator) through the same entry points
    nu = O.ref_cg_probe([4, 4, 4, 4], [1, 1, 1, 1], 3, rep, 0.1, 1, True, 500, tol=1e-10, links=O.LINKS_NEAR_UNIT)
    assert nu["true_rel_residual"] < 2e-10 and nu["iterations"] > 0


@needs_ref
def test_near_unit_generator_parallel_matches_golden():
    """The threaded near-unit generator reproduces the committed fixture."""
    z = golden("near_unit")
    with O.exact_reference():  # the fixture came from the FMA-free build
        assert np.array_equal(O.ref_gauge_near_unit([2, 2, 2, 2], 3, 0.3, 1), z["links"])


REPORT = {
    "format_version": 1, "regime": "balance", "timestamp": "2026-10-20T00:00:00Z",
    "geometry": {"lattice": [16, 8, 8, 8], "grid": [1, 1, 1, 1], "local": [16, 8, 8, 8], "workers": 1},
    "group_rank": 3, "representation": "fundamental", "mass": 0.1, "seed": 1,
    "kernels": [{"kernel": k, "iterations": 7, "seconds": 0.25, "flops": f * 7 * 8192, "flops_per_sec": 1.5e9,
                 "flops_per_sec_per_worker": 1.5e9, "short_run": False, "reference_ratio": None}
                for k, f in (("sqnorm", 48), ("muladd", 96), ("dirac", 1512))],
    "consistency": {"status": "passed", "iterations": 23, "residual": 4.2e-11, "seconds": 0.001, "solver": "eo"},
    "model": {"sqnorm_flops_per_site": 48, "muladd_flops_per_site": 96, "dirac_flops_per_site": 1512,
              "halo_bytes_per_exchange": 0, "dirac_intensity": 0.0},
    "device": "B200 (sm_100a), latbench-b200",
}


@needs_ref
def test_report_reader_interop():
    """report.cpp:182-217: the reference's report_from_json accepts the
    driver's format-1 JSON (extra keys ignored) and round-trips every field;
    a format_version it does not know is a ConfigError (rc 2)."""
    import json
    if not hasattr(O.ref_lib(), "ref_report_reformat"):
        pytest.skip("reference built without report.cpp")
    back = json.loads(O.ref_report_reformat(json.dumps(REPORT), "json"))
    for k in ("format_version", "regime", "timestamp", "geometry", "group_rank", "representation", "mass", "seed",
              "kernels", "model"):
        assert back[k] == REPORT[k], k
    assert back["consistency"] == {k: v for k, v in REPORT["consistency"].items() if k != "solver"}
    csv = O.ref_report_reformat(json.dumps(REPORT), "csv").splitlines()
    assert csv[0] == "kernel,iterations,seconds,flops,flops_per_sec,flops_per_sec_per_worker"
    assert csv[3].startswith("dirac,7,2.500000000e-01,")
    bad = dict(REPORT, format_version=2)
    with pytest.raises(O.OracleError) as e:
        O.ref_report_reformat(json.dumps(bad), "json")
    assert e.value.code == 2


@needs_ref
def test_b200_driver_report_reads_back_in_the_reference():
    """A report written by the B200 driver (tools/latbench_b200 run --emit-all
    on the GPU box, committed as tests/golden/report_b200.*) parses with the
    reference's report_from_json, and the reference's own writers reproduce
    the driver's CSV byte for byte and its JSON field for field."""
    import json
    if not hasattr(O.ref_lib(), "ref_report_reformat"):
        pytest.skip("reference built without report.cpp")
    ours = open(os.path.join(GOLD, "report_b200.json")).read()
    assert O.ref_report_reformat(ours, "csv") == open(os.path.join(GOLD, "report_b200.csv")).read()
    back, mine = json.loads(O.ref_report_reformat(ours, "json")), json.loads(ours)
    for k in ("format_version", "regime", "timestamp", "geometry", "group_rank", "representation", "mass", "seed",
              "kernels", "model"):
        assert back[k] == mine[k], k
    text = O.ref_report_reformat(ours, "text")
    assert "dirac" in text and "consistency    passed (23 iterations" in text


def test_fullsize_reference_cg_counts_are_pinned():
    """tests/golden/cg_cfg*.npz (make_fullsize_cg.py, the unmodified reference
    at BASELINE.json's full sizes): every config has plain and eo counts, the
    solves met their tolerance, and config 1 agrees with cfg1.npz."""
    want = {1: (47, 23), 2: (48, 23), 3: (389, 128), 4: (49, 23), 5: (47, 23)}
    for c, (h, eo) in want.items():
        z = np.load(os.path.join(GOLD, f"cg_cfg{c}.npz"))
        assert (int(z["h_iterations"]), int(z["eo_iterations"])) == (h, eo)
        assert z["h_true"] < 2 * z["tol"] and z["eo_true"] < 2 * z["tol"]
        assert len(z["h_history"]) == h and len(z["eo_history"]) == eo
    z1 = golden("cfg1")
    assert int(z1["cg_h_iterations"]) == 47 and int(z1["cg_eo_iterations"]) == 23
