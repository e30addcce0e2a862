"""Host-side checks of the product library (CPU only, no GPU compute):
the C-ABI exports, bit-identical seeded inputs, decomposition rules, and the
face schedule of the N > 1 halo exchange (including a 2-process gloo run)."""
import os
import re
import socket

import numpy as np
import pytest

import oracle as O
import paper_1401_3733_b200 as lb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.exists(O.REF_EXACT_SO)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "lbcu.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lbcu_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = lb.lib()
    syms = declared_symbols()
    assert len(syms) >= 45
    for s in syms:
        assert hasattr(L, s), s
    assert L.lbcu_abi_version() == 1


def test_product_has_no_cpu_fallback_or_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_1401_3733_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cpp", ".cu", ".hpp", ".cuh")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle/_ref" not in src, f


def test_context_fails_loudly_without_device():
    if lb.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(lb.CudaError):
        lb.Context([4, 4, 4, 4])


@needs_ref
@pytest.mark.parametrize("n,rep", [(3, 0), (2, 0), (2, 1), (4, 3), (3, 2), (3, 3)])
def test_host_generators_bit_identical_to_reference(n, rep):
    L = [4, 2, 4, 2]
    dr = O.rep_dim(rep, n)
    with O.exact_reference():
        assert np.array_equal(lb.init_gauge_random(L, n, rep, 5), O.ref_gauge_random(L, n, rep, 5))
        assert np.array_equal(lb.init_gauge_random(L, n, rep, 5, links=lb.LINKS_UNIT), O.ref_gauge_unit(L, n, rep))
    assert np.array_equal(lb.init_spinor_random(L, dr, 5, 2), O.ref_spinor_random(L, dr, 5, 2))


def test_host_generators_match_golden():
    import hashlib
    for name in ("su3f", "su2f", "su2a", "su4as", "su3s"):
        d = np.load(os.path.join(ROOT, "tests", "golden", f"{name}.npz"))
        L, n, rep = list(d["lattice"]), int(d["n"]), int(d["rep"])
        g = lb.init_gauge_random(L, n, rep, 1)
        assert hashlib.sha256(g.tobytes()).hexdigest() == str(d["gauge_sha"]), name
        s = lb.init_spinor_random(L, lb.rep_dim(rep, n), 1, 0)
        assert hashlib.sha256(s.tobytes()).hexdigest() == str(d["spinor_sha"]), name
    nu = np.load(os.path.join(ROOT, "tests", "golden", "near_unit.npz"))["links"]
    mine = lb.init_gauge_random([2, 2, 2, 2], 3, lb.FUNDAMENTAL, 1, links=lb.LINKS_NEAR_UNIT, eps=0.3)
    assert np.abs(mine - nu).max() < 1e-14
    # the near-unit links are SU(3) to rounding
    u = mine.reshape(-1, 3, 3)
    assert np.abs(np.einsum("kij,kil->kjl", u.conj(), u) - np.eye(3)).max() < 1e-13
    assert np.abs(np.linalg.det(u) - 1).max() < 1e-13


def test_local_generation_is_decomposition_invariant():
    L = [8, 4, 4, 8]
    grid = [2, 1, 1, 2]
    from helpers import global_index
    gs = lb.init_spinor_random(L, 3, 1, 0)
    gg = lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1)
    for r in range(4):
        idx = global_index(L, grid, r)
        assert np.array_equal(lb.init_spinor_random(L, 3, 1, 0, grid=grid, rank=r), gs[idx])
        assert np.array_equal(lb.init_gauge_random(L, 3, lb.FUNDAMENTAL, 1, grid=grid, rank=r), gg[idx])


def test_decomposition_errors_mirror_reference():
    """geometry.cpp:75-95 -> DecompositionError; the eo layout needs even local extents."""
    with pytest.raises(lb.DecompositionError):
        lb.local_extents([7, 4, 4, 4], [1, 1, 1, 1])
    with pytest.raises(lb.DecompositionError):
        lb.local_extents([8, 4, 4, 4], [3, 1, 1, 1])
    with pytest.raises(lb.DecompositionError):
        lb.local_extents([8, 4, 4, 4], [2, 1, 1, 1], enforce_floor=True)
    with pytest.raises(lb.DecompositionError):
        lb.local_extents([8, 4, 4, 4], [8, 1, 1, 1])
    with pytest.raises(lb.ContractViolation):
        lb.local_extents([8, 4, 4, 4], [2, 1, 1, 1], rank=2)
    assert lb.local_extents([96, 48, 48, 48], [8, 1, 1, 1]) == (12, 48, 48, 48)
    with pytest.raises(lb.ConfigError):
        lb.rep_dim(lb.FUNDAMENTAL, 1)


def test_flops_model_matches_reference():
    for dr in (2, 3, 6, 8):
        for real in (False, True):
            for k in (lb.SQNORM, lb.MULADD, lb.DIRAC):
                assert lb.flops_per_site(k, dr, real) == O.port_flops_per_site(k, dr, real)
    assert lb.flops_per_site(lb.DIRAC, 3, False) == 1512
    assert lb.flops_per_site(lb.DIRAC, 6, False) == 5328


def _coords(idx, loc):
    c = []
    for d in (3, 2, 1, 0):
        c.append(idx % loc[d])
        idx //= loc[d]
    return c[::-1]


def _rank_coords(r, grid):
    c = []
    for d in (3, 2, 1, 0):
        c.append(r % grid[d])
        r //= grid[d]
    return c[::-1]


@pytest.mark.parametrize("grid", [(2, 1, 1, 1), (4, 1, 1, 2), (2, 2, 1, 2), (1, 1, 2, 2)])
@pytest.mark.parametrize("qpar", [0, 1])
def test_face_schedule_pairs_halo_records(grid, qpar):
    """Record j of rank r's face (mu, dir) is exactly the neighbour site the
    receiving rank's boundary site with in-face index j needs."""
    L = [8, 4, 4, 8]
    loc = [L[d] // grid[d] for d in range(4)]
    nr = int(np.prod(grid))
    plans = [lb.plan_faces(L, grid, r, qpar) for r in range(nr)]
    for r in range(nr):
        partner, count, sites = plans[r]
        rc = _rank_coords(r, grid)
        off = 0
        for f in range(8):
            mu, dr_ = divmod(f, 2)
            if grid[mu] == 1:
                assert partner[f] == -1 and count[f] == 0
                continue
            assert count[f] == int(np.prod(loc)) // loc[mu] // 2
            recv = partner[f]
            others = [d for d in range(4) if d != mu]
            for j in range(count[f]):
                c = _coords(int(sites[off + j]), loc)
                assert c[mu] == (0 if dr_ == 0 else loc[mu] - 1)
                assert sum(c) % 2 == qpar
                fp = ((c[others[0]] * loc[others[1]] + c[others[1]]) * loc[others[2]] + c[others[2]])
                assert fp >> 1 == j
                # the receiver's boundary site: global neighbour relation
                g_send = [rc[d] * loc[d] + c[d] for d in range(4)]
                rcv = _rank_coords(recv, grid)
                x = list(c)
                x[mu] = loc[mu] - 1 if dr_ == 0 else 0
                g_recv = [rcv[d] * loc[d] + x[d] for d in range(4)]
                step = 1 if dr_ == 0 else -1  # receiver's +mu (dir 0) / -mu (dir 1) neighbour
                g_recv[mu] = (g_recv[mu] + step) % L[mu]
                assert g_recv == g_send
            off += count[f]


def test_bench_decompose_rules():
    """bench.py: T first while the local T stays >= 8 and even, then Z."""
    import bench
    assert bench.decompose([32, 32, 32, 32], 8) == [4, 1, 1, 2]
    assert bench.decompose([96, 48, 48, 48], 8) == [8, 1, 1, 1]
    assert bench.decompose([40, 40, 40, 40], 8) == [4, 1, 1, 2]
    assert bench.decompose([64, 32, 32, 32], 8) == [8, 1, 1, 1]
    assert bench.decompose([32, 32, 32, 32], 2) == [2, 1, 1, 1]
    for L in ([32] * 4, [96, 48, 48, 48], [40] * 4, [64, 32, 32, 32]):
        for n in (1, 2, 4, 8):
            g = bench.decompose(L, n)
            assert int(np.prod(g)) == n
            assert lb.local_extents(L, g)  # valid even-odd decomposition


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, L, grid, q, result):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        loc = [L[d] // grid[d] for d in range(4)]
        spinor = lb.init_spinor_random(L, 2, 1, 0, grid=grid, rank=rank)
        glob = lb.init_spinor_random(L, 2, 1, 0)
        partner, count, sites = lb.plan_faces(L, grid, rank, q)
        # pack raw records face by face, exchange exactly as the library pairs
        # messages: send face f to partner[f], receive its halo from partner[f ^ 1]
        off, ok = 0, True
        offs = np.cumsum([0] + count)
        for f in range(8):
            if count[f] == 0:
                continue
            send = torch.from_numpy(spinor[sites[offs[f]:offs[f + 1]]].copy())
            recv = torch.empty_like(send)
            reqs = [dist.isend(send, partner[f]), dist.irecv(recv, partner[f ^ 1])]
            for rq in reqs:
                rq.wait()
            # check what arrived against the global field at the receiver's neighbours
            mu, d = divmod(f, 2)
            others = [x for x in range(4) if x != mu]
            rc = _rank_coords(rank, grid)
            p = 1 - q
            edge = loc[mu] - 1 if d == 0 else 0  # dir-0 records feed my forward halo
            for j in range(count[f]):
                pass
            for sidx in range(int(np.prod(loc))):
                c = _coords(sidx, loc)
                if c[mu] != edge or sum(c) % 2 != p:
                    continue
                fp = ((c[others[0]] * loc[others[1]] + c[others[1]]) * loc[others[2]] + c[others[2]])
                g = [rc[k] * loc[k] + c[k] for k in range(4)]
                g[mu] = (g[mu] + (1 if d == 0 else -1)) % L[mu]
                gi = ((g[0] * L[1] + g[1]) * L[2] + g[2]) * L[3] + g[3]
                ok &= bool(np.array_equal(recv.numpy()[fp >> 1], glob[gi]))
            off += count[f]
        result[rank] = ok
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_halo_exchange():
    """world_size 2 over gloo on CPU: the face schedule + message pairing of the
    N > 1 path deliver every boundary site's neighbour record."""
    import torch.multiprocessing as mp
    L, grid = [8, 4, 4, 4], [2, 1, 1, 1]
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    result = mgr.dict()
    for q in (0, 1):
        ctx = mp.get_context("spawn")
        ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port + q, L, grid, q, result)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(120)
            assert p.exitcode == 0
        assert result[0] and result[1]


def _ipc_bootstrap(rank, nranks, name, q):
    import paper_1401_3733_b200 as lbm
    try:
        w = lbm.World.ipc(nranks, rank, name)  # shared-memory bootstrap + barrier, no CUDA call
        w.close()                              # collective teardown barrier
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


def test_ipc_world_bootstrap_on_host():
    """lbcu_world_ipc's POSIX shared-memory bootstrap (rank 0 creates the
    segment, the others attach), its generation barrier and its collective
    teardown, across three processes; the segment name is unlinked once every
    rank holds the mapping. Bad arguments fail with a config error."""
    import multiprocessing as mp
    import uuid

    name = f"/lbcu_host_{uuid.uuid4().hex[:12]}"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ipc_bootstrap, args=(r, 3, name, q)) for r in range(3)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok", 2: "ok"}
    assert not os.path.exists("/dev/shm" + name)
    with pytest.raises(lb.ConfigError):
        lb.World.ipc(2, 0, "no-leading-slash")
    with pytest.raises(lb.ConfigError):
        lb.World.ipc(9, 0, "/lbcu_too_many")


def test_handle_ownership_releases_children_first(monkeypatch):
    """paper_1401_3733_b200._Owned: whatever order the garbage collector
    finalises a cycle in, a field's handle is freed before its context's and
    a context's before its world's, each exactly once (a fake library records
    the destroy calls; no device needed)."""
    import gc
    import paper_1401_3733_b200 as lb

    calls = []

    class FakeLib:
        def __getattr__(self, name):
            return lambda h: calls.append((name, h))

    monkeypatch.setattr(lb, "_lib", FakeLib())

    class W(lb._Owned):
        _destroy = "world_destroy"

    class Cx(lb._Owned):
        _destroy = "ctx_destroy"

    class F(lb._Owned):
        _destroy = "field_destroy"

    def make(tag):
        w = W()
        w._own(f"w{tag}")
        c = Cx()
        c._own(f"c{tag}", w)
        fs = [F() for _ in range(3)]
        for k, f in enumerate(fs):
            f._own(f"f{tag}{k}", c)
        return w, c, fs

    # explicit close of a middle node
    w, c, fs = make("a")
    fs[0].close()
    c.close()
    assert calls[0] == ("field_destroy", "fa0") and calls[-1] == ("ctx_destroy", "ca")
    assert sorted(h for _, h in calls) == ["ca", "fa0", "fa1", "fa2"]
    fs[1].close()
    w.close()
    assert calls[-1] == ("world_destroy", "wa") and len(calls) == 5
    # a garbage cycle through all three levels
    calls.clear()
    w, c, fs = make("b")
    w.cycle, c.cycle = (c, fs), (w, fs)
    for f in fs:
        f.cycle = (w, c)
    del w, c, fs, f
    gc.collect()
    order = [h for _, h in calls]
    assert sorted(order) == ["cb", "fb0", "fb1", "fb2", "wb"]
    assert order.index("cb") > max(order.index(f"fb{k}") for k in range(3))
    assert order.index("wb") == len(order) - 1


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblatbench_ref.so")),
                    reason="reference not built")
def test_reference_arm_reports_the_gpu_arms_workload():
    """bench.py --impl reference: the unmodified reference on the host on the
    GPU arm's exact workload description (config dict identical, so the
    driver can pair the arms), with its own cpu_baseline and a zero-copy e2e."""
    import json
    import subprocess
    import sys
    import bench
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"] == json.loads(json.dumps(bench.config_dict(bench.CONFIGS[1], 1)))
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
