#!/usr/bin/env python
"""Benchmark driver: Dphi GFLOP/s and CG time-to-solution on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
    python bench.py --regime comms|balance|compute      (stock regimes, 64x32^3)

Mirrors the reference's Dirac kernel benchmark (proj/src/bench.cpp:190-248:
FLOPs = flops_per_site x global volume x applications, exact integers) on
BASELINE.json's configs. Default workload: configs[2], SU(3) fundamental
96x48^3 with near-unit links — the largest single-GPU configuration, and the
lattice the north star's scaling target is stated on. A step is one full Dphi
application over the lattice, inputs resident in HBM. One JSON line on
rank 0, which also carries

* ``cg``: even-odd CG time to solution (and plain CG on D^dag D, the
  reference's own algorithm) at the config's tolerance;
* ``cpu_baseline``: the unmodified reference on this host's cores, measured
  in a fresh subprocess (median of 3 Dphi samples; CG time to solution as
  measured ms per iteration x the reference's iteration count, flagged
  extrapolated when the full solve does not fit the CPU budget);
* ``configs``: Dphi, eo hop and eo CG for every BASELINE config (1-5) on the
  same GPU and run, each with its roofline fraction and a short CPU sample.

Under torchrun (N > 1) each rank owns one GPU and one sub-lattice (T split
first, then Z: SURVEY.md §8e). Halos go straight from the pack kernel into
the neighbour's receive arena over NVLink (the library's IPC world), checked
once per run bit for bit against NCCL send/recv halos (LBCU_TRANSPORT=nccl
forces NCCL); CG sums use NCCL. Time is the max over ranks of CUDA-event
time.

--impl reference times the reference's own CPU apply_dirac (oracle/_ref, the
unmodified latbench compiled from its sources) with all host threads on the
same config and workload (same links, antiperiodic t).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs: (name, lattice T,X,Y,Z, N, rep, m0, links, cg tol)
CONFIGS = {
    1: dict(name="cfg1 SU(3)F 8^4", L=[8, 8, 8, 8], n=3, rep=0, mass=0.1, links="haar", tol=1e-10),
    2: dict(name="cfg2 SU(2)F 32^4", L=[32, 32, 32, 32], n=2, rep=0, mass=0.05, links="haar", tol=1e-10),
    3: dict(name="cfg3 SU(3)F 96x48^3 near-unit", L=[96, 48, 48, 48], n=3, rep=0, mass=0.02,
            links="near_unit", tol=1e-12),
    4: dict(name="cfg4 SU(2)A 40^4", L=[40, 40, 40, 40], n=2, rep=1, mass=0.05, links="haar", tol=1e-10),
    5: dict(name="cfg5 SU(4)AS 64x32^3", L=[64, 32, 32, 32], n=4, rep=3, mass=0.1, links="haar", tol=1e-10),
}
# the reference's stock regimes at the paper's 64x32^3 (proj/src/bench.cpp:26-42)
REGIMES = {
    "comms": dict(name="regime comms SU(2)A 64x32^3", L=[64, 32, 32, 32], n=2, rep=1, mass=0.1, links="haar",
                  tol=1e-10),
    "balance": dict(name="regime balance SU(3)F 64x32^3", L=[64, 32, 32, 32], n=3, rep=0, mass=0.1,
                    links="haar", tol=1e-10),
    "compute": dict(name="regime compute SU(6)F 64x32^3", L=[64, 32, 32, 32], n=6, rep=0, mass=0.1,
                    links="haar", tol=1e-10),
}
DEFAULT_CONFIG = 3
METRIC = "Dphi GFLOP/s and CG time-to-solution vs GPUs (1/2/4/8), % of HBM roofline"
L2_BYTES = 126e6


def decompose(L, n):
    """T first while the local T stays >= 8 and even, then Z."""
    grid = [1, 1, 1, 1]
    left = n

    def can_halve(d, floor):
        loc = L[d] // (grid[d] * 2)
        return left > 1 and left % 2 == 0 and L[d] % (grid[d] * 2) == 0 and loc % 2 == 0 and loc >= floor

    while can_halve(0, 8):
        grid[0] *= 2
        left //= 2
    for d in (3, 2, 1):
        while can_halve(d, 2):
            grid[d] *= 2
            left //= 2
    if left != 1:
        raise SystemExit(f"cannot decompose {L} over {n} ranks")
    return grid


def rep_dim(rep, n):
    return {0: n, 1: n * n - 1, 2: n * (n + 1) // 2, 3: n * (n - 1) // 2}[rep]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def link_bytes(dr, real, fmt="full"):
    """Bytes of one link as stored on the device (links.cuh)."""
    return {"full": dr * dr * (8 if real else 16), "su2": 32, "r12": 96, "r10": 80, "as4": 256, "as4r": 288}[fmt]


def bytes_full_dphi(dr, real, fmt="full"):
    """SURVEY.md §8(d) compulsory bytes per site of a full Dphi: spinor in + out
    (128 d) + each of the 4 links of the site once; with fmt = "full" this is
    SURVEY's 128 d + 32 c d^2."""
    return 128 * dr + 4 * link_bytes(dr, real, fmt)


def bytes_eo_hop(dr, real, fmt="full"):  # per output site: 128 d + 8 links
    return 128 * dr + 8 * link_bytes(dr, real, fmt)


def bytes_eo_cg_iter(dr, real, fmt="full"):  # per even site 4 B_hop + 11 * 64 d
    return 4 * bytes_eo_hop(dr, real, fmt) + 11 * 64 * dr


def bytes_h_cg_iter(dr, real, fmt="full"):  # per site 2 B_full + 9 * 64 d
    return 2 * bytes_full_dphi(dr, real, fmt) + 9 * 64 * dr


def config_dict(cfg, ws):
    """The workload description, identical in both arms (same_config)."""
    L, n, rep = cfg["L"], cfg["n"], cfg["rep"]
    dr = rep_dim(rep, n)
    V = int(np.prod(L))
    dense = bytes_full_dphi(dr, rep == 1) * V
    grid = decompose(L, ws) if ws > 1 else [1, 1, 1, 1]
    return {"workload": cfg["name"], "lattice_TXYZ": L, "group_rank": n, "rep": rep, "dr": dr,
            "mass": cfg["mass"], "links": cfg["links"] + (" (U = exp(i 0.3 H))" if cfg["links"] == "near_unit"
                                                          else " (Haar)"),
            "bc": "periodic space, antiperiodic time", "seed": 1, "cg_tolerance": cfg["tol"], "grid": grid,
            "parallelism": f"domain decomposition, grid {grid} over {ws} rank(s)",
            "l2": (f"inputs larger than L2 ({dense / 1e6:.0f} MB touched per step vs 126 MB)" if dense > L2_BYTES
                   else f"L2-resident ({dense / 1e6:.1f} MB per step): launch-bound, not gated on HBM")}


def duplex_copy_ms(hin, hout, nbytes, reps=10):
    """The bound of the e2e number: pinned H2D and D2H copies of a step's
    bytes, alone and running concurrently on two streams (plain
    cudaMemcpyAsync through cuda-python; tools/pcie_probe.cu measures the
    same), best of 3 passes, ms per step: {"both", "h2d", "d2h"}."""
    try:
        import torch
        from cuda.bindings import runtime as rt
    except Exception:  # noqa: BLE001
        return None
    dbuf = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    sh, sd = torch.cuda.Stream(), torch.cuda.Stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h2d, d2h = rt.cudaMemcpyKind.cudaMemcpyHostToDevice, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost

    def run(mode):
        torch.cuda.synchronize()
        t0.record()
        sh.wait_event(t0)
        sd.wait_event(t0)
        for k in range(reps):
            if mode != "d2h":
                rt.cudaMemcpyAsync(dbuf[0].data_ptr(), hin[k % 2].data_ptr(), nbytes, h2d, sh.cuda_stream)
            if mode != "h2d":
                rt.cudaMemcpyAsync(hout[k % 2].data_ptr(), dbuf[1].data_ptr(), nbytes, d2h, sd.cuda_stream)
        cur = torch.cuda.current_stream()
        cur.wait_stream(sh)
        cur.wait_stream(sd)
        t1.record()
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / reps

    res = {mode: min(run(mode) for _ in range(3)) for mode in ("both", "h2d", "d2h")}
    del dbuf
    torch.cuda.empty_cache()
    return res


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler run DURING the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device=0):
        self.samples, self.reasons, self.ok = [], 0, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _sample(self):
        nv = self.nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.reasons |= nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            if not self.samples:
                self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and k != 0x1]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def traffic_from_profiles(key, ws):
    """dram bytes per launch of the kernel from the committed single-GPU ncu
    summary; None at N > 1 (a rank's launch covers 1/N of the lattice plus
    its faces, never profiled)."""
    if ws > 1:
        return None
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def golden_cg_iterations(c):
    """The reference's own iteration counts at full size (tests/golden/cg_cfg<c>.npz,
    tests/golden/make_fullsize_cg.py): {"eo": .., "h": ..} or {}."""
    path = os.path.join(ROOT, "tests", "golden", f"cg_cfg{c}.npz")
    try:
        z = np.load(path)
        return {"eo": int(z["eo_iterations"]), "h": int(z["h_iterations"])}
    except Exception:
        return {}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------- CPU (reference)
def cpu_leg(configs, budget, cg_configs, gpu_its):
    """The unmodified reference (oracle/_ref) on this host's cores, each config
    a bounded sample: median of 3 Dphi samples; for cg_configs also the
    reference CG (its own plain CG on H, and the cg_solve driven by the
    composed eo operator): a full solve when it fits the budget, else the
    measured seconds per iteration x the reference's iteration count
    (extrapolated). Run in a fresh subprocess (bench.py --cpu-leg)."""
    import oracle as O

    host = O.host_cpu()
    nthreads = host["logical_cpus"]
    out = {}
    for c in configs:
        cfg = CONFIGS[c]
        cbudget = budget if c in cg_configs else budget / 2
        L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
        links = O.LINKS_NEAR_UNIT if cfg["links"] == "near_unit" else O.LINKS_HAAR
        dr = O.rep_dim(rep, n)
        V = int(np.prod(L))
        fps = O.ref_flops_per_site(O.DIRAC, dr, O.rep_is_real(rep))
        grid = O.grid_for_threads_balanced(L, nthreads)
        cores = int(np.prod(grid))
        one = O.ref_bench_dirac(L, grid, n, rep, mass, 1, 1, links=links, nwarm=0)
        napps = int(max(1, min(200, cbudget / 3.0 / max(one, 1e-6))))
        t = O.ref_bench_dirac(L, grid, n, rep, mass, 1, napps, links=links, nwarm=1, nsamples=3)
        med = statistics.median(t)
        rec = {"value": fps * V * napps / med / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
               "ms_per_dphi": med / napps * 1e3,
               "samples_gflops": [fps * V * napps / x / 1e9 for x in t],
               "sample": f"median of 3 samples of {napps} apply_dirac of the unmodified reference on "
                         f"{cfg['name']} (antiperiodic t, {cfg['links']} links), {cores} worker threads, "
                         f"grid {grid}, fresh subprocess",
               **{k: host[k] for k in ("model", "logical_cpus", "physical_cores", "reference_isa")}}
        if c in cg_configs:
            golden = golden_cg_iterations(c)
            cg = {}
            for kind, eo, per_it_dphi in (("eo", True, 4), ("plain", False, 2)):
                its_ref = golden.get("eo" if eo else "h") or gpu_its.get(str(c), {}).get(kind)
                est = (its_ref or 100) * per_it_dphi * med / napps
                if est < budget:
                    r = O.ref_cg_probe(L, grid, n, rep, mass, 1, eo, 20000, tol=cfg["tol"], links=links)
                    cg[kind] = {"seconds": r["seconds"], "iterations": r["iterations"],
                                "true_rel_residual": r["true_rel_residual"], "extrapolated": False}
                else:
                    k = int(max(3, min(20, budget / 2.0 / (per_it_dphi * med / napps))))
                    r = O.ref_cg_probe(L, grid, n, rep, mass, 1, eo, k, tol=0.0, links=links)
                    per_it = r["seconds_per_iteration"]
                    cg[kind] = {"seconds": per_it * its_ref if its_ref else None, "iterations": its_ref,
                                "seconds_per_iteration": per_it, "sampled_iterations": k,
                                "method": "(t(k iterations) - t(1 iteration)) / (k - 1) x the iteration count",
                                "extrapolated": True,
                                "iterations_source": "reference at full size (tests/golden/cg_cfg%d.npz)" % c
                                if golden else "GPU solve (reference count unavailable)"}
                cg[kind]["solver"] = ("reference cg_solve on the composed g5 Mhat g5 Mhat (eo oracle)" if eo
                                      else "reference cg_solve(make_h_operator) on D^dag D (its own algorithm)")
            rec["cg"] = cg
        out[str(c)] = rec
    return out


def run_cpu_leg_subprocess(configs, budget, cg_configs, gpu_its, timeout=900):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--cpu-leg", ",".join(map(str, configs)),
           "--cpu-seconds", str(budget), "--cpu-cg", ",".join(map(str, cg_configs)),
           "--cpu-gpu-its", json.dumps(gpu_its)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
        for line in reversed(r.stdout.splitlines()):
            if line.startswith("{"):
                return json.loads(line)
        return {"error": (r.stderr or r.stdout)[-400:]}
    except Exception as e:  # the CPU baseline is reported, not required
        return {"error": str(e)}


def run_reference(args, cfg):
    import oracle as O

    ws, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference (its threads use every core)
    L, n, rep = cfg["L"], cfg["n"], cfg["rep"]
    links = O.LINKS_NEAR_UNIT if cfg["links"] == "near_unit" else O.LINKS_HAAR
    dr = O.rep_dim(rep, n)
    host = O.host_cpu()
    grid = O.grid_for_threads_balanced(L, host["logical_cpus"])
    cores = int(np.prod(grid))
    fps = O.ref_flops_per_site(O.DIRAC, dr, O.rep_is_real(rep))
    V = int(np.prod(L))
    # each step = one apply_dirac (bench.cpp:209) over the whole lattice, the
    # same workload as the GPU arm (links, antiperiodic t, seed 1)
    secs = O.ref_bench_dirac(L, grid, n, rep, cfg["mass"], 1, args.steps, links=links, nwarm=max(1, args.warmup))
    value = fps * V * args.steps / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference keyed RNG, seed 1 (Haar / near-unit links, Gaussian spinor)",
        "config": config_dict(cfg, ws),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} apply_dirac of the unmodified reference on {cfg['name']}, "
                                   f"{cores} worker threads, grid {grid}",
                         **{k: host[k] for k in ("model", "logical_cpus", "physical_cores", "reference_isa")}},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm
class Run:
    """Per-process GPU state shared by the measurements (world, timing helpers)."""

    def __init__(self, args):
        import paper_1401_3733_b200 as lb

        self.lb, self.args = lb, args
        self.ws, self.rank, self.local = dist_env()
        self.dist, self.world, self.transport = None, None, "none (one rank)"
        if self.ws > 1:
            import uuid

            import torch
            import torch.distributed as dist
            self.dist = dist
            if args.emulate:  # test mode: every rank on GPU 0, gloo, no NCCL at all
                self.local = 0
                torch.cuda.set_device(0)
                dist.init_process_group("gloo")
            else:
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            obj = [(None if args.emulate else lb.World.nccl_unique_id(), f"/lbcu_{uuid.uuid4().hex[:16]}")
                   if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid, shm_name = obj[0]
            # halos: direct peer-memory stores by the pack kernel (IPC world;
            # NCCL for the CG sums), checked against NCCL send/recv halos;
            # LBCU_TRANSPORT=nccl forces the NCCL world
            transport = os.environ.get("LBCU_TRANSPORT", "ipc")
            if transport == "ipc":
                try:
                    self.world = lb.World.ipc(self.ws, self.rank, shm_name, uid)
                except Exception as e:  # noqa: BLE001
                    transport = f"nccl (ipc world unavailable: {e})"
            if self.world is None:
                if args.emulate:
                    raise SystemExit(f"--emulate needs the IPC world: {transport}")
                self.world = lb.World.nccl(self.ws, self.rank, uid)
            self.transport = transport
        self.checked_direct = False

    def barrier(self, ctx):
        ctx.synchronize()
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, x):
        if self.dist is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if self.args.emulate else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def setup(self, cfg):
        lb = self.lb
        L, n, rep = cfg["L"], cfg["n"], cfg["rep"]
        grid = decompose(L, self.ws) if self.ws > 1 else [1, 1, 1, 1]
        links = {"haar": lb.LINKS_HAAR, "near_unit": lb.LINKS_NEAR_UNIT}[cfg["links"]]
        ctx = lb.Context(L, grid, self.rank, self.local if self.ws > 1 else 0, self.world)
        # links: the reference's keyed generator evaluated on the device (seed 1,
        # keyed by global site: identical for any decomposition)
        gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T)
        if self.args.dense_links:
            gauge.set_compact(False)
        if self.args.host_links:
            gauge.upload(lb.init_gauge_random(L, n, rep, 1, grid=grid, rank=self.rank, links=links, eps=0.3))
        else:
            gauge.generate(1, links=links, eps=0.3)
        return ctx, gauge, grid

    def check_direct_halos(self, ctx, gauge, a, mass):
        """At N > 1 the direct (IPC) halos must reproduce the NCCL send/recv halos bit for bit."""
        lb = self.lb
        if self.ws == 1 or self.checked_direct:
            return
        self.checked_direct = True
        if self.transport != "ipc":
            self.transport = self.transport if self.transport != "ipc" else "nccl"
            return
        if self.args.emulate:
            self.transport = "ipc (emulated ranks sharing GPU 0, host CG sums; timings meaningless)"
            return
        b = lb.SpinorField(ctx, a.dr)
        lb.apply_dirac(b, gauge, a, mass)
        self.world.set_direct(False)
        c2 = lb.SpinorField(ctx, a.dr)
        lb.apply_dirac(c2, gauge, a, mass)
        lb.axpy(c2, -1.0, b)
        diff = lb.sqnorm(c2)
        c2.close()
        b.close()
        if diff == 0.0:
            self.world.set_direct(True)
            self.transport = "ipc (direct peer-memory halos, checked bit-identical to NCCL send/recv)"
        else:
            self.transport = f"nccl (ipc halos differed from NCCL: |diff|^2 = {diff:.3e})"

    def dphi(self, ctx, gauge, a, b, mass, steps, warmup, clocks=False):
        """Device-resident full Dphi: (ms per step, launches, clock summary)."""
        lb = self.lb
        for _ in range(warmup):
            lb.apply_dirac(b, gauge, a, mass)
        self.barrier(ctx)
        l0 = ctx.kernel_launches()
        clk = ClockSampler(self.local) if clocks else None
        if clk:
            clk.__enter__()
        self.barrier(ctx)
        ctx.event_record(0)
        for _ in range(steps):
            lb.apply_dirac(b, gauge, a, mass)
        ctx.event_record(1)
        self.barrier(ctx)
        if clk:
            clk.__exit__()
        launches = ctx.kernel_launches() - l0
        ms = self.max_over_ranks(ctx.elapsed_ms(0, 1))
        return ms / steps, launches, (clk.summary() if clk else None)

    def eo_hop(self, ctx, gauge, ae, bo, steps, warmup):
        lb = self.lb
        for _ in range(warmup):
            lb.dphi_oe(bo, gauge, ae)
        self.barrier(ctx)
        ctx.event_record(4)
        for _ in range(steps):
            lb.dphi_oe(bo, gauge, ae)
        ctx.event_record(5)
        self.barrier(ctx)
        return self.max_over_ranks(ctx.elapsed_ms(4, 5)) / steps

    def cg(self, ctx, gauge, cfg, dr, real, fmt, peak, plain=False):
        """Time to solution: eo CG on Mhat^dag Mhat (and plain CG on D^dag D).
        The first solve on a field set captures the CUDA graph; the second is
        timed (the graph is built before the solver's start event anyway)."""
        lb = self.lb
        V = int(np.prod(cfg["L"]))
        out = {}
        kinds = [("eo", lb.EVEN, lb.cg_solve_eo)] + ([("plain", lb.FULL, lb.cg_solve_h)] if plain else [])
        for kind, sub, fn in kinds:
            rhs = lb.SpinorField(ctx, dr, sub).randomize(1, 0)
            x = lb.SpinorField(ctx, dr, sub)
            st = lb.CgSettings(cfg["tol"], 20000)
            fn(gauge, cfg["mass"], rhs, st, x)
            self.barrier(ctx)
            o = fn(gauge, cfg["mass"], rhs, st, x)
            secs = self.max_over_ranks(o.seconds)
            if kind == "eo":
                nbytes = (o.iterations * bytes_eo_cg_iter(dr, real, fmt) + 2 * bytes_eo_hop(dr, real, fmt)
                          + 3 * 64 * dr) * V / 2
                solver = "eo CG on Mhat^dag Mhat (even sites)"
            else:
                nbytes = (o.iterations * bytes_h_cg_iter(dr, real, fmt) + 2 * bytes_full_dphi(dr, real, fmt)
                          + 3 * 64 * dr) * V
                solver = "plain CG on D^dag D = g5 D g5 D (the reference's algorithm)"
            out[kind] = {"solver": solver, "tolerance": cfg["tol"], "iterations": o.iterations,
                         "seconds": secs, "true_rel_residual": o.true_rel_residual,
                         "hbm_frac": nbytes / secs / 1e9 / peak / self.ws}
            x.close()
            rhs.close()
        return out

    def measure_config(self, cfg, steps, warmup, plain_cg=False, clocks=False, keep=False):
        """Dphi, eo hop and CG of one config on this rank; returns a dict (and
        the live objects when keep)."""
        lb = self.lb
        ctx, gauge, grid = self.setup(cfg)
        L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
        dr, real = lb.rep_dim(rep, n), lb.rep_is_real(rep)
        fmt, fmt_err = gauge.storage()
        a = lb.SpinorField(ctx, dr).randomize(1, 0)
        b = lb.SpinorField(ctx, dr)
        self.check_direct_halos(ctx, gauge, a, mass)
        ms, launches, clk = self.dphi(ctx, gauge, a, b, mass, steps, warmup, clocks)
        V = int(np.prod(L))
        fps = lb.flops_per_site(lb.DIRAC, dr, real)
        peak, peak_kind = peaks()
        bpsite = bytes_full_dphi(dr, real, fmt)
        achieved = bpsite * V / self.ws / (ms * 1e-3) / 1e9
        ae = lb.SpinorField(ctx, dr, lb.EVEN).randomize(1, 0)
        bo = lb.SpinorField(ctx, dr, lb.ODD)
        hop_ms = self.eo_hop(ctx, gauge, ae, bo, steps, warmup)
        hop_gbs = bytes_eo_hop(dr, real, fmt) * V / 2 / self.ws / (hop_ms * 1e-3) / 1e9
        ae.close()
        bo.close()
        cg = None if self.args.no_cg else self.cg(ctx, gauge, cfg, dr, real, fmt, peak, plain_cg)
        res = {"dphi_ms": ms, "gflops": fps * V / (ms * 1e-3) / 1e9, "launches": launches, "clocks": clk,
               "link_storage": fmt, "link_reconstruction_err": fmt_err, "bytes_per_site": bpsite,
               "achieved_gbs": achieved, "frac": achieved / peak, "peak": peak, "peak_kind": peak_kind,
               "eo_hop_ms": hop_ms, "eo_hop_gbs": hop_gbs, "eo_hop_frac": hop_gbs / peak, "cg": cg,
               "grid": grid, "dr": dr, "real": real, "fps": fps, "V": V}
        if keep:
            return res, (ctx, gauge, a, b)
        b.close()
        a.close()
        gauge.close()
        ctx.close()
        return res


def e2e_measure(run, ctx, gauge, a, b, cfg, fps, V):
    """End to end through the C-ABI with host buffers: every step copies its
    input field from pinned host memory (reference layout), applies Dphi and
    copies the result back (lbcu_dphi_host: the copies of neighbouring steps
    overlap the kernels; PCIe duplex bound)."""
    import torch
    lb = run.lb
    dr = a.dr
    s = lb.init_spinor_random(cfg["L"], dr, 1, 0, grid=decompose(cfg["L"], run.ws) if run.ws > 1 else
                              (1, 1, 1, 1), rank=run.rank)
    nbytes = s.nbytes
    hin = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    hout = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    for h in hin:
        h.numpy()[:] = s.view(np.uint8).reshape(-1)
    # one job of e2e_steps fields (>= 40 so the pipeline's fill and drain,
    # one lone copy each, stay a small share: tools/e2e_probe.py)
    e2e_steps = max(40, min(run.args.steps, 200))
    ins = [hin[k % 2].data_ptr() for k in range(e2e_steps)]
    outs = [hout[k % 2].data_ptr() for k in range(e2e_steps)]
    lb.dphi_host(gauge, cfg["mass"], ins[:4], outs[:4])  # warm-up (buffers, first-touch)
    run.barrier(ctx)
    ctx.event_record(2)
    lb.dphi_host(gauge, cfg["mass"], ins, outs)
    ctx.event_record(3)
    run.barrier(ctx)
    e2e_ms = run.max_over_ranks(ctx.elapsed_ms(2, 3))
    e2e_value = fps * V * e2e_steps / (e2e_ms * 1e-3) / 1e9
    # the result must be the Dphi of the input (checked against the device path)
    got = hout[(e2e_steps - 1) % 2].numpy().view(np.complex128).reshape(s.shape)
    a.upload(s)
    lb.apply_dirac(b, gauge, a, cfg["mass"])
    want = b.download()
    e2e_err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    del want, got
    duplex_ms = duplex_copy_ms(hin, hout, nbytes)
    if not run.args.no_cg:  # time to solution end to end: host rhs in, host solution out
        e2e_cg(run, ctx, gauge, cfg, a.dr, hin[0], hout[0], nbytes)
    return {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "steps": e2e_steps, "ms_per_step": e2e_ms / e2e_steps,
            "api": "lbcu_dphi_host (pinned host buffers, reference layout)",
            "check_rel_err": e2e_err,
            "pcie_bound": {"duplex_copy_ms_per_step": duplex_ms and duplex_ms["both"],
                           "h2d_copy_ms_per_step": duplex_ms and duplex_ms["h2d"],
                           "d2h_copy_ms_per_step": duplex_ms and duplex_ms["d2h"],
                           "frac": duplex_ms["both"] / (e2e_ms / e2e_steps) if duplex_ms else None,
                           "note": "pinned copies of one step's bytes, concurrent H2D + D2H (duplex, "
                                   "±4 % run to run) and each direction alone (the floor); "
                                   "frac = duplex time / e2e ms per step"}}


def e2e_cg(run, ctx, gauge, cfg, dr, hin, hout, nbytes):
    """eo CG through the public API with host buffers: the rhs is uploaded
    from pinned host memory (reference layout, even sites taken), solved, and
    the solution downloaded into pinned host memory, all inside the timed
    region (host clock around the synchronous calls, max over ranks). Stored
    on the run for the `cg` block."""
    lb = run.lb
    rhs = lb.SpinorField(ctx, dr, lb.EVEN)
    x = lb.SpinorField(ctx, dr, lb.EVEN)
    st = lb.CgSettings(cfg["tol"], 20000)
    rhs.upload_ptr(hin.data_ptr())
    lb.cg_solve_eo(gauge, cfg["mass"], rhs, st, x)  # graph capture for these fields
    run.barrier(ctx)
    t0 = time.perf_counter()
    rhs.upload_ptr(hin.data_ptr())
    o = lb.cg_solve_eo(gauge, cfg["mass"], rhs, st, x)
    x.download_ptr(hout.data_ptr())
    t1 = time.perf_counter()
    run.e2e_cg = {"seconds": run.max_over_ranks(t1 - t0), "iterations": o.iterations,
                  "true_rel_residual": o.true_rel_residual, "h2d_bytes": nbytes, "d2h_bytes": nbytes,
                  "api": "SpinorField.upload_ptr + lbcu_cg_solve_eo + download_ptr (pinned host buffers, "
                         "reference layout), host clock"}
    x.close()
    rhs.close()


def run_gpu(args, cfg, cidx):
    run = Run(args)
    ws, rank = run.ws, run.rank
    res, (ctx, gauge, a, b) = run.measure_config(cfg, args.steps, args.warmup, plain_cg=not args.no_plain_cg,
                                                 clocks=True, keep=True)
    e2e = e2e_measure(run, ctx, gauge, a, b, cfg, res["fps"], res["V"])
    if res["cg"] and getattr(run, "e2e_cg", None):
        res["cg"]["eo"]["e2e"] = run.e2e_cg
    for o in (b, a, gauge, ctx):
        o.close()
    try:
        import torch
        torch.cuda.empty_cache()
    except Exception:  # noqa: BLE001
        pass

    # every BASELINE config on this GPU in the same run (the headline one reused)
    table = {}
    if not args.no_all_configs:
        for c in sorted(CONFIGS):
            r = res if c == cidx else run.measure_config(CONFIGS[c], min(args.steps, 100), args.warmup)
            table[str(c)] = {
                "workload": CONFIGS[c]["name"], "grid": r["grid"], "link_storage": r["link_storage"],
                "dphi_ms": r["dphi_ms"], "dphi_gflops_total": r["gflops"], "dphi_frac": r["frac"],
                "dphi_achieved_gbs": r["achieved_gbs"], "bytes_per_site": r["bytes_per_site"],
                "traffic": traffic_from_profiles(f"cfg{c}_dphi_{r['link_storage']}", ws),
                "eo_hop_ms": r["eo_hop_ms"], "eo_hop_frac": r["eo_hop_frac"],
                "eo_cg": r["cg"] and r["cg"]["eo"],
                "reference_cg_iterations": golden_cg_iterations(c) or None}

    # CPU baseline: the unmodified reference on this host (rank 0 at N = 1),
    # in a fresh subprocess after the GPU work (no competing host threads)
    cpu = None
    if ws == 1 and not args.no_cpu:
        gpu_its = {str(cidx): {k: v["iterations"] for k, v in (res["cg"] or {}).items()}}
        leg = run_cpu_leg_subprocess([cidx] + ([c for c in sorted(CONFIGS) if c != cidx] if table else []),
                                     args.cpu_seconds, [cidx], gpu_its)
        if "error" in leg:
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                   "sample": f"failed: {leg['error']}"}
        else:
            cpu = leg[str(cidx)]
            for c, rec in leg.items():
                if c in table:
                    table[c]["cpu_reference_gflops"] = rec["value"]
                    table[c]["cpu_sample"] = rec["sample"]
                    table[c]["speedup_vs_cpu"] = table[c]["dphi_gflops_total"] / rec["value"]
            if res["cg"] and "cg" in cpu:
                for kind in ("eo", "plain"):
                    if kind in cpu["cg"] and kind in res["cg"] and cpu["cg"][kind].get("seconds"):
                        cpu["cg"][kind]["gpu_speedup"] = cpu["cg"][kind]["seconds"] / res["cg"][kind]["seconds"]
                        if "e2e" in res["cg"][kind]:
                            cpu["cg"][kind]["gpu_e2e_speedup"] = (cpu["cg"][kind]["seconds"]
                                                                  / res["cg"][kind]["e2e"]["seconds"])

    if rank == 0:
        peak = res["peak"]
        line = {
            "metric": METRIC, "value": res["gflops"], "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["dphi_ms"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: reference keyed RNG, seed 1 (Haar / near-unit links, Gaussian spinor)",
            "config": config_dict(cfg, ws),
            "halo_transport": run.transport,
            "roofline": {"bound": "hbm", "achieved": res["achieved_gbs"], "peak": peak, "unit": "GB/s",
                         "frac": res["frac"], "peak_kind": res["peak_kind"],
                         "algorithmic_bytes_per_launch": res["bytes_per_site"] * res["V"] / ws,
                         "bytes_per_site": res["bytes_per_site"], "link_storage": res["link_storage"],
                         "link_reconstruction_err": res["link_reconstruction_err"],
                         "survey_model_bytes_per_site": bytes_full_dphi(res["dr"], res["real"], "full"),
                         "kernel": "hop_kernel (full Dphi, both parities)",
                         "kernels_per_step": res["launches"] / args.steps,
                         "traffic": traffic_from_profiles(f"cfg{cidx}_dphi_{res['link_storage']}", ws),
                         "eo_hop": {"ms": res["eo_hop_ms"], "achieved": res["eo_hop_gbs"],
                                    "frac": res["eo_hop_frac"],
                                    "bytes_per_output_site": bytes_eo_hop(res["dr"], res["real"],
                                                                          res["link_storage"]),
                                    "traffic": traffic_from_profiles(f"cfg{cidx}_hop_{res['link_storage']}", ws)}},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(res["launches"]),
            "clocks": res["clocks"],
            "cg": res["cg"],
            "configs": table or None,
        }
        print(json.dumps(line), flush=True)
    if run.dist is not None:
        run.dist.barrier()
        run.dist.destroy_process_group()


def run_regime(args):
    """A stock regime at the paper's 64x32^3 (proj/src/bench.cpp:26-42): Dphi
    on the GPU, checked against the unmodified reference apply_dirac on the
    same host-generated inputs, the eo CG, and the reference on the host."""
    import oracle as O
    import paper_1401_3733_b200 as lb

    cfg = REGIMES[args.regime]
    run = Run(args)
    L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
    dr, real = lb.rep_dim(rep, n), lb.rep_is_real(rep)
    g = lb.init_gauge_random(L, n, rep, 1)
    s = lb.init_spinor_random(L, dr, 1, 0)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T).upload(g)
    fmt, fmt_err = gauge.storage()
    a, b = lb.SpinorField(ctx, dr).upload(s), lb.SpinorField(ctx, dr)
    lb.apply_dirac(b, gauge, a, mass)
    host = O.host_cpu()
    want = O.ref_apply_dirac(L, O.grid_for_threads(L, host["logical_cpus"]), n, rep, 1, mass, g, s)
    err = float(np.linalg.norm(b.download() - want) / np.linalg.norm(want))
    del want, g
    ms, launches, clk = run.dphi(ctx, gauge, a, b, mass, args.steps, args.warmup, clocks=True)
    V = int(np.prod(L))
    fps = lb.flops_per_site(lb.DIRAC, dr, real)
    peak, peak_kind = peaks()
    bps = bytes_full_dphi(dr, real, fmt)
    ach = bps * V / (ms * 1e-3) / 1e9
    ae = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    bo = lb.SpinorField(ctx, dr, lb.ODD)
    hop_ms = run.eo_hop(ctx, gauge, ae, bo, args.steps, args.warmup)
    hop_gbs = bytes_eo_hop(dr, real, fmt) * V / 2 / (hop_ms * 1e-3) / 1e9
    cg = run.cg(ctx, gauge, cfg, dr, real, fmt, peak)
    for o in (ae, bo, b, a, gauge, ctx):
        o.close()
    cpu = None
    if not args.no_cpu:
        grid = O.grid_for_threads_balanced(L, host["logical_cpus"])
        one = O.ref_bench_dirac(L, grid, n, rep, mass, 1, 1, nwarm=0)
        napps = int(max(1, min(200, args.cpu_seconds / 3.0 / max(one, 1e-6))))
        t = O.ref_bench_dirac(L, grid, n, rep, mass, 1, napps, nsamples=3)
        med = statistics.median(t)
        cpu = {"value": fps * V * napps / med / 1e9, "unit": "GFLOP/s", "cores": int(np.prod(grid)),
               "kind": "reference", "sample": f"median of 3 x {napps} apply_dirac, grid {grid}",
               **{k: host[k] for k in ("model", "physical_cores", "reference_isa")}}
    line = {"metric": METRIC, "regime": args.regime, "value": fps * V / (ms * 1e-3) / 1e9, "unit": "GFLOP/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "dtype": "f64",
            "config": config_dict(cfg, 1), "parity_vs_reference_rel_l2": err,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "peak_kind": peak_kind, "bytes_per_site": bps, "link_storage": fmt,
                         "link_reconstruction_err": fmt_err,
                         "eo_hop": {"ms": hop_ms, "achieved": hop_gbs, "frac": hop_gbs / peak}},
            "cg": cg, "cpu_baseline": cpu, "gpu_launches": int(launches), "clocks": clk}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--regime", choices=sorted(REGIMES), help="a stock regime at 64x32^3 instead of a config")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--no-plain-cg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-all-configs", action="store_true", help="skip the per-config table")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU budget per reference sample")
    ap.add_argument("--dense-links", action="store_true", help="store links as dense matrices")
    ap.add_argument("--host-links", action="store_true", help="generate links on the host and upload")
    ap.add_argument("--emulate", action="store_true",
                    help="test the N > 1 flow with every rank on GPU 0 (gloo, IPC world, no NCCL); "
                         "correctness only, the timings are meaningless")
    ap.add_argument("--cpu-leg", help=argparse.SUPPRESS)  # internal: the CPU baseline subprocess
    ap.add_argument("--cpu-cg", default="", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-gpu-its", default="{}", help=argparse.SUPPRESS)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.cpu_leg:
        configs = [int(c) for c in args.cpu_leg.split(",")]
        cgc = [int(c) for c in args.cpu_cg.split(",") if c]
        print(json.dumps(cpu_leg(configs, args.cpu_seconds, cgc, json.loads(args.cpu_gpu_its))), flush=True)
        return
    if args.regime:
        run_regime(args)
        return
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg, args.config)


if __name__ == "__main__":
    main()
