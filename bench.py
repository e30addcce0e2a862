#!/usr/bin/env python
"""Benchmark driver: Dphi GFLOP/s and CG time-to-solution on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

Mirrors the reference's Dirac kernel benchmark (proj/src/bench.cpp:190-248:
FLOPs = flops_per_site x global volume x applications, exact integers) on
BASELINE.json's configs (default: configs[1], SU(2) fundamental 32^4, the
config the metric is quoted on at N = 1). A step is one full Dphi
application over the lattice, inputs resident in HBM. One JSON line on rank 0.

Under torchrun (N > 1) each rank owns one GPU and one sub-lattice (T split
first, then Z: SURVEY.md §8e). Halos go straight from the pack kernel into
the neighbour's receive arena over NVLink (the library's IPC world), checked
once per run bit for bit against NCCL send/recv halos (LBCU_TRANSPORT=nccl
forces NCCL); CG sums use NCCL. Time is the max over ranks of CUDA-event
time.

--impl reference times the reference's own CPU apply_dirac (oracle/_ref, the
unmodified latbench compiled from its sources) with all host threads on the
same config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
METRIC = "Dphi GFLOP/s and CG time-to-solution vs GPUs (1/2/4/8), % of HBM roofline"


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


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def link_bytes(dr, real, fmt="full"):
    """Bytes of one link as stored on the device (links.cuh)."""
    return {"full": dr * dr * (8 if real else 16), "su2": 32, "r12": 96, "as4": 256, "as4r": 288}[fmt]


def bytes_full_dphi(dr, real, fmt="full"):
    """SURVEY.md §8(d) compulsory bytes per site of a full Dphi: spinor in + out
    (128 d) + each of the 4 links of the site once; with fmt = "full" this is
    SURVEY's 128 d + 32 c d^2."""
    return 128 * dr + 4 * link_bytes(dr, real, fmt)


def bytes_eo_hop(dr, real, fmt="full"):  # per output site: 128 d + 8 links
    return 128 * dr + 8 * link_bytes(dr, real, fmt)


def bytes_eo_cg_iter(dr, real, fmt="full"):  # per even site 4 B_hop + 11 * 64 d
    return 4 * bytes_eo_hop(dr, real, fmt) + 11 * 64 * dr


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

    return {mode: min(run(mode) for _ in range(3)) for mode in ("both", "h2d", "d2h")}

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


def traffic_from_profiles(key):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(key)
    except Exception:
        return None


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    import oracle as O

    ws, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs the CPU reference (its threads use every core)
    L, n, rep = cfg["L"], cfg["n"], cfg["rep"]
    dr = O.rep_dim(rep, n)
    nthreads = os.cpu_count() or 1
    grid = O.grid_for_threads_balanced(L, nthreads)
    cores = int(np.prod(grid))
    fps = O.ref_flops_per_site(O.DIRAC, dr, O.rep_is_real(rep))
    V = int(np.prod(L))
    # each step = one apply_dirac (bench.cpp:209) over the whole lattice
    O.ref_bench_dirac(L, grid, n, rep, cfg["mass"], 1, max(1, args.warmup))
    secs = O.ref_bench_dirac(L, grid, n, rep, cfg["mass"], 1, args.steps)
    value = fps * V * args.steps / secs / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference keyed RNG, seed 1 (Haar links, Gaussian spinor)",
        "config": {"workload": cfg["name"], "lattice": L, "group_rank": n, "rep": rep, "mass": cfg["mass"],
                   "worker_grid": grid},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                         "sample": f"{args.steps} apply_dirac on {cfg['name']}, {cores} worker threads"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm
def run_gpu(args, cfg):
    import paper_1401_3733_b200 as lb

    ws, rank, local = dist_env()
    L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
    grid = decompose(L, ws) if ws > 1 else [1, 1, 1, 1]
    dist = None
    world = None
    if ws > 1:
        import torch
        import torch.distributed as dist

        import uuid
        if args.emulate:  # test mode: every rank on GPU 0, gloo, no NCCL at all
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [(None if args.emulate else lb.World.nccl_unique_id(), f"/lbcu_{uuid.uuid4().hex[:16]}")
               if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid, shm_name = obj[0]
        # halos: direct peer-memory stores by the pack kernel (IPC world; NCCL
        # for the CG sums), checked below against NCCL send/recv halos;
        # LBCU_TRANSPORT=nccl forces the NCCL world
        transport = os.environ.get("LBCU_TRANSPORT", "ipc")
        world = None
        if transport == "ipc":
            try:
                world = lb.World.ipc(ws, rank, shm_name, uid)
            except Exception as e:  # noqa: BLE001
                transport = f"nccl (ipc world unavailable: {e})"
        if world is None:
            if args.emulate:
                raise SystemExit(f"--emulate needs the IPC world: {transport}")
            world = lb.World.nccl(ws, rank, uid)
    dr = lb.rep_dim(rep, n)
    real = lb.rep_is_real(rep)
    links = {"haar": lb.LINKS_HAAR, "near_unit": lb.LINKS_NEAR_UNIT}[cfg["links"]]
    ctx = lb.Context(L, grid, rank, local if ws > 1 else 0, world)
    s = lb.init_spinor_random(L, dr, 1, 0, grid=grid, rank=rank)
    # links: the reference's keyed generator evaluated on the device (seed 1,
    # keyed by global site: identical for any decomposition). SU(4) AS links
    # are kept as their fundamental elements and represented in-kernel.
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T)
    if args.dense_links:
        gauge.set_compact(False)
    if args.host_links:
        gauge.upload(lb.init_gauge_random(L, n, rep, 1, grid=grid, rank=rank, links=links, eps=0.3))
    else:
        gauge.generate(1, links=links, eps=0.3)
    fmt, fmt_err = gauge.storage()
    a = lb.SpinorField(ctx, dr).upload(s)
    b = lb.SpinorField(ctx, dr)
    if ws > 1 and transport == "ipc" and args.emulate:
        transport = "ipc (emulated ranks sharing GPU 0, host CG sums; timings meaningless)"
    elif ws > 1 and transport == "ipc":
        # the direct halos must reproduce the NCCL send/recv halos bit for bit
        lb.apply_dirac(b, gauge, a, mass)
        world.set_direct(False)
        c2 = lb.SpinorField(ctx, dr)
        lb.apply_dirac(c2, gauge, a, mass)
        lb.axpy(c2, -1.0, b)
        diff = lb.sqnorm(c2)
        del c2
        if diff == 0.0:
            world.set_direct(True)
            transport = "ipc (direct peer-memory halos, checked bit-identical to NCCL send/recv)"
        else:
            transport = f"nccl (ipc halos differed from NCCL: |diff|^2 = {diff:.3e})"
    elif ws > 1:
        transport = transport if transport != "ipc" else "nccl"

    def barrier():
        ctx.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.emulate else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident Dphi ------------------------------------------------
    for _ in range(args.warmup):
        lb.apply_dirac(b, gauge, a, mass)
    barrier()
    l0 = ctx.kernel_launches()
    with ClockSampler(local) as clk:
        barrier()
        ctx.event_record(0)
        for _ in range(args.steps):
            lb.apply_dirac(b, gauge, a, mass)
        ctx.event_record(1)
        barrier()
    launches = ctx.kernel_launches() - l0
    ms = max_over_ranks(ctx.elapsed_ms(0, 1))
    V = int(np.prod(L))
    fps = lb.flops_per_site(lb.DIRAC, dr, real)
    flops = fps * V * args.steps
    value = flops / (ms * 1e-3) / 1e9
    peak, peak_kind = peaks()
    bpsite = bytes_full_dphi(dr, real, fmt)  # links counted as stored
    per_launch_bytes = bpsite * V / ws  # one Dphi kernel per rank per step (N = 1: a single launch)
    kernels_per_step = launches / args.steps
    achieved = bpsite * V / ws / (ms * 1e-3 / args.steps) / 1e9

    # ---- the eo hop alone (the CG's dominant kernel) ------------------------
    ae = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    bo = lb.SpinorField(ctx, dr, lb.ODD)
    for _ in range(args.warmup):
        lb.dphi_oe(bo, gauge, ae)
    barrier()
    ctx.event_record(4)
    for _ in range(args.steps):
        lb.dphi_oe(bo, gauge, ae)
    ctx.event_record(5)
    barrier()
    hop_ms = max_over_ranks(ctx.elapsed_ms(4, 5)) / args.steps
    hop_gbs = bytes_eo_hop(dr, real, fmt) * V / 2 / ws / (hop_ms * 1e-3) / 1e9

    # ---- end to end through the C-ABI with host buffers ---------------------
    # every step copies its input field from pinned host memory (reference
    # layout), applies Dphi and copies the result back (lbcu_dphi_host: the
    # copies of neighbouring steps overlap the kernels; PCIe duplex bound)
    import torch
    nbytes = s.nbytes
    hin = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    hout = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    for h in hin:
        h.numpy()[:] = s.view(np.uint8).reshape(-1)
    # one job of e2e_steps fields (>= 40 so the pipeline's fill and drain,
    # one lone copy each, stay a small share: tools/e2e_probe.py)
    e2e_steps = max(40, min(args.steps, 200))
    ins = [hin[k % 2].data_ptr() for k in range(e2e_steps)]
    outs = [hout[k % 2].data_ptr() for k in range(e2e_steps)]
    lb.dphi_host(gauge, mass, ins[:4], outs[:4])  # warm-up (buffers, first-touch)
    barrier()
    ctx.event_record(2)
    lb.dphi_host(gauge, mass, ins, outs)
    ctx.event_record(3)
    barrier()
    e2e_ms = max_over_ranks(ctx.elapsed_ms(2, 3))
    e2e_value = fps * V * e2e_steps / (e2e_ms * 1e-3) / 1e9
    # the result must be the Dphi of the input (spot check against the device path)
    got = hout[(e2e_steps - 1) % 2].numpy().view(np.complex128).reshape(s.shape)
    lb.apply_dirac(b, gauge, a, mass)
    e2e_err = float(np.linalg.norm(got - b.download()) / np.linalg.norm(got))
    duplex_ms = duplex_copy_ms(hin, hout, nbytes)

    # ---- CG time to solution (even-odd preconditioned, D^dag D) -------------
    cg = None
    if not args.no_cg:
        rhs = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
        st = lb.CgSettings(cfg["tol"], 20000)
        lb.cg_solve_eo(gauge, mass, rhs, st)  # builds and caches the CUDA graph
        barrier()
        o = lb.cg_solve_eo(gauge, mass, rhs, st)
        secs = max_over_ranks(o.seconds)
        cg_bytes = (o.iterations * bytes_eo_cg_iter(dr, real, fmt) + 2 * bytes_eo_hop(dr, real, fmt)
                    + 3 * 64 * dr) * V / 2
        cg = {"solver": "eo CG on Mhat^dag Mhat", "tolerance": cfg["tol"], "iterations": o.iterations,
              "seconds": secs, "true_rel_residual": o.true_rel_residual,
              "hbm_frac": cg_bytes / secs / 1e9 / peak / ws}

    # ---- CPU baseline (reference, rank 0 at N = 1, bounded sample) ----------
    cpu = None
    if ws == 1 and not args.no_cpu:
        try:
            import oracle as O
            nthreads = os.cpu_count() or 1
            cgrid = O.grid_for_threads_balanced(L, nthreads)
            one = O.ref_bench_dirac(L, cgrid, n, rep, mass, 1, 1)
            napps = int(max(1, min(200, args.cpu_seconds / max(one, 1e-6))))
            secs = O.ref_bench_dirac(L, cgrid, n, rep, mass, 1, napps)
            cpu = {"value": fps * V * napps / secs / 1e9, "unit": "GFLOP/s", "cores": int(np.prod(cgrid)),
                   "kind": "reference",
                   "sample": f"{napps} apply_dirac of the unmodified reference on {cfg['name']} "
                             f"({int(np.prod(cgrid))} worker threads, grid {cgrid})"}
        except Exception as e:  # the CPU baseline is reported, not required
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: reference keyed RNG, seed 1 (Haar / near-unit links, Gaussian spinor)",
            "config": {"workload": cfg["name"], "lattice_TXYZ": L, "group_rank": n, "rep": rep, "dr": dr,
                       "mass": mass, "bc": "periodic space, antiperiodic time", "grid": grid,
                       "parallelism": f"domain decomposition {grid}",
                       "halo_transport": transport if ws > 1 else "none (one rank)",
                       "l2": f"inputs larger than L2 ({(bpsite * V) / 1e6:.0f} MB touched per step vs 126 MB)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": per_launch_bytes,
                         "bytes_per_site": bpsite,
                         "link_storage": fmt, "link_reconstruction_err": fmt_err,
                         "survey_model_bytes_per_site": bytes_full_dphi(dr, real, "full"),
                         "kernel": "hop_kernel (full Dphi, both parities)",
                         "kernels_per_step": kernels_per_step,
                         "traffic": traffic_from_profiles(f"cfg{args.config}_dphi_{fmt}"),
                         "eo_hop": {"ms": hop_ms, "achieved": hop_gbs, "frac": hop_gbs / peak,
                                    "bytes_per_output_site": bytes_eo_hop(dr, real, fmt),
                                    "traffic": traffic_from_profiles(f"cfg{args.config}_hop_{fmt}")}},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes, "steps": e2e_steps, "ms_per_step": e2e_ms / e2e_steps,
                    "api": "lbcu_dphi_host (pinned host buffers, reference layout)",
                    "check_rel_err": e2e_err,
                    "pcie_bound": {"duplex_copy_ms_per_step": duplex_ms and duplex_ms["both"],
                                   "h2d_copy_ms_per_step": duplex_ms and duplex_ms["h2d"],
                                   "d2h_copy_ms_per_step": duplex_ms and duplex_ms["d2h"],
                                   "frac": duplex_ms["both"] / (e2e_ms / e2e_steps) if duplex_ms else None,
                                   "note": "pinned copies of one step's bytes, concurrent H2D + D2H (duplex, "
                                           "±4 % run to run) and each direction alone (the floor); "
                                           "frac = duplex time / e2e ms per step"}},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "cg": cg,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dense-links", action="store_true", help="store links as dense matrices")
    ap.add_argument("--host-links", action="store_true", help="generate links on the host and upload")
    ap.add_argument("--emulate", action="store_true",
                    help="test the N > 1 flow with every rank on GPU 0 (gloo, IPC world, no NCCL); "
                         "correctness only, the timings are meaningless")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_gpu(args, cfg)


if __name__ == "__main__":
    main()
