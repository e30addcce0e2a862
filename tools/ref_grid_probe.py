"""Time the unmodified reference's apply_dirac (oracle/_ref) on config 2 for
several worker grids of the host's cores, to pick a fair CPU baseline.
Test infrastructure (oracle/): python tools/ref_grid_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402

L, n, rep, m = [32, 32, 32, 32], 2, 0, 0.05
for grid in ([16, 1, 1, 1], [2, 2, 2, 2], [1, 1, 4, 4]) * 2:
    O.ref_bench_dirac(L, grid, n, rep, m, 1, 2)
    secs = O.ref_bench_dirac(L, grid, n, rep, m, 1, 30)
    fps = O.ref_flops_per_site(O.DIRAC, 2, False)
    print(json.dumps({"grid": grid, "ms_per_dphi": secs / 30 * 1e3,
                      "gflops": fps * 32 ** 4 * 30 / secs / 1e9}), flush=True)
