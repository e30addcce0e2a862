"""Generate tests/golden/cg_cfg{1..5}.npz: the reference's CG iteration counts
at BASELINE.json's FULL sizes, plain and even-odd, from the UNMODIFIED
reference (oracle/_ref/liblatbench_ref.so) on this container's host cores.

    make -C oracle ref && python tests/golden/make_fullsize_cg.py [configs...]

* plain: ``cg_solve(make_h_operator(...))`` on H = g5 D g5 D
  (/root/reference/proj/src/solver.cpp:9-22,24-82);
* eo: the same ``cg_solve`` driven by the LinearOp g5 Mhat g5 Mhat composed
  from the reference ``apply_dirac`` (oracle/ref_shim.cpp ``ref_cg_eo``,
  SURVEY.md §0), rhs = the even part of spinor field 0.

Inputs are the BASELINE configs exactly (seed 1, antiperiodic t; config 3's
near-unit links U = exp(i 0.3 H) from ``ref_gauge_near_unit``). Config 3
takes ~15 min (eo) + ~15 min (plain) on 8 cores and ~35 GB of host memory.
One file per config, written as soon as it is done.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402

CONFIGS = {  # BASELINE.json configs[0..4] (bench.CONFIGS)
    1: dict(L=[8, 8, 8, 8], n=3, rep=O.FUNDAMENTAL, mass=0.1, links="haar", tol=1e-10),
    2: dict(L=[32, 32, 32, 32], n=2, rep=O.FUNDAMENTAL, mass=0.05, links="haar", tol=1e-10),
    3: dict(L=[96, 48, 48, 48], n=3, rep=O.FUNDAMENTAL, mass=0.02, links="near_unit", tol=1e-12),
    4: dict(L=[40, 40, 40, 40], n=2, rep=O.ADJOINT, mass=0.05, links="haar", tol=1e-10),
    5: dict(L=[64, 32, 32, 32], n=4, rep=O.ANTISYMMETRIC, mass=0.1, links="haar", tol=1e-10),
}


def run(c):
    cfg = CONFIGS[c]
    L, n, rep, m, tol = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"], cfg["tol"]
    dr = O.rep_dim(rep, n)
    nthreads = os.cpu_count() or 1
    grid = O.grid_for_threads_balanced(L, nthreads)
    t0 = time.time()
    if cfg["links"] == "near_unit":
        g = O.ref_gauge_near_unit(L, n, 0.3, 1)
    else:
        g = O.ref_gauge_random(L, n, rep, 1)
    s = O.ref_spinor_random(L, dr, 1, 0)
    print(f"cfg{c}: inputs {time.time() - t0:.1f} s, grid {grid}", flush=True)
    out = dict(lattice=np.array(L), n=n, rep=rep, mass=m, tol=tol, grid=np.array(grid),
               threads=nthreads)
    for kind, fn in (("eo", O.ref_cg_eo), ("h", O.ref_cg_h)):
        t0 = time.time()
        r = fn(L, grid, n, rep, 1, m, g, s, tol, 5000)
        out[f"{kind}_iterations"] = r["iterations"]
        out[f"{kind}_rel"] = r["rel_residual"]
        out[f"{kind}_true"] = r["true_rel_residual"]
        out[f"{kind}_history"] = r["history"]
        out[f"{kind}_seconds"] = r["seconds"]
        print(f"cfg{c} {kind}: {r['iterations']} iterations, true rel residual "
              f"{r['true_rel_residual']:.3e}, cg {r['seconds']:.1f} s (wall {time.time() - t0:.1f} s)",
              flush=True)
        del r
    np.savez_compressed(os.path.join(HERE, f"cg_cfg{c}.npz"), **out)
    print(f"cg_cfg{c}.npz written", flush=True)


def main():
    which = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 5, 3]
    for c in which:
        run(c)


if __name__ == "__main__":
    main()
