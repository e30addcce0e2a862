"""Time the eo CG solve (and its four hop kernels per iteration) on one config
for A/B runs of environment knobs: python tools/cg_probe.py --config 2 --sweep LBCU_HOP_PFE=0,1,2"""
import argparse
import itertools
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1401_3733_b200 as lb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sweep", action="append", default=[])
    ap.add_argument("--maxit", type=int, default=20000, help="cap (timing experiments: non-convergence ignored)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
    dr = lb.rep_dim(rep, n)
    links = {"haar": lb.LINKS_HAAR, "near_unit": lb.LINKS_NEAR_UNIT}[cfg["links"]]
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T)
    gauge.generate(1, links=links, eps=0.3)
    rhs = lb.SpinorField(ctx, dr, lb.EVEN).upload(lb.init_spinor_random(L, dr, 1, 0))
    x = lb.SpinorField(ctx, dr, lb.EVEN)  # one solution field: the cached CUDA graph is reused
    names = [sw.split("=")[0] for sw in args.sweep]
    values = [sw.split("=")[1].split(",") for sw in args.sweep]
    for combo in itertools.product(*values) if values else [()]:
        for k, v in zip(names, combo):
            os.environ[k] = v
        st = lb.CgSettings(cfg["tol"], args.maxit)

        def solve():
            try:
                return lb.cg_solve_eo(gauge, mass, rhs, st, x)
            except lb.NonConvergence:  # capped timing runs
                return None

        solve()  # graph built for this setting
        res = [solve() for _ in range(args.reps)]
        best = min((r.seconds for r in res if r is not None), default=float("nan"))
        o = solve()
        print(json.dumps({**dict(zip(names, combo)), "config": args.config, "cg_s": best,
                          "iterations": getattr(o, "iterations", None),
                          "true_rel_residual": getattr(o, "true_rel_residual", None)}), flush=True)


if __name__ == "__main__":
    main()
