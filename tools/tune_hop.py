"""Sweep Dslash launch knobs (environment variables read by liblbcu.so) on one config.

    python tools/tune_hop.py --config 3 --sweep LBCU_HOP_SCHED=0,1 --sweep LBCU_HOP_L2MB=16,32,64

Prints ms and GB/s (links counted as stored) per full Dphi and per eo hop for
every combination, and checks each variant's output against the first one.
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1401_3733_b200 as lb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--sweep", action="append", default=[], help="NAME=v1,v2,...")
    ap.add_argument("--dense-links", action="store_true")
    ap.add_argument("--fundamental", action="store_true", help="upload fundamental links (SU(4) AS)")
    ap.add_argument("--lattice", default=None, help="T,X,Y,Z overriding the config's lattice")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
    if args.lattice:
        L = [int(v) for v in args.lattice.split(",")]
    dr = lb.rep_dim(rep, n)
    real = lb.rep_is_real(rep)
    links = {"haar": lb.LINKS_HAAR, "near_unit": lb.LINKS_NEAR_UNIT}[cfg["links"]]
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T)
    if args.dense_links:
        gauge.set_compact(False)
    if args.fundamental:
        gauge.upload_fundamental(lb.init_gauge_random(L, n, lb.FUNDAMENTAL, 1, links=links))
    else:
        gauge.upload(lb.init_gauge_random(L, n, rep, 1, links=links))
    fmt = gauge.storage()[0]
    s = lb.init_spinor_random(L, dr, 1, 0)
    a = lb.SpinorField(ctx, dr).upload(s)
    b = lb.SpinorField(ctx, dr)
    ae = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    bo = lb.SpinorField(ctx, dr, lb.ODD)
    V = int(np.prod(L))
    bfull = bench.bytes_full_dphi(dr, real, fmt) * V
    bhop = bench.bytes_eo_hop(dr, real, fmt) * V / 2
    names = [sw.split("=")[0] for sw in args.sweep]
    values = [sw.split("=")[1].split(",") for sw in args.sweep]
    ref = None
    res = []
    for combo in itertools.product(*values) if values else [()]:
        for k, v in zip(names, combo):
            os.environ[k] = v
        r = dict(zip(names, combo), fmt=fmt)
        try:
            for _ in range(3):
                lb.apply_dirac(b, gauge, a, mass)
            ctx.synchronize()
            ctx.event_record(0)
            for _ in range(args.steps):
                lb.apply_dirac(b, gauge, a, mass)
            ctx.event_record(1)
            t_full = ctx.elapsed_ms(0, 1) / args.steps
            for _ in range(3):
                lb.dphi_oe(bo, gauge, ae)
            ctx.event_record(2)
            for _ in range(args.steps):
                lb.dphi_oe(bo, gauge, ae)
            ctx.event_record(3)
            t_hop = ctx.elapsed_ms(2, 3) / args.steps
            out = b.download()
            if ref is None:
                ref = out
            err = float(np.linalg.norm(out - ref) / np.linalg.norm(ref))
            r.update(full_ms=t_full, full_gbs=bfull / t_full / 1e6, hop_ms=t_hop,
                     hop_gbs=bhop / t_hop / 1e6, err=err)
        except Exception as e:  # noqa: BLE001
            r.update(error=str(e))
        res.append(r)
        print(json.dumps(r), flush=True)
    print(json.dumps({"config": cfg["name"], "results": res}))


if __name__ == "__main__":
    main()
