"""Sweep Dslash launch variants (register cap / min blocks per SM) on one config.

    python tools/tune_hop.py --config 2 [--steps 50]

Prints ms per full Dphi and per eo hop for every variant and checks each
variant's output against the first variant.
"""
import argparse
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
    ap.add_argument("--minb", default="1,3")
    ap.add_argument("--compact", default="0,1")
    ap.add_argument("--s2", default=None, help="LBCU_HOP_S2 values to sweep (spin-split kernel)")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
    dr = lb.rep_dim(rep, n)
    real = lb.rep_is_real(rep)
    links = {"haar": lb.LINKS_HAAR, "near_unit": lb.LINKS_NEAR_UNIT}[cfg["links"]]
    ctx = lb.Context(L)
    links_host = lb.init_gauge_random(L, n, rep, 1, links=links)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T)
    s = lb.init_spinor_random(L, dr, 1, 0)
    a = lb.SpinorField(ctx, dr).upload(s)
    b = lb.SpinorField(ctx, dr)
    ae = lb.SpinorField(ctx, dr, lb.EVEN).upload(s)
    bo = lb.SpinorField(ctx, dr, lb.ODD)
    V = int(np.prod(L))
    bfull = bench.bytes_full_dphi(dr, real) * V
    bhop = (128 * dr + 64 * (1 if real else 2) * dr * dr) * V / 2
    ref = None
    res = []
    for cp in [int(x) for x in args.compact.split(",")]:
      os.environ["LBCU_GAUGE_COMPACT"] = str(cp)
      gauge.upload(links_host)
      fmt = gauge.storage()
      sweep = [(mb, s2) for mb in [int(x) for x in args.minb.split(",")]
               for s2 in ([int(x) for x in args.s2.split(",")] if args.s2 else [None])]
      for mb, s2 in sweep:
        if True:
            os.environ["LBCU_HOP_MINB"] = str(mb)
            if s2 is not None:
                os.environ["LBCU_HOP_S2"] = str(s2)
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
                r = dict(compact=cp, fmt=fmt, minb=mb, s2=s2, full_ms=t_full, full_gbs=bfull / t_full / 1e6,
                         hop_ms=t_hop, hop_gbs=bhop / t_hop / 1e6, err=err)
            except Exception as e:  # noqa: BLE001
                r = dict(minb=mb, error=str(e))
            res.append(r)
            print(json.dumps(r), flush=True)
    print(json.dumps({"config": cfg["name"], "results": res}))


if __name__ == "__main__":
    main()
