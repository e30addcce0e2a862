"""Time lbcu_dphi_host (pinned host buffers, reference layout) against the
number of fields per call, to separate the pipeline's steady state from its
fill and drain. python tools/e2e_probe.py [--config 2]"""
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
    ap.add_argument("--counts", default="2,4,10,20,40,80")
    args = ap.parse_args()
    import torch
    cfg = bench.CONFIGS[args.config]
    L, n, rep, mass = cfg["L"], cfg["n"], cfg["rep"], cfg["mass"]
    dr = lb.rep_dim(rep, n)
    ctx = lb.Context(L)
    gauge = lb.GaugeField(ctx, n, rep, lb.ANTIPERIODIC_T)
    gauge.generate(1)
    s = lb.init_spinor_random(L, dr, 1, 0)
    nbytes = s.nbytes
    hin = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    hout = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    for h in hin:
        h.numpy()[:] = s.view(np.uint8).reshape(-1)
    lb.dphi_host(gauge, mass, [hin[0].data_ptr()] * 2, [hout[0].data_ptr()] * 2)
    for k in [int(v) for v in args.counts.split(",")]:
        ins = [hin[j % 2].data_ptr() for j in range(k)]
        outs = [hout[j % 2].data_ptr() for j in range(k)]
        ts = []
        for _ in range(3):
            ctx.event_record(0)
            lb.dphi_host(gauge, mass, ins, outs)
            ctx.event_record(1)
            ts.append(ctx.elapsed_ms(0, 1))
        ms = min(ts)
        print(json.dumps({"fields": k, "ms": ms, "ms_per_field": ms / k,
                          "gbs_per_dir": nbytes * k / ms / 1e6}), flush=True)


if __name__ == "__main__":
    main()
