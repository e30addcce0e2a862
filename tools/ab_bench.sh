#!/bin/bash
# Usage (GPU box): TAG=x bash tools/ab_bench.sh "<configs>" "<env assignment A>" "<env assignment B>" ...
# A/B bench lines (no CPU leg, no per-config table), alternating the variants
# twice so box drift shows up: gpurun_out/$TAG/ab_cfg<C>_<k>_<rep>.json
TAG=${TAG:-ab}
mkdir -p gpurun_out/$TAG
cfgs=$1; shift
for rep in 1 2; do
  k=0
  for v in "$@"; do
    for c in $cfgs; do
      env $v python bench.py --config $c --no-cpu --no-all-configs --steps 100 \
        > gpurun_out/$TAG/ab_cfg${c}_${k}_${rep}.json 2> gpurun_out/$TAG/ab_cfg${c}_${k}_${rep}.err
      python - "$v" gpurun_out/$TAG/ab_cfg${c}_${k}_${rep}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    r, cg = d["roofline"], d["cg"]
    print(f"{sys.argv[1]:40s} {d['config']['workload']:32s} {r['link_storage']:5s} dphi {d['ms_per_step']:.4f} ms "
          f"frac {r['frac']:.3f} | hop {r['eo_hop']['ms']:.4f} ms frac {r['eo_hop']['frac']:.3f} | "
          f"cg eo {cg['eo']['iterations']} its {cg['eo']['seconds']*1e3:.2f} ms | plain {cg['plain']['seconds']*1e3:.1f} ms "
          f"| {d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']}")
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
      k=$((k+1))
    done
  done
done
