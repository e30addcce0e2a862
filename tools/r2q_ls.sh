#!/bin/bash
# Usage (GPU box): TAG=r2q bash tools/r2q_ls.sh — A/B of the warp-private link staging (LBCU_HOP_LS)
TAG=${TAG:-r2q}
mkdir -p gpurun_out/$TAG
for c in 2 3 4 5; do
  timeout 600 python tools/tune_hop.py --config $c --steps 100 --sweep LBCU_HOP_LS=0,1,0,1 ${EXTRA:-} > gpurun_out/$TAG/tune_ls_cfg$c.log 2>&1
  echo "cfg $c rc=$?"; grep -v '^{"config' gpurun_out/$TAG/tune_ls_cfg$c.log | tail -4
done
