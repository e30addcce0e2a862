#!/bin/bash
# Usage (GPU box): TAG=r2g bash tools/r2_sweep.sh — launch-knob sweeps (register caps, block size)
TAG=${TAG:-r2}
mkdir -p gpurun_out
for rep in 1 2; do
  python tools/tune_hop.py --config 4 --steps 100 --sweep LBCU_HOP_MINB=3,4,1 | grep -v results >> gpurun_out/${TAG}_tune_minb_cfg4.log
  python tools/tune_hop.py --config 3 --steps 50 --sweep LBCU_HOP_MINB=3,4 --sweep LBCU_HOP_BLOCK=64,128 | grep -v results >> gpurun_out/${TAG}_tune_minb_block_cfg3.log
  python tools/tune_hop.py --config 5 --steps 50 --fundamental --sweep LBCU_HOP_BLOCK=64,128 | grep -v results >> gpurun_out/${TAG}_tune_block_cfg5.log
  python tools/cg_probe.py --config 4 --sweep LBCU_HOP_MINB=3,4 >> gpurun_out/${TAG}_cg_minb_cfg4.log
done
