#!/bin/bash
# Usage (GPU box): TAG=r2j bash tools/r2_fused.sh — fused Mhat sweep: parity, then CG A/B
TAG=${TAG:-r2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "fused" > gpurun_out/${TAG}_fused_tests.log 2>&1; echo "fused tests rc=$?"; tail -3 gpurun_out/${TAG}_fused_tests.log
for rep in 1 2; do
  for c in 3 2 4; do
    timeout 600 python tools/cg_probe.py --config $c --reps 3 --sweep LBCU_CG_FUSED_MHAT=0,1 --sweep LBCU_FUSED_L2MB=12,24,48 >> gpurun_out/${TAG}_fused_cg.log
  done
done
