#!/bin/bash
# Usage (GPU box): TAG=r2h bash tools/r2_wps.sh — warp-pair direction split A/B
TAG=${TAG:-r2}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "wps" > gpurun_out/${TAG}_wps_tests.log 2>&1; echo "wps tests rc=$?"
for rep in 1 2; do
  python tools/tune_hop.py --config 3 --steps 50 --sweep LBCU_HOP_WPS=0,1 --sweep LBCU_HOP_WPS_MINB=3,4,5 | grep -v results >> gpurun_out/${TAG}_wps_cfg3.log
  python tools/tune_hop.py --config 4 --steps 100 --sweep LBCU_HOP_WPS=0,1 --sweep LBCU_HOP_WPS_MINB=3,4,5 | grep -v results >> gpurun_out/${TAG}_wps_cfg4.log
  python tools/cg_probe.py --config 3 --reps 2 --sweep LBCU_HOP_WPS=0,1 --sweep LBCU_HOP_WPS_MINB=3,4 >> gpurun_out/${TAG}_wps_cg_cfg3.log
  python tools/cg_probe.py --config 4 --sweep LBCU_HOP_WPS=0,1 --sweep LBCU_HOP_WPS_MINB=3,4,5 >> gpurun_out/${TAG}_wps_cg_cfg4.log
done
