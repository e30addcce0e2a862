#!/bin/bash
# Usage (on the GPU box): tools/profile_round.sh TAG [configs...]
# One `ncu --set full` capture of the full Dphi and of the eo hop per config
# (tools/tune_hop.py, 10 timed steps: full-Dphi launches 0..12, eo hop 13..25),
# exported as CSV under gpurun_out/ (tools/ncu_capture.sh); summarise with
#   python profiles/ncu_summary.py gpurun_out/<TAG>_cfgN_{dphi,hop}_raw.csv
set -e
tag=$1; shift
cfgs=${*:-2 3 4 5}
for c in $cfgs; do
  extra=""
  [ "$c" = 5 ] && extra="--fundamental"
  bash tools/ncu_capture.sh ${tag}_cfg${c}_dphi 5 1 -- python tools/tune_hop.py --config $c --steps 10 $extra
  bash tools/ncu_capture.sh ${tag}_cfg${c}_hop 18 1 -- python tools/tune_hop.py --config $c --steps 10 $extra
done
