#!/bin/bash
# Usage (GPU box): TAG=r2f bash tools/r2_profile.sh
# The default bench line (config 3) + the reference arm, the ncu launch list
# of the same bench command (GPU legs only), one ncu --set full capture of the
# full Dphi and the eo hop of config 3 (tools/profile_round.sh), and the three
# stock regimes at 64x32^3.
TAG=${TAG:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg3.json 2> gpurun_out/${TAG}_bench_cfg3.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_cfg3.json 2>&1; echo "ref rc=$?"
for r in comms balance compute; do
  timeout 900 python bench.py --regime $r --steps 100 > gpurun_out/${TAG}_regime_$r.json 2> gpurun_out/${TAG}_regime_$r.err
  echo "regime $r rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches_cfg3.csv python bench.py --no-cpu --no-all-configs --steps 10 > /dev/null 2>&1
echo "launches rc=$?"
timeout 1200 bash tools/profile_round.sh $TAG 3; echo "profile rc=$?"
