#!/bin/bash
# Usage (on the GPU box): tools/round_measure.sh TAG
# Bench lines for all five configs, the ncu launch list of the default bench
# (CG kernels visible: LBCU_CG_GRAPH=0) and one ncu --set full capture of the
# full Dphi and the eo hop per config (tools/profile_round.sh).
tag=$1
for c in 1 2 3 4 5; do
  python bench.py --config $c > gpurun_out/${tag}_bench_cfg$c.json 2> gpurun_out/${tag}_bench_cfg$c.err
  echo "bench cfg$c rc=$?"
done
python bench.py --impl reference --config 2 --steps 5 --warmup 3 > gpurun_out/${tag}_bench_reference_cfg2.json 2>&1
LBCU_CG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches_cfg2.csv python bench.py --config 2 --no-cpu --steps 10 > /dev/null 2>&1
echo "launches rc=$?"
bash tools/profile_round.sh $tag 2 3 4 5
echo "profile rc=$?"
