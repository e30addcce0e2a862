#!/bin/bash
# Usage (GPU box): bash tools/r2v_sweep.sh "<lib suffixes>" "<configs>" — A/B of library variants (tools/build_variant.sh)
mkdir -p gpurun_out/r2v
P=$PWD/paper_1401_3733_b200
for rep in 1 2; do
for c in $2; do
for lib in $1; do
  [ "$lib" = default ] && L=$P/liblbcu.so || L=$P/liblbcu_$lib.so
  LBCU_LIBRARY=$L timeout 600 python tools/tune_hop.py --config $c --steps 100 2>&1 | grep -v '^{"config' | sed "s/^/cfg$c $lib /" | tee -a gpurun_out/r2v/sweep.log | cut -c1-200
done; done; done
