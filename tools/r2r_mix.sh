mkdir -p gpurun_out/r2r
for c in 2 3 4 5; do
  timeout 600 python tools/tune_hop.py --config $c --steps 100 --sweep LBCU_HOP_LS=0 --sweep LBCU_HOP_MIX=0,1,0,1 > gpurun_out/r2r/tune_mix_cfg$c.log 2>&1
  echo "cfg $c rc=$?"; grep -v '^{"config' gpurun_out/r2r/tune_mix_cfg$c.log | tail -4
done
for c in 2 3; do
bash tools/ncu_traffic.sh r2r_mix0 $c LBCU_HOP_LS=0 LBCU_HOP_MIX=0
bash tools/ncu_traffic.sh r2r_mix1 $c LBCU_HOP_LS=0 LBCU_HOP_MIX=1
bash tools/ncu_traffic.sh r2r_ls1 $c LBCU_HOP_LS=1 LBCU_HOP_MIX=0
done
