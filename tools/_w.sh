for v in "" _nored _nox _both; do
  LBCU_LIBRARY=$PWD/paper_1401_3733_b200/liblbcu$v.so LBCU_CG_GRAPH=0 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/r03_cgvar$v.csv python tools/cg_probe.py --config 2 --reps 1 --maxit 24 > gpurun_out/r03_cgvar$v.log 2>&1
done
