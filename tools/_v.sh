tag=$1; shift; cfgs=$1; shift
for c in $cfgs; do
 for v in base "$@" base; do
  if [ $v = base ]; then lib=paper_1401_3733_b200/liblbcu.so; else lib=paper_1401_3733_b200/liblbcu_$v.so; fi
  echo "== $v" >> gpurun_out/${tag}_cfg$c.log
  LBCU_LIBRARY=$PWD/$lib python tools/tune_hop.py --config $c --steps 50 | head -1 >> gpurun_out/${tag}_cfg$c.log 2>&1
 done
done
