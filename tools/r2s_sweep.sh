#!/bin/bash
# Usage (GPU box): bash tools/r2s_sweep.sh — link staging (slots per warp: default / nl4 / nl2 library
# variants) x register cap x mixed-parity blocks, configs 2-4
mkdir -p gpurun_out/r2s
P=$PWD/paper_1401_3733_b200
run() { # cfg lib-suffix sweeps...
  c=$1; lib=$2; shift 2
  L=$P/liblbcu${lib}.so
  LBCU_LIBRARY=$L timeout 600 python tools/tune_hop.py --config $c --steps 100 "$@" 2>&1 | grep -v '^{"config' | sed "s/^/cfg$c lib${lib:-_default} /" >> gpurun_out/r2s/sweep_cfg$c.log
}
for rep in 1 2; do
run 3 "" --sweep LBCU_HOP_LS=0,1 --sweep LBCU_HOP_MIX=0,1 --sweep LBCU_HOP_MINB=3
run 3 "_nl4" --sweep LBCU_HOP_LS=1 --sweep LBCU_HOP_MIX=0,1 --sweep LBCU_HOP_MINB=3,4
run 3 "_nl2" --sweep LBCU_HOP_LS=1 --sweep LBCU_HOP_MIX=0,1 --sweep LBCU_HOP_MINB=3,4
run 2 "" --sweep LBCU_HOP_LS=0,1 --sweep LBCU_HOP_MIX=0,1
run 2 "_nl4" --sweep LBCU_HOP_LS=1 --sweep LBCU_HOP_MIX=0,1
run 2 "_nl2" --sweep LBCU_HOP_LS=1 --sweep LBCU_HOP_MIX=0,1
run 4 "" --sweep LBCU_HOP_LS=0,1 --sweep LBCU_HOP_MIX=0,1 --sweep LBCU_HOP_MINB=3,4
run 4 "_nl4" --sweep LBCU_HOP_LS=1 --sweep LBCU_HOP_MIX=0,1 --sweep LBCU_HOP_MINB=3,4
run 4 "_nl2" --sweep LBCU_HOP_LS=1 --sweep LBCU_HOP_MIX=0,1 --sweep LBCU_HOP_MINB=3,4
done
cat gpurun_out/r2s/sweep_cfg*.log | python -c "
import sys, json
for l in sys.stdin:
    p = l.split(' ', 2)
    try: d = json.loads(p[2])
    except Exception: print(l.strip()[:200]); continue
    k = {a: b for a, b in d.items() if a.startswith('LBCU')}
    print(p[0], p[1], k, 'full %.4f hop %.4f err %.1e' % (d['full_ms'], d['hop_ms'], d['err']))
"
