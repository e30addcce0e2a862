#!/bin/bash
# Usage (GPU box): tools/ncu_traffic.sh NAME CONFIG [ENV=VAL ...]
# L2->SM and DRAM bytes of one full-Dphi launch and one eo-hop launch of
# tools/tune_hop.py (launch 5 = timed full Dphi, 18 = timed eo hop), a short
# metric list instead of --set full.
name=$1; cfg=$2; shift 2
M=gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sector_hit_rate.pct,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,lts__lts2xbar_cycles_active.avg.pct_of_peak_sustained_elapsed
for leg in dphi:5 hop:18; do
  l=${leg%%:*}; k=${leg##*:}
  env "$@" ncu --metrics $M --clock-control none -k regex:hop_kernel -s $k -c 1 --csv \
    --log-file gpurun_out/${name}_cfg${cfg}_${l}.csv python tools/tune_hop.py --config $cfg --steps 10 > /dev/null 2>&1
  python - gpurun_out/${name}_cfg${cfg}_${l}.csv "$name cfg$cfg $l $*" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; out = {}
for r in rows[1:]:
    d = dict(zip(h, r)); out[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
print(sys.argv[2], {k.split(".")[0].replace("l1tex__m_xbar2l1tex_read_bytes", "l2_to_sm").replace("__bytes", ""): " ".join(v) for k, v in out.items()})
PY
done
