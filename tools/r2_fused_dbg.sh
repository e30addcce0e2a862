#!/bin/bash
# bisect the fused-Mhat crash: small lattice graph/no-graph, then config 2
cat > /tmp/f.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import bench, paper_1401_3733_b200 as lb
c = int(sys.argv[1])
cfg = bench.CONFIGS[c]
ctx = lb.Context(cfg["L"])
g = lb.GaugeField(ctx, cfg["n"], cfg["rep"], lb.ANTIPERIODIC_T).generate(1, links={"haar": lb.LINKS_HAAR, "near_unit": lb.LINKS_NEAR_UNIT}[cfg["links"]])
dr = lb.rep_dim(cfg["rep"], cfg["n"])
e = lb.SpinorField(ctx, dr, lb.EVEN).randomize(1, 0)
o = lb.SpinorField(ctx, dr, lb.EVEN)
print("mhat", flush=True)
lb.mhat(o, g, e, cfg["mass"]); ctx.synchronize()
print("mhat ok", lb.sqnorm(o), flush=True)
r = lb.cg_solve_eo(g, cfg["mass"], e, lb.CgSettings(cfg["tol"], 5000))
print("cg", r.iterations, r.true_rel_residual, r.seconds, flush=True)
PY
for c in 1 2; do
  for gr in 0 1; do
    echo "== cfg $c graph $gr"; LBCU_CG_FUSED_MHAT=1 LBCU_CG_GRAPH=$gr timeout 300 python /tmp/f.py $c 2>&1 | tail -5
  done
done
