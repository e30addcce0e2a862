#!/bin/bash
# Usage (GPU box): TAG=r2a bash tools/r2_measure.sh — GPU tests, the default bench line,
# the reference arm and one driver report in every format, under gpurun_out/$TAG.
TAG=${TAG:-r2}
set -x
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG/smi.txt 2>&1
lscpu > gpurun_out/$TAG/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/$TAG/gputest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/$TAG/bench_ref.json 2> gpurun_out/$TAG/bench_ref.err; echo "ref rc=$?"
printf 'test = balance\nlattice = 16x8x8x8\ngrid = 1x1x1x1\nenforce_local_floor = false\nspinor_fields = 3\nmass = 0.1\nkernel_seconds = 0.05\ncg_tolerance = 1e-10\nseed = 1\nbc_time = antiperiodic\neo = true\n' > gpurun_out/$TAG/p.params
tools/latbench_b200 run gpurun_out/$TAG/p.params --format json --emit-all gpurun_out/$TAG/report > /dev/null; echo "report rc=$?"
tail -5 gpurun_out/$TAG/gputest.log
