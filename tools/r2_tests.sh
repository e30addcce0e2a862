#!/bin/bash
# Usage (GPU box): TAG=r2b bash tools/r2_tests.sh — the GPU test suite and smoke().
TAG=${TAG:-r2}
mkdir -p gpurun_out/$TAG
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/$TAG/gputest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"
tail -15 gpurun_out/$TAG/gputest.log
