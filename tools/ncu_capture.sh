#!/bin/bash
# Usage (on the GPU box): tools/ncu_capture.sh NAME SKIP COUNT -- <command...>
# Runs the command once plainly, then one `ncu --set full` capture of
# hop_kernel launches, exports the raw page as CSV + the source page, and
# deletes the .ncu-rep so gpurun_out stays small.
set -e
name=$1; skip=$2; count=$3; shift 4
"$@" > gpurun_out/${name}_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hop_kernel -s "$skip" -c "$count" \
    -o gpurun_out/${name} "$@" > gpurun_out/${name}_ncu.log 2>&1
ncu -i gpurun_out/${name}.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
ncu -i gpurun_out/${name}.ncu-rep --page source --csv > gpurun_out/${name}_source.csv 2>/dev/null || true
rm -f gpurun_out/${name}.ncu-rep
