#!/bin/bash
# One ncu --set full capture of one kernel of tools/run_layer.py (GPU box).
#   tools/capture.sh NAME KERNEL_REGEX SKIP run_layer-args...
# Runs the command once without ncu first (it must exit 0), then the capture
# into gpurun_out/NAME.ncu-rep.
set -e
name=$1; kre=$2; skip=$3; shift 3
python tools/run_layer.py "$@" --iters 2 > gpurun_out/$name.plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" \
  --launch-skip "$skip" -c 1 -o gpurun_out/$name -f python tools/run_layer.py "$@" --iters 2 \
  > gpurun_out/$name.ncu.log 2>&1
