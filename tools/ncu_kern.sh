#!/bin/bash
# ncu --set full capture (with source) of one kernel inside tools/jv_time.py (bench.py's kernel-timing leg)
# usage: ncu_kern.sh <kernel regex> <tag> [config] [launch-skip]
mkdir -p gpurun_out
timeout 600 ncu --kernel-name-base demangled -k "regex:$1" --launch-skip ${4:-0} -c 1 --set full --import-source on \
  --clock-control none -o gpurun_out/$2 -f python tools/jv_time.py ${3:-large} 1 > gpurun_out/$2.log 2>&1
tail -2 gpurun_out/$2.log
