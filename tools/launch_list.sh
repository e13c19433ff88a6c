#!/bin/bash
# ncu launch list (gpu__time_duration.sum) of one profiled large-cell step at Krylov 1e-10, summarised
# usage: launch_list.sh <tag> [config]
mkdir -p gpurun_out
LS=0 HC_KRYLOV_WHILE=0 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$1_launches.csv python tools/prof_step.py ${2:-large} > gpurun_out/$1_launches.log 2>&1
python tools/launch_sum.py gpurun_out/$1_launches.csv > gpurun_out/$1_launches.txt; cat gpurun_out/$1_launches.txt
