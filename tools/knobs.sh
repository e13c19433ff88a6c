#!/bin/bash
# usage: tools/knobs.sh CONFIG "ENV=..;ENV=.." ...
cfg=$1; shift
for s in "$@"; do
  ( eval "export $s"; timeout 600 python tools/amg_sweep.py $cfg 2,${HC_AMG_OMEGA:-0.6},1.0 2>&1 | tail -1 | sed "s/^/[$s] /" )
done
