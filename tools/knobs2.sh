#!/bin/bash
cfg=$1; n=$2; shift; shift
for s in "$@"; do ( eval "export $s"; timeout 900 python tools/steps_sweep.py $cfg $n 2>&1 | tail -1 | sed "s/^/[$s] /" ); done
