#!/bin/bash
# sliced-ELL lanes-per-row sweep on the large and medium cells (exact Krylov tolerance)
run() { echo "== $*"; env "$@" LS=0 timeout 300 python tools/steps_sweep.py large 16 2>&1 | tail -1; env "$@" LS=0 timeout 300 python tools/steps_sweep.py medium 30 2>&1 | tail -1; }
run X=0
run HC_AMG_SELL=512 HC_AMG_SELL_LANE=48
run HC_AMG_SELL=512 HC_AMG_SELL_LANE=16
run HC_AMG_SELL=512 HC_AMG_SELL_LANE=8
run HC_AMG_SELL=512 HC_AMG_SELL_LANE=32
run HC_AMG_SELL=512 HC_AMG_SELL_LANE=16 HC_AMG_SELL_ROWS=32768
run HC_AMG_SELL=512 HC_AMG_SELL_LANE=8 HC_AMG_SELL_ROWS=32768
