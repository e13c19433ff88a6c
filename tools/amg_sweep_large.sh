#!/bin/bash
# AMG knob sweep on a config at the exact Krylov tolerance (LS=0): steps/s and Krylov
# iterations per step for each setting (run on the GPU box; one line per setting).
cfg=${1:-large}; n=${2:-16}
run() { echo "== $*"; env "$@" LS=0 timeout 300 python tools/steps_sweep.py $cfg $n 2>&1 | tail -1; }
run X=0
run HC_AMG_PRE_C=1 HC_AMG_POST_C=1
run HC_AMG_GAMMA=2 HC_AMG_WMIN=1 HC_AMG_WDEPTH=1
run HC_AMG_GAMMA=2 HC_AMG_WMIN=2 HC_AMG_WDEPTH=3
run HC_AMG_GAMMA=2 HC_AMG_WMIN=3 HC_AMG_WDEPTH=5
run HC_AMG_NU=2 HC_AMG_NU_C=2
run HC_AMG_OMEGA=0.8
run HC_AMG_OMEGA=1.0
run HC_AMG_SA_LEVELS=1
run HC_AMG_SA_LEVELS=3
run HC_AMG_SA_ROWS=0
run HC_AMG_CF=3
run HC_AMG_OMEGA_P=0.5
run HC_AMG_OMEGA_P=0.8
run HC_AMG_COARSE_MAX=64
run HC_AMG_BDIAG=0
run HC_AMG_SA_C=1
run HC_AMG_NU_C0=2
