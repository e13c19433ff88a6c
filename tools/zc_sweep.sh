#!/bin/bash
# z-chunking sweep: medium bench steps/s and large-grid kernel times per (HC_ZC_TARGET, HC_ZC_MIN)
for c in "12 2" "12 4" "12 5" "12 6" "6 5" "8 5" "6 8" "4 5"; do
  set -- $c
  b=$(HC_ZC_TARGET=$1 HC_ZC_MIN=$2 timeout 200 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"])')
  l=$(HC_ZC_TARGET=$1 HC_ZC_MIN=$2 timeout 100 python tools/stencil_ab.py large 3 2>&1 | grep kind)
  m=$(HC_ZC_TARGET=$1 HC_ZC_MIN=$2 timeout 100 python tools/stencil_ab.py medium 3 2>&1 | grep kind)
  echo "T=$1 MIN=$2 | bench $b | large $l | medium $m"
done
