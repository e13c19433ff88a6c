#!/bin/bash
# env-knob A/B on the medium bench: tools/ab.sh "" "HC_X=1" "HC_Y=2 HC_Z=3" ...
for s in "$@"; do
  r=$(env $s timeout 200 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"])')
  echo "[$s] $r"
done
