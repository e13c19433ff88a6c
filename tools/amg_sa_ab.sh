#!/bin/bash
# smoothed-prolongator depth A/B: medium (tools/ab.sh) and large step rates
#   tools/amg_sa_ab.sh "<medium knobs>..." -- "<large knobs>..."
cd "$(dirname "$0")/.."
med=(); lrg=(); side=m
for a in "$@"; do
  if [ "$a" = "--" ]; then side=l; continue; fi
  if [ $side = m ]; then med+=("$a"); else lrg+=("$a"); fi
done
[ ${#med[@]} -gt 0 ] && bash tools/ab.sh "${med[@]}"
for s in "${lrg[@]}"; do
  r=$(env $s timeout 400 python bench.py --config large --steps 10 --warmup 3 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],3), d.get("krylov_iters_per_step"))')
  echo "[$s] large $r"
done
