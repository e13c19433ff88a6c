#!/bin/bash
# c-block smoothed first transfer (HC_AMG_SA_C=1): large and batched step rates
cd "$(dirname "$0")/.."
bash tools/amg_sa_ab.sh -- "HC_AMG_SA_C=1" "" > gpurun_out/sac.log 2>&1
for s in "HC_AMG_SA_C=1" ""; do
  r=$(env $s timeout 500 python bench.py --config batched --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2))')
  echo "[$s] batched $r" >> gpurun_out/sac.log
done
