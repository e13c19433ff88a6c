#!/bin/bash
# third smoothed transfer by level size (HC_AMG_SA_ROWS / HC_AMG_SA_ROWS_MIN): medium, large and batched step rates
cd "$(dirname "$0")/.."
bash tools/amg_sa_ab.sh "" "HC_AMG_SA_ROWS=0" -- "" > gpurun_out/sa_rows2.log 2>&1
for s in "" "HC_AMG_SA_ROWS=0"; do
  r=$(env $s timeout 500 python bench.py --config batched --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2))')
  echo "[$s] batched $r" >> gpurun_out/sa_rows2.log
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests3.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests3.log
