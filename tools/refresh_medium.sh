#!/bin/bash
# Re-measure the default (medium) bench line and its launch list, plus smoke (run on the GPU box)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke2.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_medium.json 2> gpurun_out/bench_medium.err
HC_KRYLOV_WHILE=0 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/medium_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-at-scale \
  > gpurun_out/ncu_medium.log 2>&1
