#!/bin/bash
# Re-measure the bench lines and the launch list committed under profiles/ (run on the GPU box)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_medium.json 2> gpurun_out/bench_medium.err
for c in large batched rom pod; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
HC_KRYLOV_WHILE=0 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/medium_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-at-scale \
  > gpurun_out/ncu_medium.log 2>&1
tail -c 300 gpurun_out/bench_*.json
