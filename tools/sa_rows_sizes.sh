#!/bin/bash
# phi level-2 sizes of the batched cells (HC_AMG_VERBOSE)
cd "$(dirname "$0")/.."
HC_AMG_VERBOSE=1 timeout 500 python bench.py --config batched --steps 1 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "field 1 level 2" | awk '{print $6}' | sort | uniq -c | sort -k2 > gpurun_out/batched_l2.log
