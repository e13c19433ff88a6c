#!/bin/bash
# env-knob A/B on the large-cell headline (Krylov 1e-10): coarse-tail fusion, graph form
#   tools/tail_knobs.sh "" "HC_AMG_FUSE_ROWS=3000" ...
cd "$(dirname "$0")/.."
for s in "$@"; do
  r=$(env $s bash tools/quick_bench.sh --steps ${STEPS:-10} --warmup 3 2>&1 | tail -1)
  echo "[$s] $r"
done
