#!/bin/bash
# env-knob A/B on the batched parameter study (config 3): tools/batched_knobs.sh "" "HC_AMG_FUSE_ROWS=6000" ...
cd "$(dirname "$0")/.."
for s in "$@"; do
  r=$(env $s timeout 400 python bench.py --config batched --no-cpu-baseline --steps ${STEPS:-3} --warmup 1 2>/dev/null \
      | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("%.1f cell-steps/s  %.1f ms/step  krylov/cell-step %.1f" % (d["value"], d["ms_per_step"], d.get("krylov_iters_per_cell_step", -1)))')
  echo "[$s] $r"
done
