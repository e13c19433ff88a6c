#!/bin/bash
# headline only: large-cell step rate (no CPU baseline, no other configs); prints ms/step and Krylov iterations
timeout ${T:-300} python bench.py --no-cpu-baseline --no-at-scale --no-inexact --no-config0 --no-other-configs "$@" 2>/dev/null \
  | python3 -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print("ms/step %.2f  steps/s %.3f  krylov/step %.1f  newton/step %.1f  e2e %.3f  jv %.1f us" % (d["ms_per_step"], d["value"], d["krylov_iters_per_step"], d["newton_iters_per_step"], d["e2e"]["value"], d["kernel_ms"]["jvp_stencil"]*1e3))'
