#!/bin/bash
# compile-time knob sweep of the TMA stencil: tools/tma_variants.sh "" "-DHC_TMA_SLOTCAP=128" ...
# each variant: rebuild, large-grid kernel timings, medium step rate
cd "$(dirname "$0")/.."
for v in "$@"; do
  make -s -C paper_1704_04139_b200/csrc clean >/dev/null
  make -s -j8 -C paper_1704_04139_b200/csrc EXTRA="$v" >/dev/null 2>&1 || { echo "[$v] build failed"; continue; }
  regs=$(grep -A3 "k_fine_tmaILi0ELi0ELb1" paper_1704_04139_b200/csrc/hc_operator.o.ptxas.log | grep -o "Used [0-9]* registers" | head -1)
  k=$(timeout 300 python tools/stencil_ab.py large 3 2>/dev/null | grep kind)
  s=$(timeout 200 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"])')
  echo "[$v] $regs | $k | medium $s"
done
make -s -C paper_1704_04139_b200/csrc clean >/dev/null; make -s -j8 -C paper_1704_04139_b200/csrc >/dev/null 2>&1
