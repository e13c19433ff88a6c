#!/bin/bash
# compile-time knob sweep of the persistent J v stencil (rebuilds hc_operator.o only):
#   tools/jv_variants.sh "" "-DHC_JV_STAGES=5 -DHC_JV_SLOTCAP=128" ...
cd "$(dirname "$0")/.."
C=paper_1704_04139_b200/csrc
for v in "$@"; do
  rm -f $C/hc_operator.o
  make -s -j8 -C $C EXTRA="$v" >/dev/null 2>&1 || { echo "[$v] build failed"; continue; }
  regs=$(grep -A3 "k_jv_tmaILb1ELb0" $C/hc_operator.o.ptxas.log | grep -o "Used [0-9]* registers" | head -1)
  k=$(timeout 120 python tools/jv_time.py large 20 2>&1 | tail -1)
  echo "[$v] $regs | $k"
done
rm -f $C/hc_operator.o; make -s -j8 -C $C >/dev/null 2>&1
