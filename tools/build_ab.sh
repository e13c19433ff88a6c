#!/bin/bash
# compile-time A/B on the large-cell headline: tools/build_ab.sh "" "-DHC_TMA_DOTPF=0" ...
# each variant: full rebuild with EXTRA flags, headline step rate (quick_bench); default build restored
cd "$(dirname "$0")/.."
C=paper_1704_04139_b200/csrc
for v in "$@"; do
  make -s -C $C clean >/dev/null
  make -s -j8 -C $C EXTRA="$v" >/dev/null 2>&1 || { echo "[$v] build failed"; continue; }
  regs=$(grep -A3 "k_fine_tmaILi0ELi0ELb1" $C/hc_operator.o.ptxas.log | grep -o "Used [0-9]* registers" | head -1)
  spill=$(grep -A3 "k_fine_tmaILi0ELi0ELb1" $C/hc_operator.o.ptxas.log | grep -o "[0-9]* bytes spill stores" | head -1)
  k=$(timeout 200 python tools/jv_time.py large 20 2>&1 | tail -1)
  r=$(bash tools/quick_bench.sh --steps ${STEPS:-10} --warmup 3 2>&1 | tail -1)
  echo "[$v] $regs, $spill | $k | $r"
done
make -s -C $C clean >/dev/null; make -s -j8 -C $C >/dev/null 2>&1
