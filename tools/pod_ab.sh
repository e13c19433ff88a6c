#!/bin/bash
# compile-time A/B of the DMMA GEMM (hc_pod.cu only): tools/pod_ab.sh "" "-DHC_DGEMM_MINB=4" ...
cd "$(dirname "$0")/.."
C=paper_1704_04139_b200/csrc
for v in "$@"; do
  rm -f $C/hc_pod.o
  make -s -j8 -C $C EXTRA="$v" >/dev/null 2>&1 || { echo "[$v] build failed"; continue; }
  regs=$(grep -A2 "k_dgemmILb1ELb1" $C/hc_pod.o.ptxas.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' ')
  t=$(timeout 300 python -m pytest tests/test_gpu_batch_pod.py -m gpu -x -q 2>&1 | tail -1)
  r=$(timeout 300 python bench.py --config pod --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print("gram %.2f ms %.1f TF/s frac %.3f | projection %.2f ms frac %.3f | err %.1e" % (d["ms_per_step"], d["value"]/1e3, d["roofline"]["frac"], d["projection"]["ms"], d["projection"]["frac_of_dmma_peak"], d["max_rel_err_vs_cublas"]))')
  echo "[$v] $regs | $t | $r"
done
rm -f $C/hc_pod.o; make -s -j8 -C $C >/dev/null 2>&1
