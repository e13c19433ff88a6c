#!/bin/bash
# ncu --set full captures (with source) of the J v and residual stencils inside one profiled large-cell step
mkdir -p gpurun_out
cap() {  # regex tag count
  LS=0 HC_KRYLOV_WHILE=0 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k "regex:$1" \
    -c $3 --set full --import-source on --clock-control none -o gpurun_out/$2 -f \
    python tools/prof_step.py ${4:-large} > gpurun_out/$2.log 2>&1
  tail -1 gpurun_out/$2.log
}
cap 'k_fine_tma<\(int\)0, \(int\)0, \(bool\)1>' ${TAG:-s3}_ncu_jv 1
cap 'k_fine_tma<\(int\)4' ${TAG:-s3}_ncu_res 1
ls -la gpurun_out/*.ncu-rep
