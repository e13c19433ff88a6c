#!/bin/bash
# ncu --set full captures of the large cell's top preconditioner kernels and the J v stencil
# (the first launches inside tools/prof_step.py's profiled step; run on the GPU box)
mkdir -p gpurun_out
cap() {  # regex tag count
  LS=0 HC_KRYLOV_WHILE=0 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k "regex:$1" \
    -c $3 --set full --import-source on --clock-control none -o gpurun_out/r02_ncu_$2 -f \
    python tools/prof_step.py large > gpurun_out/r02_ncu_$2.log 2>&1
  tail -1 gpurun_out/r02_ncu_$2.log
}
cap 'k_csr_x<\(int\)8, float, \(int\)0>' csr8 2
cap 'k_csr_x<\(int\)32, float, \(int\)1>' csr32 2
cap 'k_restrict_v' restrict 4
cap 'k_prolong0_s' prolong0 2
cap 'k_fine_tma<\(int\)1, \(int\)4' fine_phi_resid0 1
cap 'k_fine_tma<\(int\)0, \(int\)0, \(bool\)1>|k_jv_y' jv 1
cap 'k_fine_tma<\(int\)4' residual 1
ls -la gpurun_out/*.ncu-rep
