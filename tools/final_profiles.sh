#!/bin/bash
# Round-end ncu --set full captures (run on the GPU box): the standalone J v / residual stencils
# of bench.py's kernel-timing leg, and the step's top multigrid kernels inside one profiled step.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-r02f}
bash tools/ncu_kern.sh 'k_fine_tma<\(int\)0, \(int\)0, \(bool\)1>' ${T}_jv_standalone large
bash tools/ncu_kern.sh 'k_fine_tma<\(int\)4' ${T}_res_standalone large
cap() {  # regex tag count
  LS=0 HC_KRYLOV_WHILE=0 timeout 900 ncu --profile-from-start off --kernel-name-base demangled -k "regex:$1" \
    -c $3 --set full --import-source on --clock-control none -o gpurun_out/${T}_$2 -f \
    python tools/prof_step.py large > gpurun_out/${T}_$2.log 2>&1
  tail -1 gpurun_out/${T}_$2.log
}
cap 'k_sell_xp<\(int\)1, \(int\)0>' sell_l1 4
cap 'k_csr_xp<\(int\)8, \(int\)0>' csr8 2
cap 'k_restrict_v' restrict 4
cap 'k_prolong0_s' prolong0 2
cap 'k_fine_tma<\(int\)1, \(int\)(1|4)' fine_phi 2
cap 'k_dev_(xr|s|p)' krylov_vec 3
# text summaries on the box (the reports together exceed what gpurun copies back): details page of
# every report, one-screen brief of all, SASS hot lines of the two standalone stencils
: > gpurun_out/${T}_brief.txt
for f in gpurun_out/${T}_*.ncu-rep; do
  ncu -i $f --page details > ${f%.ncu-rep}_details.txt 2>/dev/null
  python tools/ncu_brief.py $f >> gpurun_out/${T}_brief.txt 2>&1
done
for k in jv_standalone res_standalone; do
  python tools/ncu_hot.py gpurun_out/${T}_$k.ncu-rep 30 > gpurun_out/${T}_${k}_hot.txt 2>&1
done
for f in gpurun_out/${T}_*.ncu-rep; do
  case $f in *standalone*) ;; *) rm -f $f ;; esac
done
du -sh gpurun_out
