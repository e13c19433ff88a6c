for lib in paper_1704_04139_b200/libhalfcell_b200.so paper_1704_04139_b200/libhc_s6.so; do for zc in 12 6; do
  echo "$lib zc=$zc: $(HC_LIB=$lib HC_ZC_TARGET=$zc timeout 120 python tools/stencil_ab.py large 3 2>&1 | grep kind)"
done; done
