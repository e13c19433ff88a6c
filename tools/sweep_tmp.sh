for lib in paper_1704_04139_b200/libhalfcell_b200.so paper_1704_04139_b200/libhc_s5_c128.so paper_1704_04139_b200/libhc_s6_c128.so paper_1704_04139_b200/libhc_s8_c64.so paper_1704_04139_b200/libhc_s4_c128.so; do
  echo "$lib: $(HC_LIB=$lib timeout 120 python tools/stencil_ab.py large 3 2>&1 | grep kind) | $(HC_LIB=$lib timeout 120 python tools/stencil_ab.py medium 3 2>&1 | grep kind | cut -c1-60)"
done
