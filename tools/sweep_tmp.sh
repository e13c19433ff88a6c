for zc in 0 3 6 12 24; do
  echo "medium zc=$zc: $(HC_ZC_TARGET=$zc timeout 120 python tools/stencil_ab.py medium 3 2>&1 | grep kind)"
done
for zc in 0 6 18; do
  echo "large zc=$zc: $(HC_ZC_TARGET=$zc timeout 120 python tools/stencil_ab.py large 3 2>&1 | grep kind)"
done
