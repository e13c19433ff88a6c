for cfg in medium large; do
for cfgs in "2 2" "1 2" "1 1"; do
  set -- $cfgs
  echo "$cfg nu=$1 nu_c=$2: $(HC_AMG_NU=$1 HC_AMG_NU_C=$2 timeout 200 python bench.py --config $cfg --steps 6 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"], d["newton_iters_per_step"])')"
done; done
