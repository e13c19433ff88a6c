for cfg in "1 1" "0 1" "1 0" "0 0"; do set -- $cfg
echo "newton_dev=$1 pdl=$2: $(HC_NEWTON_DEV=$1 HC_PDL=$2 timeout 150 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2))')"
done
