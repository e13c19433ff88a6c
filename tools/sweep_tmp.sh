for d in 0 1; do
echo "batched newton_dev=$d: $(HC_NEWTON_DEV=$d timeout 500 python bench.py --config batched --steps 3 --warmup 3 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],1))')"
done
echo "batched newton_dev=1 threads=32: $(HC_BATCH_THREADS=32 HC_NEWTON_DEV=1 timeout 500 python bench.py --config batched --steps 3 --warmup 3 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],1))')"
