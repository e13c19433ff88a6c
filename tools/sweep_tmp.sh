timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for w in 1 0; do
echo "while=$w: $(HC_KRYLOV_WHILE=$w timeout 150 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"], d["gpu_launches"])')"
done
