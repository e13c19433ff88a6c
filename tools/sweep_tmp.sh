timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 8 16; do
  echo "refresh_solves=$r: $(HC_AMG_REFRESH_SOLVES=$r timeout 150 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"], d["gpu_launches"])')"
done
for r in 8 16; do
  echo "large refresh_solves=$r: $(HC_AMG_REFRESH_SOLVES=$r timeout 250 python bench.py --config large --steps 6 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"], d["gpu_launches"])')"
done
