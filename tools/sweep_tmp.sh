for ls in 0.1 0.3 1.0; do
  echo "ls=$ls: $(HC_BENCH_LINEAR_SAFETY=$ls timeout 150 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"], d["newton_iters_per_step"])')"
done
