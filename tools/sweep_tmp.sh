timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 300 python tools/stencil_ab.py large 2 3 2>&1 | grep -v Warn
timeout 300 python tools/stencil_ab.py medium 3 2>&1 | grep kind
echo "medium: $(timeout 150 python bench.py --steps 10 --no-cpu-baseline --no-at-scale 2>/dev/null | python3 -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],2), d["krylov_iters_per_step"], d["roofline"]["frac"])')"
