timeout 300 python tools/stencil_ab.py large 2 3 2>&1 | grep -v Warn
timeout 300 python tools/stencil_ab.py medium 2 3 2>&1 | grep -v Warn
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
