#!/bin/bash
# GPU tests, smoke, and the large / batched bench lines (run on the GPU box)
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests4.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke4.log 2>&1
timeout 600 python bench.py --config large --no-cpu-baseline > gpurun_out/bench_large.json 2> gpurun_out/bench_large.err
timeout 600 python bench.py --config batched --no-cpu-baseline > gpurun_out/bench_batched.json 2> gpurun_out/bench_batched.err
