#!/bin/bash
# GPU tests + per-code sweep + C2/C5 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python tools/exp/percode.py > gpurun_out/percode.log 2>&1
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c5.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c2.log 2>&1
tail -3 gpurun_out/gpu_tests.log
