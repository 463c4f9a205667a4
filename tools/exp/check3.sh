#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
timeout 600 python tools/exp/percode.py > gpurun_out/percode.log 2>&1
grep i16 gpurun_out/percode.log
for c in C5 C3; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/bench_$c.log 2>&1
tail -1 gpurun_out/bench_$c.log | cut -c1-200
done
