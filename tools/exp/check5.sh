#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests.log
for c in C2 C5 C3 C4 C1; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/bench_$c.log 2>&1
echo -n "$c "; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
