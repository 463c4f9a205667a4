#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 600 python tools/exp/percode.py > gpurun_out/percode.log 2>&1
cat gpurun_out/percode.log
for c in C2 C5 C3 C1 C4; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/bench_$c.log 2>&1
tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
