#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "encode or foreign" > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5.log 2>&1
tail -3 gpurun_out/gpu_tests.log
tail -1 gpurun_out/bench_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['encode']))"
