#!/bin/bash
# A/B libs over C2 C5 C3 C4 C1 (1 rep) + parity tests on the default lib
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/ab_tests.log 2>&1; tail -1 gpurun_out/ab_tests.log
for lib in "$@"; do
  for c in C2 C5 C3 C4 C1; do
    echo -n "$lib $c: "
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done
