#!/bin/bash
# A/B libs on the float32 configs (C2 C4 C1), 2 reps, + parity tests on each variant
mkdir -p gpurun_out
for lib in "$@"; do
  echo -n "$lib tests: "; QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
done
for rep in 1 2; do
for lib in "$@"; do
  for c in C2 C4 C1; do
    echo -n "$lib $c: "
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done
done
