#!/bin/bash
# A/B: default lib vs variant libs on C5 / C3 (and C2 sanity)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "126 or golden or KAT or known" > gpurun_out/ab_tests.log 2>&1; tail -1 gpurun_out/ab_tests.log
for rep in 1 2; do
for lib in "$@"; do
  for c in C5 C3; do
    echo -n "$lib $c: "
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done
done
