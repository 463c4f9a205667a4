#!/bin/bash
mkdir -p gpurun_out
QCB_SLOTS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/slots_tests.log 2>&1; tail -1 gpurun_out/slots_tests.log
for v in "default:0" "slots:1"; do
  IFS=: read name sl <<< "$v"
  for c in C2 C5 C3; do
    echo -n "$name $c: "
    QCB_SLOTS=$sl timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done
