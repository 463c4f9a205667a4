#!/bin/bash
# A/B libs on the int16 configs (C3 C5) + percode i16
for rep in 1 2; do
for lib in "$@"; do
  for c in C3 C5; do
    echo -n "$lib $c: "
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done
done
