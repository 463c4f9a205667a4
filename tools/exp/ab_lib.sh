#!/bin/bash
# usage: ab_lib.sh "C3 C5" libA.so libB.so ...  -- GPU parity suite on each
# non-default lib, then interleaved bench A/B (2 reps)
CFGS="$1"; shift
for lib in "$@"; do
  if [ "$lib" != "libqcb200.so" ]; then
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_$lib.log 2>&1; echo "$lib tests rc=$? $(tail -1 gpurun_out/t_$lib.log)"
  fi
done
for rep in 1 2; do
for c in $CFGS; do
for lib in "$@"; do
    echo -n "$lib $c: "
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
done
done
