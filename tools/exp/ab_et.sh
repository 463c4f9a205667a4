#!/bin/bash
# A/B of early-termination variants (libs given as arguments) with tools/exp/et_perf.py
for lib in "$@"; do
  echo "== $lib"
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python tools/exp/et_perf.py 2>&1 | grep " ET "
done
