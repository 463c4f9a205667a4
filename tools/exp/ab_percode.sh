#!/bin/bash
# per-code A/B of libs given as arguments (tools/exp/percode.py), f32 rows only
for lib in "$@"; do
  echo "== $lib"
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 900 python tools/exp/percode.py 2>&1 | grep "'f32'"
done
