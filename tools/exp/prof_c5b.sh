#!/bin/bash
mkdir -p gpurun_out
python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/p_plain_c5.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o gpurun_out/prof_c5q -f \
  python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/p_ncu_c5.log 2>&1
