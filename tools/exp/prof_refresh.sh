#!/bin/bash
# Refresh the round-1 ncu evidence for the current build, plus the C3 SASS
# source page (per-line bank conflicts) and the C5 source page.
bash tools/exp/profile_r01.sh > gpurun_out/profile_r01.log 2>&1; echo "profile rc=$?"
ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o /tmp/prof_c3p -f \
  python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu -i /tmp/prof_c3p.ncu-rep --page source --csv --print-source sass > gpurun_out/c3_sass.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o /tmp/prof_c5p -f \
  python bench.py --config C5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-encode > /dev/null 2>&1
ncu -i /tmp/prof_c5p.ncu-rep --page source --csv --print-source sass > gpurun_out/c5_sass.csv 2>&1
ncu -i /tmp/prof_c5p.ncu-rep --page raw --csv > gpurun_out/c5_raw.csv 2>&1
ls -la gpurun_out
