#!/bin/bash
# C3 pair16 kernel: per-SASS-line shared-memory excess wavefronts (bank conflicts)
mkdir -p gpurun_out
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_plain_c3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o /tmp/prof_c3p -f \
  python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_c3.log 2>&1
ncu -i /tmp/prof_c3p.ncu-rep --page source --csv --print-source sass > gpurun_out/c3_sass.csv 2>&1
ncu -i /tmp/prof_c3p.ncu-rep --page raw --csv > gpurun_out/c3_raw.csv 2>&1
ls -la gpurun_out/c3_sass.csv
