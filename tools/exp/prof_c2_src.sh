#!/bin/bash
# C2 pair16 kernel: per-SASS-line shared-memory excess wavefronts (bank conflicts)
mkdir -p gpurun_out
python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_plain_c2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 1 -c 1 -o /tmp/prof_c2p -f \
  python bench.py --config C2 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_c2.log 2>&1
ncu -i /tmp/prof_c2p.ncu-rep --page source --csv --print-source sass > gpurun_out/c2_sass.csv 2>&1
ncu -i /tmp/prof_c2p.ncu-rep --page raw --csv > gpurun_out/c2_raw.csv 2>&1
ls -la gpurun_out/c2_sass.csv
