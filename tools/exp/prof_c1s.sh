#!/bin/bash
QCB_SPLIT=1 python bench.py --config C1 --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1 || exit 1
QCB_SPLIT=1 ncu --set full --clock-control none --import-source on -k regex:decode_split -s 3 -c 1 -o gpurun_out/prof_c1s -f python bench.py --config C1 --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
python tools/profile_summary.py gpurun_out/prof_c1s.ncu-rep C1S gpurun_out/c1s.json > /dev/null
python tools/profile_summary.py --phases gpurun_out/prof_c1s.ncu-rep C1S gpurun_out/c1s.json > /dev/null
