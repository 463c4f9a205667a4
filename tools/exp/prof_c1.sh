#!/bin/bash
mkdir -p gpurun_out
python bench.py --config C1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_plain_c1.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 3 -c 1 -o gpurun_out/prof_c1 -f python bench.py --config C1 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_c1.log 2>&1
python tools/profile_summary.py gpurun_out/prof_c1.ncu-rep C1 gpurun_out/c1.json > /dev/null
python tools/profile_summary.py --phases gpurun_out/prof_c1.ncu-rep C1 gpurun_out/c1.json > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|zero|fill" --csv --log-file gpurun_out/launches_c1.csv python bench.py --config C1 --steps 10 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
