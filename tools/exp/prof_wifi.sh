#!/bin/bash
mkdir -p gpurun_out
python tools/exp/one_code.py wifi 648 1/2 f32 65536 || exit 1
ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 2 -c 1 -o gpurun_out/prof_w648 -f python tools/exp/one_code.py wifi 648 1/2 f32 65536 > gpurun_out/p_w648.log 2>&1
python tools/profile_summary.py gpurun_out/prof_w648.ncu-rep W648 gpurun_out/w648.json > /dev/null
python tools/profile_summary.py --phases gpurun_out/prof_w648.ncu-rep W648 gpurun_out/w648.json > /dev/null
