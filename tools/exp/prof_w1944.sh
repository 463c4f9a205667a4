#!/bin/bash
python tools/exp/one_code.py wifi 1944 1/2 f32 65536 || exit 1
ncu --set full --clock-control none -k regex:decode_layered -s 2 -c 1 -o gpurun_out/prof_w1944 -f python tools/exp/one_code.py wifi 1944 1/2 f32 65536 > /dev/null 2>&1
python tools/profile_summary.py gpurun_out/prof_w1944.ncu-rep W1944 gpurun_out/w1944.json > /dev/null
python tools/exp/one_code.py wifi 1944 5/6 i16 65536
ncu --set full --clock-control none -k regex:decode_pair16 -s 2 -c 1 -o gpurun_out/prof_w1944i -f python tools/exp/one_code.py wifi 1944 5/6 i16 65536 > /dev/null 2>&1
python tools/profile_summary.py gpurun_out/prof_w1944i.ncu-rep W1944I gpurun_out/w1944.json > /dev/null
