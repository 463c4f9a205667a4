#!/bin/bash
# Round-1 profiles: launch list of the default bench command + one full capture
# per headline kernel, summarised on the box (tools/profile_summary.py).
# Each bench command is first run WITHOUT ncu (must exit 0).
mkdir -p gpurun_out
OUT=gpurun_out/r01_ncu_summary.json
rm -f $OUT
set -x
python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/p_plain_c2.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/p_ncu_list_c2.log 2>&1
python tools/profile_summary.py --launches gpurun_out/launches_c2.csv C2 gpurun_out/r01_launches_c2.json
ncu --set full --clock-control none --import-source on -k regex:decode_layered -s 2 -c 1 -o gpurun_out/prof_c2 -f \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_c2.log 2>&1
python tools/profile_summary.py gpurun_out/prof_c2.ncu-rep C2 $OUT
python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_plain_c5.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|encode" -c 100 --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_list_c5.log 2>&1
python tools/profile_summary.py --launches gpurun_out/launches_c5.csv C5 gpurun_out/r01_launches_c5.json
ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o gpurun_out/prof_c5 -f \
  python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_c5.log 2>&1
python tools/profile_summary.py gpurun_out/prof_c5.ncu-rep C5 $OUT && rm -f gpurun_out/prof_c5.ncu-rep
ncu --set full --clock-control none --import-source on -k regex:encode_z96 -s 1 -c 1 -o gpurun_out/prof_enc -f \
  python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_enc.log 2>&1
python tools/profile_summary.py gpurun_out/prof_enc.ncu-rep ENC $OUT && rm -f gpurun_out/prof_enc.ncu-rep
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_plain_c3.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o gpurun_out/prof_c3 -f \
  python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/p_ncu_c3.log 2>&1
python tools/profile_summary.py gpurun_out/prof_c3.ncu-rep C3 $OUT && rm -f gpurun_out/prof_c3.ncu-rep
ls -la gpurun_out
