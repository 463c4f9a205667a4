cd $GRAFT_REPO_ROOT
python tools/exp/et_one.py wifi 648 1/2 i16 2.5 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 1 -c 1 -o gpurun_out/prof_et648 -f python tools/exp/et_one.py wifi 648 1/2 i16 2.5 > gpurun_out/c47_ncu.log 2>&1; echo "ncu=$?"
ncu -i gpurun_out/prof_et648.ncu-rep --page source --csv --print-source sass > gpurun_out/et648_sass.csv 2>&1
ncu -i gpurun_out/prof_et648.ncu-rep --page raw --csv > gpurun_out/et648_raw.csv 2>&1
ls -la gpurun_out/et648_sass.csv
