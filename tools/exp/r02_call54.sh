# round 2 (session 4): per-structure TMEM register cap (C5 code and Wi-Fi 1944 R3/4 at 112): suite, default bench, C3, Wi-Fi 1944 R3/4
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c54_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c54_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/c54_smoke.log 2>&1; echo "smoke=$?"
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/c54_bench.log 2>&1; echo "bench=$?"; tail -1 gpurun_out/c54_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'], d['e2e']['value'], d['e2e']['pinned']['value'])"
timeout 600 python bench.py --config C3 > gpurun_out/c54_bench_C3.log 2>&1; tail -1 gpurun_out/c54_bench_C3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
timeout 600 python tools/codebench.py --codes wimax-2304-r34A,wimax-2304-r56,wifi-1944-r34A,wifi-1944-r56 --arith i16 --w 262144 2>&1 | grep gbit_s | cut -c1-90
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 3 -c 1 -o gpurun_out/prof_final_C5 -f python bench.py --config C5 --steps 3 --warmup 3 --no-cpu --no-e2e --no-encode > gpurun_out/c54_ncu.log 2>&1; echo "ncu=$?"
ncu -i gpurun_out/prof_final_C5.ncu-rep --page source --csv --print-source sass > gpurun_out/final_C5_sass.csv 2>&1
