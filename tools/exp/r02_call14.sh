# round 2: padded pair-block stride for multi-pair CTAs -- parity, C3 bench, ncu conflicts
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c14.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_c14.log
timeout 300 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/bench_c3_pad.json 2>/dev/null; echo "c3 rc=$?"; cut -c1-160 gpurun_out/bench_c3_pad.json
timeout 600 python tools/codebench.py --codes wifi-1944-r12,wifi-1944-r23A,wifi-1944-r34A,wifi-1944-r56 --arith i16 --w 262144 --iters 8 > gpurun_out/c14_native.log 2>&1; grep gbit gpurun_out/c14_native.log | cut -c1-100
timeout 300 python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/plain_c3c.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 3 -c 1 -o gpurun_out/prof_c3c python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/ncu_c3c.log 2>&1; echo ncu_c3=$?
