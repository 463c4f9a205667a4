# round 2: parity with three pairs per CTA on the Z = 81 int16 codes (TMEM tiers incl.), C3 bench + ncu
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c13.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_c13.log
timeout 300 python bench.py --config C3 --no-cpu > gpurun_out/bench_c3_g3.json 2> gpurun_out/bench_c3_g3.err; echo "c3 rc=$?"; cut -c1-200 gpurun_out/bench_c3_g3.json
timeout 300 python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/plain_c3b.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 3 -c 1 -o gpurun_out/prof_c3b python bench.py --config C3 --profile --steps 3 --warmup 2 > gpurun_out/ncu_c3b.log 2>&1; echo ncu_c3=$?
