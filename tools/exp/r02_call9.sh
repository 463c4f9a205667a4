# round 2: debug-check library (negative control included) + full default bench + C5 ncu refresh
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_c9.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c9.log
bash tools/debug_checks.sh run
timeout 900 python bench.py > gpurun_out/bench_c5_full.json 2> gpurun_out/bench_c5_full.err; echo "bench rc=$?"; cut -c1-200 gpurun_out/bench_c5_full.json
timeout 300 python bench.py --profile --steps 2 --warmup 1 > gpurun_out/prof_plain9.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_pair16 -s 2 -c 1 -o gpurun_out/prof_c5b python bench.py --profile --steps 2 --warmup 1 > gpurun_out/ncu_c5b.log 2>&1; echo "ncu rc=$?"
