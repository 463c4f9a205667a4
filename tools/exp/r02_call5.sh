# round 2: parity incl. the scaled plan-size test; per-code refresh; C3 bench with its address table
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_c5.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c5.log
timeout 900 python tools/codebench.py --codes all --w 65536 --json gpurun_out/ct3_default.json > /dev/null 2>&1; echo "default rc=$?"
timeout 300 python bench.py --config C3 --no-cpu --no-e2e > gpurun_out/bench_c3b.json 2> gpurun_out/bench_c3b.err; echo "c3 rc=$?"; cut -c1-200 gpurun_out/bench_c3b.json
