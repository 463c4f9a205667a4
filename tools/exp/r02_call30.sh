# round 2 (session 4): state check after the container was re-created: GPU suite, smoke, default bench, C1/C3 lines
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c30_pytest.log 2>&1; echo "pytest=$?"
timeout 300 python __graft_entry__.py --smoke > gpurun_out/c30_smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > gpurun_out/c30_bench_c5.log 2>&1; echo "bench=$?"
for c in C1 C3; do timeout 600 python bench.py --config $c > gpurun_out/c30_bench_$c.log 2>&1; echo "$c=$?"; done
tail -3 gpurun_out/c30_pytest.log; tail -1 gpurun_out/c30_bench_c5.log | cut -c1-600
