# round 2 (session 4): final validation of the committed build: GPU suite, smoke, default bench (C5), reference arm
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c46_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c46_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/c46_smoke.log 2>&1; echo "smoke=$?"; tail -1 gpurun_out/c46_smoke.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/c46_ref.log 2>&1; echo "ref=$?"; tail -1 gpurun_out/c46_ref.log | cut -c1-260
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/c46_bench.log 2>&1; echo "bench=$?"; tail -1 gpurun_out/c46_bench.log | cut -c1-260
