# round 2 (session 4): two-lanes-per-row small-batch kernel (decode_split.cuh): parity, C1 scaling with / without it, C1 bench (ring timing)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "small_batch or all_126 or goldens or misaligned or empty" > gpurun_out/c31_pytest.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/c31_pytest.log
timeout 300 python tools/exp/c1_scaling.py > gpurun_out/c31_scaling_split.log 2>&1; echo "split=$?"; cat gpurun_out/c31_scaling_split.log
QCB_SPLIT_MAX_W=0 timeout 300 python tools/exp/c1_scaling.py > gpurun_out/c31_scaling_one.log 2>&1; echo "one=$?"; cat gpurun_out/c31_scaling_one.log
QCB_SPLIT_MAX_W=100000 timeout 300 python tools/exp/c1_scaling.py > gpurun_out/c31_scaling_all.log 2>&1; echo "all=$?"; cat gpurun_out/c31_scaling_all.log
timeout 600 python bench.py --config C1 > gpurun_out/c31_bench_C1.log 2>&1; echo "C1=$?"; tail -1 gpurun_out/c31_bench_C1.log | cut -c1-300
QCB_SPLIT_MAX_W=0 timeout 600 python bench.py --config C1 --no-e2e --no-cpu > gpurun_out/c31_bench_C1_one.log 2>&1; echo "C1one=$?"; tail -1 gpurun_out/c31_bench_C1_one.log | cut -c1-300
