# round 2: parity incl. the (now non-vacuous) scaled plan-size test; native int16 multi-pair plan; debug run
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c11.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_c11.log
timeout 600 python tools/codebench.py --codes wifi-1944-r12,wifi-1944-r23A,wifi-1944-r56 --arith i16 --w 262144 --iters 8 > gpurun_out/c11_native.log 2>&1; grep gbit gpurun_out/c11_native.log | cut -c1-120
bash tools/debug_checks.sh run
