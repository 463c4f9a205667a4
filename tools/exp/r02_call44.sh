# round 2 (session 4): int16 early-termination flag by byte stores instead of atomicOr: suite, ET table
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c44_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c44_pytest.log
timeout 900 python tools/exp/et_perf.py > gpurun_out/c44_et.log 2>&1; echo "et=$?"; grep i16 gpurun_out/c44_et.log
