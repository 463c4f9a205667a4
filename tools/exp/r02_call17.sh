# round 2: parity + debug checks with the chunked plan; per-code refresh
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c17.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_c17.log
bash tools/debug_checks.sh run
timeout 900 python tools/codebench.py --codes all --w 65536 --json gpurun_out/final_codebench.json > /dev/null 2>&1; echo "codebench rc=$?"
