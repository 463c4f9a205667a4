# round 2: final scaled plan (TMEM for R5/6 f32 Z = 68-76 restored, v1 caps accounted) -- parity + per-code refresh
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c18.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c18.log
timeout 900 python tools/codebench.py --codes all --w 65536 --json gpurun_out/final_codebench.json > /dev/null 2>&1; echo "codebench rc=$?"
