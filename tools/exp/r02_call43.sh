# round 2 (session 4): int16 early termination writes a converged lane's outputs at once (no snapshot block): suite, ET table, C5 / C3 unchanged?
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c43_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c43_pytest.log
timeout 900 python tools/exp/et_perf.py > gpurun_out/c43_et.log 2>&1; echo "et=$?"; grep i16 gpurun_out/c43_et.log
for c in C5 C3; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
