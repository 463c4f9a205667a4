# round 2 (session 4): one-instruction hard-decision sign in the int16 syndrome (VIADDMNMX): suite, C5 / C3 lines, ET throughput
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c39_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c39_pytest.log
for rep in 1 2; do
for c in C5 C3; do
  timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
timeout 900 python tools/exp/et_perf.py > gpurun_out/c39_et.log 2>&1; echo "et=$?"; tail -12 gpurun_out/c39_et.log
