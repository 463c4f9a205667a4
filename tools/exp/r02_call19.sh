# round 2: L2 prefetch of the next wave's LLR chunks (A/B with QCB_PF=0)
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c19.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c19.log
for pf in 1 0 2; do
  for c in C5 C2 C3; do
    QCB_PF=$pf timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-check > gpurun_out/pf${pf}_$c.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/pf${pf}_$c.json'));print('PF=$pf $c', d['value'], d['roofline']['frac'])"
  done
done
