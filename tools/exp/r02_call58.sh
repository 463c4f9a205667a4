cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for lib in libqcb200.so lib_fa.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config C1 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C1', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config C4 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib C4', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
