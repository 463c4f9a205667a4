cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for p in 1 0; do
for k in 20 100 400; do
  QCB_PDL=$p timeout 300 python bench.py --config C1 --no-e2e --no-cpu --no-check --steps $k --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$p K=$k', d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
done
done
