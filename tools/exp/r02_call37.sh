cd $GRAFT_REPO_ROOT
for k in 20 40 100 200 20 100; do
  timeout 300 python bench.py --config C1 --no-e2e --no-cpu --no-check --steps $k --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K=$k', d['value'], d['roofline']['frac'], d['ms_per_step'], d['clocks'])"
done
