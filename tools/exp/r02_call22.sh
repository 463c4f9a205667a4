# round 2: pageable e2e vs host copy threads (C5)
cd $GRAFT_REPO_ROOT
nproc; grep -c processor /proc/cpuinfo; free -g | head -2
for t in 8 16 4 12; do
  QCB_COPY_THREADS=$t timeout 600 python bench.py --no-cpu --no-check --no-encode --steps 3 --warmup 3 > gpurun_out/e2e_t$t.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/e2e_t$t.json'));print('threads $t', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pinned'])"
done
