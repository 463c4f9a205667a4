# round 2: pageable e2e vs staging chunk size (C5)
cd $GRAFT_REPO_ROOT
for mb in 32 64 128 16; do
  QCB_HOST_CHUNK_MB=$mb timeout 600 python bench.py --no-cpu --no-check --no-encode --steps 3 --warmup 3 > gpurun_out/ck_$mb.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/ck_$mb.json'));print('chunk $mb MB', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pinned'])"
done
