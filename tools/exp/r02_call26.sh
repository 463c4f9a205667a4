# round 2: packed hard decisions through the pageable host path (A/B QCB_HOST_UNPACKED)
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c26.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c26.log
for v in packed unpacked packed unpacked; do
  if [ $v = unpacked ]; then export QCB_HOST_UNPACKED=1; else unset QCB_HOST_UNPACKED; fi
  timeout 600 python bench.py --no-cpu --no-check --no-encode --steps 3 --warmup 3 > gpurun_out/hp_$v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/hp_$v.json'));print('$v', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pinned'])"
done
unset QCB_HOST_UNPACKED
timeout 600 python bench.py --config C2 --no-cpu --no-check --steps 3 --warmup 3 > gpurun_out/hp_c2.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/hp_c2.json'));print('C2', d['e2e'])"
