# round 2: non-temporal staging copies (A/B QCB_NT_COPY) on C5's pageable e2e; host-path tests
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not debug" > gpurun_out/pytest_gpu_c25.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_c25.log
for nt in 1 0 1 0; do
  QCB_NT_COPY=$nt timeout 600 python bench.py --no-cpu --no-check --no-encode --steps 3 --warmup 3 > gpurun_out/nt$nt.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/nt$nt.json'));print('NT $nt', d['e2e']['value'], d['e2e']['ms_per_step'], d['e2e']['pinned'])"
done
