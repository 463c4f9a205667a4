# round 2 (session 4): per-structure FFMA2 sign application: suite, C1 / C2 / C4 lines, all 126 codes x both arithmetics
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/c41_pytest.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/c41_pytest.log
for c in C2 C4 C1; do
  timeout 600 python bench.py --config $c > gpurun_out/c41_bench_$c.log 2>&1; tail -1 gpurun_out/c41_bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
timeout 1800 python tools/codebench.py --codes all --arith f32,i16 --w 65536 --json gpurun_out/codebench_all.json > gpurun_out/c41_codebench.log 2>&1; echo "codebench=$?"
