# full GPU check: parity tests, then every BASELINE config through bench.py
set -o pipefail
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C2_full.log 2>&1; echo "bench C2 rc=$?"; tail -1 gpurun_out/bench_C2_full.log
for c in C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
