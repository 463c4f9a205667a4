timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -2
for c in C2 C3 C5 C4 C1; do
  echo "== $c"
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
done
echo "== C5 TMEM"; QCB_TMEM=1 timeout 300 python bench.py --config C5 --steps 5 --warmup 2 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
