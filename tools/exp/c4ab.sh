timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "grouped" 2>&1 | tail -3
for rep in 1 2; do
for v in 1 0; do
  if [ $v = 1 ]; then export QCB_GROUPED_SERIAL=1; else unset QCB_GROUPED_SERIAL; fi
  echo -n "serial=$v C4: "; timeout 300 python bench.py --config C4 --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
done; done
