timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -3
for tm in 0 1; do
  for c in C2 C3; do
    echo "== QCB_TMEM=$tm $c"
    QCB_TMEM=$tm timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done
QCB_TMEM=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "goldens or 126" 2>&1 | tail -2
