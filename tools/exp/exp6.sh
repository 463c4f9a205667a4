for rep in 1 2; do
for lib in libqcb200.so libqcb200_nr.so; do
  for c in C2 C5; do
    echo "== $lib $c"
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['clocks'])"
  done
done
done
