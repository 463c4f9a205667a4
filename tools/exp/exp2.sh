for lib in libqcb200.so libqcb200_t96_5.so libqcb200_t96_6.so libqcb200_t192_3.so; do
  for cw in 1 2; do
    echo "== $lib cw=$cw"
    QCB_LIB=$PWD/paper_2306_12063_b200/$lib QCB_F32_CW=$cw python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['ms_per_step'])"
  done
done
python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "goldens or 126" 2>&1 | tail -2
