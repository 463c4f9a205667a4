# C3 (and C5) against single-knob variants of the final int16 kernel: late table fetch, anchor-only 3-input minima, per-tier TMEM store wait, caps 124 / 116
cd $GRAFT_REPO_ROOT
for c in C3 C5; do
for lib in libqcb200.so lib_tl1.so lib_m31.so lib_tw0.so lib_c124.so lib_c116.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
