# C3 / C5 re-sweep of the TMEM tier count and the TMEM register cap on the final kernels (three pairs per CTA, address table)
cd $GRAFT_REPO_ROOT
for c in C3 C5; do
for lib in libqcb200.so lib_tmt2.so lib_tmt4.so lib_cap120.so lib_cap112.so; do
  QCB_LIB=$PWD/paper_2306_12063_b200/$lib timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-encode 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $c', d['value'], d['roofline']['frac'], d['ms_per_step'], d['check']['result'])"
done
done
